// Exact (mults, adds) tallies of the reference walk, computed on the host.
//
// The reference kernels return, next to the transformed words, how many ring
// multiplications and additions their depth-first walk performed
// (_kernels.pyx:415-480; the pure walk counts the same, test_backends.py:43,
// 49,64,91).  The GPU schedule does different work, but the tallies are a
// function of the node lengths alone, so they are reproduced here exactly:
//
//  * node (q, r) has length m = ceil((n - q) / 2^r); its even child has
//    ceil(m/2) words, its odd child floor(m/2) (tree.py:20-54), so every
//    subtree is determined by its length;
//  * forward (tft_core, _kernels.pyx:305-335) is a post-order walk: even
//    child, odd_tail if m is odd, odd child, then the node's butterflies;
//    inverse (itft_core, :338-363): butterflies, odd child, odd_tail, even
//    child;
//  * the only state carried between nodes is whether the level base root
//    (ensure_base, :109-119) and its inverse (:125-128) exist yet, and the
//    four-slot LRU of tail roots keyed by `half` (tail_roots_k, :138-164).
//
// A subtree's cost is memoised on (length, state), so a length-n tally takes
// O(log n) distinct subtrees instead of the reference's O(n) node visits.
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

namespace tftb {

struct TallyState {
    bool has_base = false, has_inv = false;
    int64_t lru[4] = {-1, -1, -1, -1};  // tail-root halves, most recent first
    auto key() const { return std::make_tuple(has_base, has_inv, lru[0], lru[1], lru[2], lru[3]); }
};

class TallyWalk {
   public:
    TallyWalk(uint64_t p, int K, int kstar) : p_(p), K_(K), kstar_(kstar) {}

    // cost of the forward / inverse walk over a node of length m
    void walk(int64_t m, bool inverse, TallyState& s, int64_t& mu, int64_t& ad) {
        if (m <= 1) return;
        auto key = std::make_tuple(m, inverse, s.key());
        auto it = memo_.find(key);
        if (it != memo_.end()) {
            mu += it->second.mu;
            ad += it->second.ad;
            s = it->second.out;
            return;
        }
        int64_t m0 = 0, a0 = 0;
        const int64_t even = (m + 1) >> 1, odd = m >> 1;
        if (!inverse) {
            walk(even, false, s, m0, a0);
            if (m & 1) odd_tail(m, s, m0, a0);
            walk(odd, false, s, m0, a0);
            butterflies(m, false, s, m0, a0);
        } else {
            butterflies(m, true, s, m0, a0);
            walk(odd, true, s, m0, a0);
            if (m & 1) odd_tail(m, s, m0, a0);
            walk(even, true, s, m0, a0);
        }
        memo_[key] = Memo{m0, a0, s};
        mu += m0;
        ad += a0;
    }

    static int bitlen(uint64_t e) { return e ? 64 - __builtin_clzll(e) : 0; }
    static int ceil_lg(uint64_t e) { return e <= 1 ? 0 : bitlen(e - 1); }
    static uint64_t revbin(uint64_t x, int k) {
        uint64_t r = 0;
        for (int i = 0; i < k; ++i) r |= ((x >> i) & 1) << (k - 1 - i);
        return r;
    }
    // ring_pow_k (_kernels.pyx:93-106): bitlen(e)-1 squarings, popcount(e)-1 products
    static int64_t pow_cost(uint64_t e) { return e ? (bitlen(e) - 1) + (__builtin_popcountll(e) - 1) : 0; }

    // g_omega (_kernels.pyx:167-178): K - bitlen(s) squarings of top, then a power
    int64_t g_omega_cost(uint64_t s) const {
        if (!s) return 0;
        const int k = bitlen(s);
        return (K_ - k) + pow_cost(revbin(s, k));
    }

   private:
    struct Memo {
        int64_t mu, ad;
        TallyState out;
    };

    int64_t ensure_base(TallyState& s) {
        if (s.has_base) return 0;
        s.has_base = true;
        return K_ - kstar_;
    }
    // level_root_k (_kernels.pyx:122-135)
    int64_t level_root(int j, bool inverse, TallyState& s) {
        int64_t c = 0;
        if (inverse) {
            if (!s.has_inv) {
                c += ensure_base(s);
                c += pow_cost(p_ - 2);
                s.has_inv = true;
            }
        } else {
            c += ensure_base(s);
        }
        return c + (kstar_ - j);
    }
    // bf_forward / bf_inverse (_kernels.pyx:181-272)
    void butterflies(int64_t m, bool inverse, TallyState& s, int64_t& mu, int64_t& ad) {
        const int64_t bound = m >> 1;
        if (!bound) return;
        int64_t c = 0;
        int k = 1;
        if (bound >= 2) {
            k = 1 + ceil_lg((uint64_t)bound);
            c += level_root(k, inverse, s);
        }
        c += bound - 1;             // theta products (every pair but j = 0)
        c += revinc_steps(bound, k);  // twiddle advances along the bit-reversed counter
        if (inverse) c += 2 * bound;  // the two halvings by inv2
        mu += c;
        ad += 2 * bound;
    }
    // steps of c_revinc over k-1 bits until the last j < bound was emitted:
    // the largest t whose (k-1)-bit reversal is below bound
    static int64_t revinc_steps(int64_t bound, int k) {
        const int b = k - 1;
        if (b <= 0) return 0;
        uint64_t t = 0;
        for (int i = b - 1; i >= 0; --i) {
            const uint64_t cand = t | (1ull << i);
            if (revbin(cand, b) < (uint64_t)bound) t = cand;
        }
        return (int64_t)t;
    }
    // odd_tail + tail_roots_k (_kernels.pyx:138-164, 275-298)
    void odd_tail(int64_t m, TallyState& s, int64_t& mu, int64_t& ad) {
        const int64_t half = (m - 1) >> 1;
        int pos = -1;
        for (int i = 0; i < 4; ++i)
            if (s.lru[i] == half) pos = i;
        int64_t c = 0;
        if (pos < 0) {
            const int k = bitlen((uint64_t)half);
            c += level_root(k + 1, false, s);
            c += pow_cost(revbin((uint64_t)half, k));
            if (half >= 2) c += 1;
            pos = 3;  // evict the least recently used
        }
        for (int i = pos; i > 0; --i) s.lru[i] = s.lru[i - 1];
        s.lru[0] = half;
        mu += c + half;
        ad += half;
    }

    uint64_t p_;
    int K_, kstar_;
    std::map<std::tuple<int64_t, bool, decltype(TallyState().key())>, Memo> memo_;
};

// (mults, adds) of _kernels.tft / itft on a length-n buffer
inline void tally_transform(int64_t n, uint64_t p, int K, bool inverse, int64_t* mults, int64_t* adds) {
    static std::mutex mu;
    static std::map<std::tuple<int64_t, uint64_t, int, bool>, std::pair<int64_t, int64_t>> cache;
    const auto key = std::make_tuple(n, p, K, inverse);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            if (mults) *mults = it->second.first;
            if (adds) *adds = it->second.second;
            return;
        }
    }
    TallyWalk w(p, K, TallyWalk::ceil_lg((uint64_t)n));
    TallyState s;
    int64_t m = 0, a = 0;
    w.walk(n, inverse, s, m, a);
    {
        std::lock_guard<std::mutex> g(mu);
        cache[key] = {m, a};
    }
    if (mults) *mults = m;
    if (adds) *adds = a;
}

// (mults, adds) of _kernels.multiply (_kernels.pyx:433-480): the block
// schedule's folds, block transforms and pointwise products, the two Horner
// evaluations of the last slot, and the final inverse over r words
inline void tally_multiply(int64_t la, int64_t lb, uint64_t p, int K, int64_t* mults, int64_t* adds) {
    const int64_t r = la + lb - 1;
    TallyWalk g(p, K, K);
    int64_t m = 0, a = 0;
    for (int64_t q = 0; q < r - 1;) {
        const int ell = TallyWalk::bitlen((uint64_t)(r - q)) - 2;
        const int64_t L = (int64_t)1 << ell;
        for (int64_t ls : {la, lb}) {
            if (q) m += g.g_omega_cost((uint64_t)q) + 2 * (ls - 1);  // fold_twist_k
            a += ls;
            int64_t tm, ta;
            TallyWalk t(p, K, ell);
            TallyState s;
            tm = ta = 0;
            t.walk(L, false, s, tm, ta);
            m += tm;
            a += ta;
        }
        m += L;  // pointwise products
        q += L;
    }
    m += g.g_omega_cost((uint64_t)(r - 1));
    m += (la - 1) + (lb - 1) + 1;  // horner_k twice, then their product
    a += (la - 1) + (lb - 1);
    int64_t im = 0, ia = 0;
    tally_transform(r, p, K, true, &im, &ia);
    m += im;
    a += ia;
    if (mults) *mults = m;
    if (adds) *adds = a;
}

}  // namespace tftb
