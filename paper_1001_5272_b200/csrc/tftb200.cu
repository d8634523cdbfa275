// Host side of libtftb200.so: ring tables, planning, launches and the C ABI
// declared in include/tftb200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tftb200.h"
#include "kernels.cuh"

namespace {

typedef unsigned __int128 u128;

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

int fail(const std::string& msg) {
    g_err = msg;
    return -1;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return fail(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}
int ceil_lg(int64_t n) {
    int k = 0;
    while (((int64_t)1 << k) < n) k++;
    return k;
}

// -------------------------------------------------------------- ring tables
struct RingHost {
    uint64_t p, top;
    int K;
    int wbytes;      // 4 or 8
    int kind;        // 0 F30, 1 F32, 2 F62
    int zb, zh;
    void* dmem = nullptr;  // one allocation for every table
    RingDev<uint32_t> r32{};
    RingDev<uint64_t> r64{};
    ~RingHost() {
        if (dmem) cudaFree(dmem);
    }
};

template <typename W>
struct TableBuilder {
    uint64_t p;
    int bits;
    W pinv;
    uint64_t R1;  // R mod p
    uint64_t to_m(uint64_t w) const { return (uint64_t)(((u128)w << bits) % p); }
    Tw<W> tw(uint64_t w) const {
        W wm = (W)to_m(w);
        return Tw<W>{wm, (W)(wm * pinv)};
    }
};

template <typename W>
W inv_word(W p) {  // p^-1 mod 2^bits (Newton)
    W x = p;
    for (int i = 0; i < 7; i++) x *= (W)2 - p * x;
    return x;
}

template <typename W>
int build_tables(RingHost* rh, RingDev<W>* out) {
    const uint64_t p = rh->p;
    TableBuilder<W> tb{p, (int)(8 * sizeof(W)), inv_word<W>((W)p), 0};
    // omega_[k] = top^(2^(K-k))
    std::vector<uint64_t> lvl(rh->K + 1), ilvl(rh->K + 1);
    uint64_t itop = powmod(rh->top, p - 2, p);
    {
        uint64_t w = rh->top, iw = itop;
        for (int k = rh->K; k >= 0; --k) {
            lvl[k] = w;
            ilvl[k] = iw;
            w = mulmod(w, w, p);
            iw = mulmod(iw, iw, p);
        }
    }
    const int zb = rh->zb, zh = rh->zh;
    const size_t nz = (size_t)1 << zb, nh = (size_t)1 << zh;
    // Z[2^(k-1) + i] = omega_[k+1] * Z[i]  (product rule)
    auto build = [&](const std::vector<uint64_t>& L, std::vector<uint64_t>& Z, int shift) {
        // Z[i] = omega_{2 i 2^shift}; Z[2^(k-1)+i] = omega_[k+1+shift] Z[i]
        Z[0] = 1;
        for (size_t h = 1, k = 1; h < Z.size(); h <<= 1, ++k)
            for (size_t i = 0; i < h; i++) Z[h + i] = mulmod(L[k + 1 + shift], Z[i], p);
    };
    std::vector<uint64_t> zf(nz), zi(nz), zfh(nh), zih(nh);
    build(lvl, zf, 0);
    build(ilvl, zi, 0);
    build(lvl, zfh, zb);
    build(ilvl, zih, zb);
    std::vector<Tw<W>> host;
    host.reserve(2 * nz + 2 * nh + 64);
    for (auto v : zf) host.push_back(tb.tw(v));
    for (auto v : zi) host.push_back(tb.tw(v));
    for (auto v : zfh) host.push_back(tb.tw(v));
    for (auto v : zih) host.push_back(tb.tw(v));
    uint64_t inv2 = (p + 1) >> 1, ip = 1;
    for (int k = 0; k < 64; k++) {
        host.push_back(tb.tw(ip));
        ip = mulmod(ip, inv2, p);
    }
    CK(cudaMalloc(&rh->dmem, host.size() * sizeof(Tw<W>)));
    CK(cudaMemcpy(rh->dmem, host.data(), host.size() * sizeof(Tw<W>), cudaMemcpyHostToDevice));
    Tw<W>* d = (Tw<W>*)rh->dmem;
    out->Zf = d;
    out->Zi = d + nz;
    out->Zfh = d + 2 * nz;
    out->Zih = d + 2 * nz + nh;
    out->ipow2 = d + 2 * nz + 2 * nh;
    uint64_t R1 = tb.to_m(1);
    out->r2 = tb.tw(R1);  // Montgomery form of R is R^2 mod p
    out->inv2 = tb.tw(inv2);
    out->oneM = (W)R1;
    out->zb = zb;
    out->zh = zh;
    return 0;
}

std::mutex g_ring_mu;
std::map<std::tuple<uint64_t, uint64_t, int, int>, std::unique_ptr<RingHost>> g_rings;

int get_ring(uint64_t p, uint64_t top, int K, RingHost** out) {
    if (p < 3 || !(p & 1) || p >= (1ull << 62)) return fail("modulus must be an odd prime below 2^62");
    if (K < 0 || K > 62 || top == 0 || top >= p) return fail("bad root / K");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_ring_mu);
    auto key = std::make_tuple(p, top, K, dev);
    auto it = g_rings.find(key);
    if (it != g_rings.end()) {
        *out = it->second.get();
        return 0;
    }
    auto rh = std::make_unique<RingHost>();
    rh->p = p;
    rh->top = top;
    rh->K = K;
    rh->wbytes = p < (1ull << 32) ? 4 : 8;
    rh->kind = p < (1ull << 30) ? 0 : (p < (1ull << 32) ? 1 : 2);
    int km1 = K > 0 ? K - 1 : 0;
    rh->zb = std::min(km1, 14);
    rh->zh = std::min(km1 - rh->zb, 16);
    int rc = rh->wbytes == 4 ? build_tables<uint32_t>(rh.get(), &rh->r32)
                             : build_tables<uint64_t>(rh.get(), &rh->r64);
    if (rc) return rc;
    *out = rh.get();
    g_rings[key] = std::move(rh);
    return 0;
}

template <class F>
F make_field(uint64_t p) {
    F f;
    f.p = (typename F::W)p;
    f.p2 = (typename F::W)(2 * p);
    f.pinv = inv_word<typename F::W>((typename F::W)p);
    return f;
}

template <class F>
const RingDev<typename F::W>& ring_dev(const RingHost* rh);
template <>
const RingDev<uint32_t>& ring_dev<F30>(const RingHost* rh) { return rh->r32; }
template <>
const RingDev<uint32_t>& ring_dev<F32>(const RingHost* rh) { return rh->r32; }
template <>
const RingDev<uint64_t>& ring_dev<F62>(const RingHost* rh) { return rh->r64; }

// -------------------------------------------------------------- planning
constexpr int kNT = 256;

template <class F>
struct Limits {
    // log2 words of the single-vector tile and of the column / chunk tiles
    static constexpr int small_t = sizeof(typename F::W) == 4 ? 13 : 12;
    static constexpr int col_t = sizeof(typename F::W) == 4 ? 13 : 12;
    static constexpr int chunk_max = sizeof(typename F::W) == 4 ? 15 : 14;
};

struct Plan {
    bool small;
    int l, l0, l1, wlog;
};

template <class F>
int make_plan(int l, Plan* pl) {
    pl->l = l;
    if (l <= Limits<F>::small_t) {
        pl->small = true;
        pl->l0 = pl->l1 = pl->wlog = 0;
        return 0;
    }
    pl->small = false;
    int l0 = std::min(l / 2, Limits<F>::col_t - 4);
    int l1 = l - l0;
    if (l1 > Limits<F>::chunk_max) {
        l1 = Limits<F>::chunk_max;
        l0 = l - l1;
    }
    int wlog = std::max(1, std::min(4, Limits<F>::col_t - l0));
    if (l0 + wlog > Limits<F>::col_t + 1) return fail("transform length too large for the two-pass plan");
    pl->l0 = l0;
    pl->l1 = l1;
    pl->wlog = wlog;
    return 0;
}

template <class K_>
int set_smem(K_ kern, size_t bytes) {
    if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return 0;
}

struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    int get(size_t b, cudaStream_t st) {
        s = st;
        if (b == 0) return 0;
        CK(cudaMallocAsync(&p, b, st));
        bytes = b;
        return 0;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

// One group of vectors that share a plan.
template <class F>
int run_group(const RingHost* rh, typename F::W* x, const typename F::W* in, const typename F::W* pre,
              int64_t count, VecDesc<typename F::W> xd, VecDesc<typename F::W> ind, int64_t maxn,
              bool inverse, cudaStream_t st) {
    using W = typename F::W;
    Plan pl;
    if (make_plan<F>(ceil_lg(maxn), &pl)) return -1;
    LaunchArgs<F> a{};
    a.f = make_field<F>(rh->p);
    a.R = ring_dev<F>(rh);
    a.x = x;
    a.xd = xd;
    a.in = in ? in : x;
    a.ind = in ? ind : xd;
    a.pre = pre;
    a.l0 = pl.l0;
    a.l1 = pl.l1;
    a.wlog = pl.wlog;
    if (pl.small) {
        size_t smem = padded_words(1u << pl.l) * sizeof(W);
        int nt = std::max(32, std::min(kNT, (1 << pl.l) / 16));
        if (inverse) {
            if (set_smem(k_small_inv<F>, smem)) return -1;
        } else {
            if (set_smem(k_small_fwd<F>, smem)) return -1;
        }
        for (int64_t v0 = 0; v0 < count; v0 += (1ll << 30)) {
            a.vbase = v0;
            unsigned nb = (unsigned)std::min<int64_t>(count - v0, 1ll << 30);
            if (inverse) k_small_inv<F><<<nb, nt, smem, st>>>(a);
            else k_small_fwd<F><<<nb, nt, smem, st>>>(a);
            g_launches++;
            CK(cudaGetLastError());
        }
        return 0;
    }
    const uint32_t C = 1u << pl.l1;
    const int64_t maxchunks = (maxn + C - 1) / C;
    const int64_t vchunk = 65535;
    Scratch stash;
    if (stash.get((size_t)std::min(count, vchunk) * C * sizeof(W), st)) return -1;
    a.stash = (W*)stash.p;
    const size_t sm_col = padded_words(1u << (pl.l0 + pl.wlog)) * sizeof(W) + (kNT + 64) * sizeof(W);
    const size_t sm_chunk = (padded_words(C) + C + 64) * sizeof(W);
    const size_t sm_last = (padded_words(C) + 2 * C + 64) * sizeof(W);
    if (set_smem(k_col_fwd<F>, sm_col) || set_smem(k_col_inv<F>, sm_col) || set_smem(k_chunk_fwd<F>, sm_chunk) ||
        set_smem(k_chunk_inv<F>, sm_chunk) || set_smem(k_last_inv<F>, sm_last))
        return -1;
    for (int64_t v0 = 0; v0 < count; v0 += vchunk) {
        a.vbase = v0;
        unsigned nv = (unsigned)std::min(count - v0, vchunk);
        dim3 gcol(C >> pl.wlog, nv), gchunk((unsigned)maxchunks, nv), glast(1, nv);
        if (!inverse) {
            k_col_fwd<F><<<gcol, kNT, sm_col, st>>>(a);
            k_chunk_fwd<F><<<gchunk, kNT, sm_chunk, st>>>(a);
            g_launches += 2;
        } else {
            k_chunk_inv<F><<<gchunk, kNT, sm_chunk, st>>>(a);
            k_col_inv<F><<<gcol, kNT, sm_col, st>>>(a, 0);
            k_last_inv<F><<<glast, kNT, sm_last, st>>>(a);
            k_col_inv<F><<<gcol, kNT, sm_col, st>>>(a, 1);
            g_launches += 4;
        }
        CK(cudaGetLastError());
    }
    return 0;
}

// Partition a batch by plan (ceil_lg of the length class) and run each group.
template <class F>
int run_batch(const RingHost* rh, void* data, const void* in, int64_t count, int64_t n, int64_t stride,
              const int64_t* h_off, const int64_t* h_len, const void* in_data, int64_t in_n,
              int64_t in_stride, const void* pre, bool inverse, cudaStream_t st) {
    using W = typename F::W;
    if (count <= 0) return 0;
    if (!h_off && !h_len) {
        VecDesc<W> xd{nullptr, nullptr, stride, n};
        VecDesc<W> ind{nullptr, nullptr, in_stride, in_n};
        return run_group<F>(rh, (W*)data, (const W*)in_data, (const W*)pre, count, xd, ind, n, inverse, st);
    }
    (void)in;
    // group vectors by the plan they need
    std::map<int, std::vector<int64_t>> groups;
    for (int64_t v = 0; v < count; v++) {
        int64_t nv = h_len ? h_len[v] : n;
        if (nv <= 0) return fail("vector length must be positive");
        int l = ceil_lg(nv);
        Plan pl;
        if (make_plan<F>(l, &pl)) return -1;
        int key = pl.small ? -1 : l;  // one small group (t varies per vector inside the kernel)
        groups[key].push_back(v);
    }
    for (auto& kv : groups) {
        auto& idx = kv.second;
        std::vector<int64_t> off(idx.size()), len(idx.size());
        int64_t maxn = 0;
        for (size_t i = 0; i < idx.size(); i++) {
            off[i] = h_off ? h_off[idx[i]] : idx[i] * stride;
            len[i] = h_len ? h_len[idx[i]] : n;
            maxn = std::max(maxn, len[i]);
        }
        Scratch d;
        if (d.get(2 * idx.size() * sizeof(int64_t), st)) return -1;
        int64_t* doff = (int64_t*)d.p;
        CK(cudaMemcpyAsync(doff, off.data(), idx.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(doff + idx.size(), len.data(), idx.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        VecDesc<W> xd{doff, doff + idx.size(), 0, 0};
        if (run_group<F>(rh, (W*)data, nullptr, (const W*)pre, (int64_t)idx.size(), xd, xd, maxn, inverse, st))
            return -1;
        // host vectors off/len must outlive the async copies
        CK(cudaStreamSynchronize(st));
    }
    return 0;
}

template <class F>
int dispatch_tft(const RingHost* rh, void* data, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                 const int64_t* h_len, int inverse, cudaStream_t st) {
    return run_batch<F>(rh, data, nullptr, count, n, stride, h_off, h_len, nullptr, 0, 0, nullptr, inverse != 0, st);
}

template <class F>
int dispatch_mul(const RingHost* rh, const void* a, int64_t la, int64_t sa, const void* b, int64_t lb, int64_t sb,
                 void* x, int64_t sx, int64_t count, void* scratch, cudaStream_t st) {
    using W = typename F::W;
    const int64_t r = la + lb - 1;
    if (sx != r) return fail("multiply_dev: output stride must equal la+lb-1");
    Scratch own;
    if (!scratch) {
        if (own.get((size_t)count * r * sizeof(W), st)) return -1;
        scratch = own.p;
    }
    // X_v <- TFT_r(a_v || 0), Y_v <- TFT_r(b_v || 0), X_v <- ITFT_r(X_v * Y_v)
    if (run_batch<F>(rh, x, nullptr, count, r, sx, nullptr, nullptr, a, la, sa, nullptr, false, st)) return -1;
    if (run_batch<F>(rh, scratch, nullptr, count, r, r, nullptr, nullptr, b, lb, sb, nullptr, false, st)) return -1;
    if (run_batch<F>(rh, x, nullptr, count, r, sx, nullptr, nullptr, nullptr, 0, 0, scratch, true, st)) return -1;
    return 0;
}

// model op counts of the device algorithm
void model_counts(int64_t n, bool inverse, int64_t* mults, int64_t* adds) {
    int l = ceil_lg(n);
    int64_t N = (int64_t)1 << l;
    int64_t bf = (N / 2) * l;
    if (mults) *mults = inverse ? bf + n : bf;
    if (adds) *adds = 2 * bf;
}

int host_tft_common(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, bool inverse, int64_t* mults,
                    int64_t* adds) {
    if (n <= 0) return fail("cannot transform an empty buffer");
    if (K < 62 && n > (1ll << K)) return fail("length exceeds 2^K");
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    cudaStream_t st = nullptr;
    const size_t wb = rh->wbytes;
    Scratch buf;
    if (buf.get((size_t)n * 8 + (wb == 4 ? (size_t)n * 4 : 0), st)) return -1;
    uint64_t* d64 = (uint64_t*)buf.p;
    CK(cudaMemcpyAsync(d64, x, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    int rc = 0;
    if (wb == 4) {
        uint32_t* dw = (uint32_t*)(d64 + n);
        int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        k_u64_to_w<uint32_t><<<nb, 256, 0, st>>>(d64, dw, n);
        rc = rh->kind == 0 ? dispatch_tft<F30>(rh, dw, 1, n, n, nullptr, nullptr, inverse, st)
                           : dispatch_tft<F32>(rh, dw, 1, n, n, nullptr, nullptr, inverse, st);
        if (rc) return rc;
        k_w_to_u64<uint32_t><<<nb, 256, 0, st>>>(dw, d64, n);
        g_launches += 2;
    } else {
        rc = dispatch_tft<F62>(rh, d64, 1, n, n, nullptr, nullptr, inverse, st);
        if (rc) return rc;
    }
    CK(cudaMemcpyAsync(x, d64, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    model_counts(n, inverse, mults, adds);
    return 0;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int tftb_tft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, int64_t* mults, int64_t* adds) {
    return host_tft_common(x, n, p, top, K, false, mults, adds);
}

int tftb_itft_u64(uint64_t* x, int64_t n, uint64_t p, uint64_t top, int K, uint64_t inv2, int64_t* mults,
                  int64_t* adds) {
    if (inv2 != (p + 1) / 2) return fail("inv2 must be (p+1)/2");
    return host_tft_common(x, n, p, top, K, true, mults, adds);
}

int tftb_multiply_u64(const uint64_t* a, int64_t la, const uint64_t* b, int64_t lb, uint64_t* x, uint64_t p,
                      uint64_t top, int K, uint64_t inv2, int64_t* mults, int64_t* adds) {
    if (la <= 0 || lb <= 0) return fail("cannot multiply an empty polynomial");
    if (inv2 != (p + 1) / 2) return fail("inv2 must be (p+1)/2");
    const int64_t r = la + lb - 1;
    if (K < 62 && r > (1ll << K)) return fail("product length exceeds 2^K");
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    cudaStream_t st = nullptr;
    const size_t wb = rh->wbytes;
    // device: a, b, x as u64 staging + (u32 field) word copies + the Y scratch
    Scratch buf;
    size_t words64 = (size_t)(la + lb + r);
    if (buf.get(words64 * 8 + (size_t)(la + lb + 2 * r) * wb, st)) return -1;
    uint64_t* da64 = (uint64_t*)buf.p;
    uint64_t* db64 = da64 + la;
    uint64_t* dx64 = db64 + lb;
    unsigned char* wbase = (unsigned char*)(dx64 + r);
    CK(cudaMemcpyAsync(da64, a, (size_t)la * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(db64, b, (size_t)lb * 8, cudaMemcpyHostToDevice, st));
    int rc;
    if (wb == 4) {
        uint32_t* da = (uint32_t*)wbase;
        uint32_t* db = da + la;
        uint32_t* dx = db + lb;
        uint32_t* dy = dx + r;
        k_u64_to_w<uint32_t><<<592, 256, 0, st>>>(da64, da, la + lb);  // a and b are adjacent
        rc = rh->kind == 0 ? dispatch_mul<F30>(rh, da, la, la, db, lb, lb, dx, r, 1, dy, st)
                           : dispatch_mul<F32>(rh, da, la, la, db, lb, lb, dx, r, 1, dy, st);
        if (rc) return rc;
        k_w_to_u64<uint32_t><<<592, 256, 0, st>>>(dx, dx64, r);
        g_launches += 2;
    } else {
        uint64_t* dy = (uint64_t*)wbase;
        rc = dispatch_mul<F62>(rh, da64, la, la, db64, lb, lb, dx64, r, 1, dy, st);
        if (rc) return rc;
    }
    CK(cudaMemcpyAsync(x, dx64, (size_t)r * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t m1, a1, m2, a2;
    model_counts(r, false, &m1, &a1);
    model_counts(r, true, &m2, &a2);
    if (mults) *mults = 2 * m1 + m2 + r;
    if (adds) *adds = 2 * a1 + a2;
    return 0;
}

struct tftb_ring {
    RingHost* h;
};

int tftb_ring_get(uint64_t p, uint64_t top, int K, tftb_ring** out) {
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    static std::mutex mu;
    static std::map<RingHost*, std::unique_ptr<tftb_ring>> handles;
    std::lock_guard<std::mutex> lk(mu);
    auto& h = handles[rh];
    if (!h) h.reset(new tftb_ring{rh});
    *out = h.get();
    return 0;
}

int tftb_ring_word_bytes(const tftb_ring* ring) { return ring ? ring->h->wbytes : -1; }

int tftb_tft_dev(const tftb_ring* ring, void* data, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                 const int64_t* h_len, int inverse, void* stream) {
    if (!ring) return fail("null ring");
    const RingHost* rh = ring->h;
    cudaStream_t st = (cudaStream_t)stream;
    switch (rh->kind) {
        case 0: return dispatch_tft<F30>(rh, data, count, n, stride, h_off, h_len, inverse, st);
        case 1: return dispatch_tft<F32>(rh, data, count, n, stride, h_off, h_len, inverse, st);
        default: return dispatch_tft<F62>(rh, data, count, n, stride, h_off, h_len, inverse, st);
    }
}

int tftb_multiply_dev(const tftb_ring* ring, const void* a, int64_t la, int64_t sa, const void* b, int64_t lb,
                      int64_t sb, void* x, int64_t sx, int64_t count, void* scratch, void* stream) {
    if (!ring) return fail("null ring");
    if (la <= 0 || lb <= 0) return fail("cannot multiply an empty polynomial");
    const RingHost* rh = ring->h;
    cudaStream_t st = (cudaStream_t)stream;
    switch (rh->kind) {
        case 0: return dispatch_mul<F30>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
        case 1: return dispatch_mul<F32>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
        default: return dispatch_mul<F62>(rh, a, la, sa, b, lb, sb, x, sx, count, scratch, st);
    }
}

int tftb_words_from_u64(const tftb_ring* ring, const uint64_t* d_src, void* d_dst, int64_t n, void* stream) {
    if (!ring) return fail("null ring");
    cudaStream_t st = (cudaStream_t)stream;
    if (ring->h->wbytes == 8) {
        CK(cudaMemcpyAsync(d_dst, d_src, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (nb < 1) nb = 1;
    k_u64_to_w<uint32_t><<<nb, 256, 0, st>>>(d_src, (uint32_t*)d_dst, n);
    g_launches++;
    CK(cudaGetLastError());
    return 0;
}

int tftb_words_to_u64(const tftb_ring* ring, const void* d_src, uint64_t* d_dst, int64_t n, void* stream) {
    if (!ring) return fail("null ring");
    cudaStream_t st = (cudaStream_t)stream;
    if (ring->h->wbytes == 8) {
        CK(cudaMemcpyAsync(d_dst, d_src, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    int nb = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (nb < 1) nb = 1;
    k_w_to_u64<uint32_t><<<nb, 256, 0, st>>>((const uint32_t*)d_src, d_dst, n);
    g_launches++;
    CK(cudaGetLastError());
    return 0;
}

const char* tftb_last_error(void) { return g_err.c_str(); }
const char* tftb_version(void) { return "tftb200 0.1.0 (sm_100a)"; }
int64_t tftb_launch_count(int reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

}  // extern "C"
