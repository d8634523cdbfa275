// Batch planning and launches (instantiated once per field type).
#pragma once
#include "p2r.cuh"
#include "small.cuh"
#include "host.h"

namespace tftb {

constexpr int kGroupStreams = 4;  // side streams per forking plan

// whole-vector tiles of one size class T = ceil_lg(n)
template <class F, int T>
int launch_tiles(LaunchArgs<F> a, int64_t count, bool inverse, cudaStream_t st) {
    using SH = TileShape<T>;
    const size_t smem = SH::smem(sizeof(typename F::W));
    auto k = inverse ? k_tile_inv<F, T> : k_tile_fwd<F, T>;
    if (set_smem(k, smem)) return -1;
    const int64_t per = (int64_t)SH::VPB << 30;  // vectors per launch (grid.x < 2^31)
    for (int64_t v0 = 0; v0 < count; v0 += per) {
        a.vbase = v0;
        const int64_t nv = std::min(count - v0, per);
        const unsigned nb = (unsigned)((nv + SH::VPB - 1) / SH::VPB);
        k<<<nb, 256, smem, st>>>(a, v0 + nv);
        g_launches++;
        CK(cudaGetLastError());
    }
    return 0;
}

template <class F>
int run_tiles(LaunchArgs<F> a, int T, int64_t count, bool inverse, cudaStream_t st) {
    static_assert(Limits<F>::CL <= 14, "tile instantiations stop at 2^14");
    switch (T) {
#define TFTB_TILE_CASE(t) \
    case t:              \
        if constexpr (t <= Limits<F>::CL) return launch_tiles<F, t>(a, count, inverse, st); \
        break;
        TFTB_TILE_CASE(0) TFTB_TILE_CASE(1) TFTB_TILE_CASE(2) TFTB_TILE_CASE(3) TFTB_TILE_CASE(4)
        TFTB_TILE_CASE(5) TFTB_TILE_CASE(6) TFTB_TILE_CASE(7) TFTB_TILE_CASE(8) TFTB_TILE_CASE(9)
        TFTB_TILE_CASE(10) TFTB_TILE_CASE(11) TFTB_TILE_CASE(12) TFTB_TILE_CASE(13) TFTB_TILE_CASE(14)
#undef TFTB_TILE_CASE
    }
    return fail("tile size class out of range");
}

static_assert(kP2RMax == kP2RMaxDev, "p2r bound mismatch");

// omega_s (modring.py:223-234) on the host
inline uint64_t omega_host(const RingHost* rh, uint64_t s) {
    if (!s) return 1;
    const int k = 64 - __builtin_clzll(s);
    uint64_t rev = 0;
    for (int i = 0; i < k; ++i) rev |= ((s >> i) & 1) << (k - 1 - i);
    return powmod(powmod(rh->top, 1ull << (rh->K - k), rh->p), rev, rh->p);
}

// a field twiddle for w (canonical residue): Shoup pair for F30, Montgomery
// pair otherwise (the device forms, field.cuh)
template <class F>
Tw<typename F::W> host_tw(uint64_t w, uint64_t p) {
    using W = typename F::W;
    constexpr int bits = 8 * sizeof(W);
    if constexpr (std::is_same<F, F30>::value) {
        return Tw<W>{(W)w, (W)(((u128)w << 32) / p)};
    } else {
        const W wm = (W)(((u128)w << bits) % p);
        return Tw<W>{wm, (W)(wm * inv_word<W>((W)p))};
    }
}

// the powers k_p2r reads, per s < r: rho_s, rho_s^(1024 nb), rho_s^(4t)
// (t < 256), rho_s^(1024 b) (b < nb) -- built once per (ring, k, r, nb)
template <class F>
const Tw<typename F::W>* p2r_tables(const RingHost* rh, int k, int r, int nb) {
    using W = typename F::W;
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, int, int>, void*> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    void*& d = cache[{(const void*)rh, k, r, nb, dev}];
    if (!d) {
        const uint64_t p = rh->p;
        std::vector<Tw<W>> h;
        for (int s = 0; s < r; ++s) {
            const uint64_t rho = omega_host(rh, (1ull << k) + s);
            h.push_back(host_tw<F>(rho, p));
            h.push_back(host_tw<F>(powmod(rho, 1024ull * nb, p), p));
            const uint64_t r4 = powmod(rho, 4, p), r1024 = powmod(rho, 1024, p);
            uint64_t w = 1;
            for (int t = 0; t < 256; ++t, w = mulmod(w, r4, p)) h.push_back(host_tw<F>(w, p));
            w = 1;
            for (int b = 0; b < nb; ++b, w = mulmod(w, r1024, p)) h.push_back(host_tw<F>(w, p));
        }
        if (cudaMalloc(&d, h.size() * sizeof(Tw<W>)) != cudaSuccess ||
            cudaMemcpy(d, h.data(), h.size() * sizeof(Tw<W>), cudaMemcpyHostToDevice) != cudaSuccess) {
            d = nullptr;
            fail("p2r: table upload failed");
            return nullptr;
        }
    }
    return (const Tw<W>*)d;
}

// blocks per vector of k_p2r: ~8 per SM over the whole batch (full
// occupancy for a streaming pass; per-thread setup is a few table loads) and
// at least 16 1024-word rows per block, so a block's fixed cost (setup,
// reduction tree, ticket) stays small against its streaming (single 2^22 + 1
// vector: -9%)
inline int p2r_blocks(int64_t count, int64_t H, int r) {
    const int64_t rows = (H + r + 1023) / 1024;
    return (int)std::max<int64_t>(1, std::min<int64_t>({8 * 148, (8 * 148 + count - 1) / count, rows / 16}));
}

// n = 2^k + r: fold + r dot products + the 2^k transform (p2r.cuh)
template <class F>
int run_p2r(const RingHost* rh, LaunchArgs<F> a, int k, int r, int64_t count, VecDesc<typename F::W> xd,
            bool inverse, cudaStream_t st, typename F::W* stash_buf);

// One group of vectors that share a plan.
template <class F>
int run_group(const RingHost* rh, typename F::W* x, const typename F::W* in, const typename F::W* pre,
              int64_t count, VecDesc<typename F::W> xd, VecDesc<typename F::W> ind, int64_t maxn,
              bool inverse, cudaStream_t st, typename F::W* stash_buf = nullptr, int64_t uni_n = 0) {
    using W = typename F::W;
    Plan pl;
    if (make_plan<F>(maxn, &pl)) return -1;
    LaunchArgs<F> a{};
    a.f = make_field<F>(rh->p);
    a.R = ring_dev<F>(rh);
    a.x = x;
    a.xd = xd;
    a.in = in ? in : x;
    a.ind = in ? ind : xd;
    a.pre = pre;
    a.timing = g_tail_timing;  // debug: stamps of the large inverse's tail kernels (null in production)
    static const int dense_cols = getenv("TFTB_DENSE_COLS") != nullptr;  // A/B knob
    a.dense_cols = dense_cols;
    a.l0 = pl.l0;
    a.l1 = pl.l1;
    a.wlog = pl.wlog;
    if (pl.kind == kCluster) {
        constexpr int CL = Limits<F>::CL;
        const size_t smem = padded_words(1u << CL) * sizeof(W);
        const int gam = pl.l - CL;
        // (the chunk count is a template argument: rows past it are known zeros)
        void (*kg)(LaunchArgs<F>) = gam == 1 ? k_clg_fwd<F, CL, 1>
                                   : gam == 2 ? (pl.G == 3 ? k_clg_fwd<F, CL, 2, 3> : k_clg_fwd<F, CL, 2>)
                                              : k_clg_fwd<F, CL, 3>;
        void (*kf)(LaunchArgs<F>) = gam == 1 ? k_clf_cols<F, CL, 1>
                                   : gam == 2 ? k_clf_cols<F, CL, 2> : k_clf_cols<F, CL, 3>;
        // forward: the cone kernel needs a G-CTA cluster (in-place order);
        // from 5 chunks on, co-scheduling such clusters costs more than the
        // split forward's second pass (measured)
        const bool fsplit = pl.G >= 5;
        if (inverse ? (set_smem(k_cli_chunks<F, CL>, smem) || set_smem(k_cli_cols<F, CL>, smem))
                    : fsplit ? (set_smem(kf, smem) || set_smem(k_clf_chunks<F, CL>, smem)) : set_smem(kg, smem))
            return -1;
        // fused split inverse: per-vector chunk tickets (zeroed once here,
        // self-resetting in the kernel); TFTB_SPLIT_INV=1 keeps the two launches
        static const bool two_launch = getenv("TFTB_SPLIT_INV") != nullptr;
        Scratch tickets;
        if (inverse && !two_launch) {
            const size_t tb = (size_t)std::min<int64_t>(count, 65535) * sizeof(unsigned);
            if (tickets.get(tb, st)) return -1;
            CK(cudaMemsetAsync(tickets.p, 0, tb, st));
            a.done = (unsigned*)tickets.p;
        }
        for (int64_t v0 = 0; v0 < count; v0 += 65535) {
            a.vbase = v0;
            unsigned nv = (unsigned)std::min<int64_t>(count - v0, 65535);
            if (inverse && !two_launch) {
                k_cli_chunks<F, CL><<<dim3(pl.G, nv, 1), kNT, smem, st>>>(a);
                CK(cudaGetLastError());
                g_launches += 1;
            } else if (inverse) {
                // split inverse: per-chunk launch, then one CTA per vector
                k_cli_chunks<F, CL><<<dim3(pl.G, nv, 1), kNT, smem, st>>>(a);
                CK(cudaGetLastError());
                k_cli_cols<F, CL><<<nv, kNT, smem, st>>>(a);
                CK(cudaGetLastError());
                g_launches += 2;
            } else if (fsplit) {
                kf<<<nv, kNT, smem, st>>>(a);
                CK(cudaGetLastError());
                k_clf_chunks<F, CL><<<dim3(pl.G, nv, 1), kNT, smem, st>>>(a);
                CK(cudaGetLastError());
                g_launches += 2;
            } else {
                // forward: rows re-read through L2; the G CTAs of a vector form
                // a cluster only for the split barrier ordering in-place stores
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(pl.G, nv, 1);
                lc.blockDim = dim3(kNT, 1, 1);
                lc.dynamicSmemBytes = smem;
                lc.stream = st;
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = pl.G;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                // let the hardware place a cluster's CTAs on any free SMs of
                // the GPC (measured: config-2 forward -5%, 2-chunk vectors -25%)
                at[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
                at[1].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
                lc.numAttrs = 2;
                CK(cudaLaunchKernelEx(&lc, kg, a));
                g_launches++;
            }
        }
        return 0;
    }
    if (pl.kind == kSmall) return run_tiles<F>(a, pl.l, count, inverse, st);
    if (pl.kind == kP2R) {
        if (in && in != x) {  // the fold rewrites the input: transforms in place only
            if (make_plan<F>(maxn, &pl, false)) return -1;
        } else {
            return run_p2r<F>(rh, a, pl.l - 1, pl.G, count, xd, inverse, st, stash_buf);
        }
    }
    const uint32_t C = 1u << pl.l1;
    const int64_t maxchunks = (maxn + C - 1) / C;
    const int64_t vchunk = 65535;
    Scratch stash;
    if (!stash_buf && stash.get((size_t)std::min(count, vchunk) * C * sizeof(W), st, true)) return -1;
    a.stash = stash_buf ? stash_buf : (W*)stash.p;
    // column tile + the inverse's per-column sums (blockDim words of partials,
    // one word per column)
    const size_t sm_col = (padded_words(1u << (pl.l0 + pl.wlog)) + kNT + (1u << pl.wlog) + 8) * sizeof(W);
    const size_t sm_chunk = padded_words(C) * sizeof(W);
    // compile-time column kernels, one instantiation per l0
    // forward of a zero-padded operand (a product's A or B, uniform input
    // length): the column networks' top zt <= 2 layers see zero upper rows
    static const bool no_zt = getenv("TFTB_NO_ZT") != nullptr;  // A/B knob
    int zt = 0;
    if (!inverse && in && in != x && !ind.len && !no_zt) {
        const int64_t rows_in = (ind.n0 + C - 1) / C;
        while (zt < 2 && pl.l0 - zt - 1 >= 0 && rows_in <= (1ll << (pl.l0 - zt - 1))) ++zt;
    }
    void (*colf)(LaunchArgs<F>) = nullptr;
    void (*coli)(LaunchArgs<F>, int) = nullptr;
    void (*col1)(LaunchArgs<F>) = nullptr;  // per-column step 2 (long columns only)
    switch (pl.l0) {
#define TFTB_COL(L)                                   \
    case L:                                           \
        colf = k_colc_fwd<F, L>;                      \
        if constexpr (L >= 6) {                       \
            if (zt == 1) colf = k_colc_fwd<F, L, 1>;  \
            if (zt == 2) colf = k_colc_fwd<F, L, 2>;  \
        }                                             \
        coli = k_colc_inv<F, L>;                      \
        if constexpr (L >= 8) col1 = k_col1_inv<F, L>; \
        break;
        TFTB_COL(4) TFTB_COL(5) TFTB_COL(6) TFTB_COL(7) TFTB_COL(8) TFTB_COL(9)
        TFTB_COL(10) TFTB_COL(11) TFTB_COL(12) TFTB_COL(13) TFTB_COL(14)
#undef TFTB_COL
        default: return fail("no column kernel for this plan");
    }
    // Step 2 of the inverse by column when the batch has few columns c >= h
    // (uniform lengths with a nearly full last chunk): at most two CTAs per SM
    static const bool no_col1 = getenv("TFTB_NO_COL1") != nullptr;  // A/B knob
    const uint32_t h_uni = uni_n ? (uint32_t)(uni_n & (C - 1)) : 0;
    const int64_t cols2 = h_uni ? (int64_t)(C - h_uni) : 0;
    const size_t sm_col1 = (padded_words(1u << pl.l0) + kNT + 8) * sizeof(W);
    const bool narrow = inverse && col1 && !no_col1 && cols2 > 0 && cols2 * count <= 296;
    if (narrow && set_smem(col1, sm_col1)) return -1;
    if (pl.wlog != std::max(0, std::min(10, Limits<F>::col_t - pl.l0))) return fail("column plan mismatch");
    if (set_smem(colf, sm_col) || set_smem(coli, sm_col)) return -1;
    // chunk kernels for this plan's chunk size (2^CL, or 2^14 for the u64 words
    // past 2^26, make_plan)
    auto chunks = [&](auto cl) -> int {
        constexpr int CLK = decltype(cl)::value;
        if (set_smem(k_chunk_fwd<F, CLK>, sm_chunk) || set_smem(k_chunk_inv<F, CLK>, sm_chunk) ||
            set_smem(k_last_inv<F, CLK>, sm_chunk))
            return -1;
        for (int64_t v0 = 0; v0 < count; v0 += vchunk) {
            a.vbase = v0;
            unsigned nv = (unsigned)std::min(count - v0, vchunk);
            dim3 gcol(C >> pl.wlog, nv), gchunk((unsigned)maxchunks, nv), glast(1, nv);
            if (!inverse) {
                colf<<<gcol, kNT, sm_col, st>>>(a);
                k_chunk_fwd<F, CLK><<<gchunk, kNT, sm_chunk, st>>>(a);
                g_launches += 2;
            } else {
                k_chunk_inv<F, CLK><<<gchunk, kNT, sm_chunk, st>>>(a);
                if (narrow) col1<<<dim3((unsigned)cols2, nv), kNT, sm_col1, st>>>(a);
                else coli<<<gcol, kNT, sm_col, st>>>(a, 0);
                g_launches += 2;
                // uniform lengths that are whole chunks (2^k, 3 2^k, a p2r
                // prefix) have no partial chunk: steps 3 and 4 would be two
                // empty launches (~8 us of a single vector's inverse)
                if (!(uni_n && !h_uni)) {
                    k_last_inv<F, CLK><<<glast, kNT, sm_chunk, st>>>(a);
                    coli<<<gcol, kNT, sm_col, st>>>(a, 1);
                    g_launches += 2;
                }
            }
            CK(cudaGetLastError());
        }
        return 0;
    };
    if (pl.l1 == Limits<F>::CL) return chunks(std::integral_constant<int, Limits<F>::CL>{});
    if constexpr (Limits<F>::CL < 14) {
        if (pl.l1 == 14) return chunks(std::integral_constant<int, 14>{});
    }
    return fail("no chunk kernel for this plan");
}

// Build a reusable batch plan: vectors grouped by kernel plan, per-group
// device offset/length arrays and the largest stash, all allocated once.
template <class F>
int run_p2r(const RingHost* rh, LaunchArgs<F> a, int k, int r, int64_t count, VecDesc<typename F::W> xd,
            bool inverse, cudaStream_t st, typename F::W* stash_buf) {
    using W = typename F::W;
    const int64_t H = 1ll << k;
    VecDesc<W> pre_d = xd;  // the 2^k prefix of every vector
    pre_d.len = nullptr;
    pre_d.n0 = H;
    const int nb = p2r_blocks(count, H, r);
    const Tw<W>* tab = p2r_tables<F>(rh, k, r, nb);
    if (!tab) return -1;
    const int64_t vchunk = 65535;
    const int64_t cmax = std::min(count, vchunk);
    Scratch part;
    if (part.get((size_t)cmax * nb * kP2RMax * sizeof(W) + (size_t)cmax * sizeof(unsigned), st, true)) return -1;
    unsigned* ticket = reinterpret_cast<unsigned*>((W*)part.p + (size_t)cmax * nb * kP2RMax);
    CK(cudaMemsetAsync(ticket, 0, (size_t)cmax * sizeof(unsigned), st));
    P2RConsts<F> c{};
    auto launch = [&](bool inv) -> int {
        for (int64_t v0 = 0; v0 < count; v0 += vchunk) {
            a.vbase = v0;
            const unsigned nv = (unsigned)std::min(count - v0, vchunk);
            if (inv) k_p2r<F, true><<<dim3(nb, nv), 256, 0, st>>>(a, k, r, H, (W*)part.p, ticket, tab, c);
            else k_p2r<F, false><<<dim3(nb, nv), 256, 0, st>>>(a, k, r, H + r, (W*)part.p, ticket, tab, c);
            g_launches++;
            CK(cudaGetLastError());
        }
        return 0;
    };
    if (!inverse) {
        if (launch(false)) return -1;
        return run_group<F>(rh, a.x, nullptr, nullptr, count, pre_d, pre_d, H, false, st, stash_buf, H);
    }
    if (run_group<F>(rh, a.x, nullptr, a.pre, count, pre_d, pre_d, H, true, st, stash_buf, H)) return -1;
    // V[s][t] = rho_s^t, rho_s = omega_{2^k + s}: its inverse on the host
    {
        const uint64_t p = rh->p;
        uint64_t A[kP2RMax][2 * kP2RMax] = {};
        for (int s2 = 0; s2 < r; ++s2) {
            const uint64_t rho = omega_host(rh, (uint64_t)H + s2);
            uint64_t pw = 1;
            for (int t = 0; t < r; ++t) {
                A[s2][t] = pw;
                pw = mulmod(pw, rho, p);
            }
            A[s2][r + s2] = 1;
        }
        for (int col = 0; col < r; ++col) {
            int piv = col;
            while (piv < r && !A[piv][col]) ++piv;
            if (piv == r) return fail("p2r: singular Vandermonde system");
            for (int q = 0; q < 2 * r; ++q) std::swap(A[col][q], A[piv][q]);
            const uint64_t inv = powmod(A[col][col], p - 2, p);
            for (int q = 0; q < 2 * r; ++q) A[col][q] = mulmod(A[col][q], inv, p);
            for (int row = 0; row < r; ++row) {
                if (row == col || !A[row][col]) continue;
                const uint64_t fct = A[row][col];
                for (int q = 0; q < 2 * r; ++q) A[row][q] = (A[row][q] + p - mulmod(fct, A[col][q], p)) % p;
            }
        }
        for (int t = 0; t < r; ++t)
            for (int s2 = 0; s2 < r; ++s2) c.vinv[t][s2] = host_tw<F>(A[t][r + s2], p);
    }
    return launch(true);
}

template <class F>
int plan_create(const RingHost* rh, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                const int64_t* h_len, PlanImpl* P, cudaStream_t async_st, bool async,
                bool allow_fork) {
    using W = typename F::W;
    P->rh = rh;
    P->count = count;
    P->async = async;
    P->async_st = async_st;
    std::map<int, std::vector<int64_t>> groups;
    for (int64_t v = 0; v < count; v++) {
        int64_t nv = h_len ? h_len[v] : n;
        if (nv <= 0) return fail("vector length must be positive");
        Plan pl;
        if (make_plan<F>(nv, &pl)) return -1;
        groups[pl.key()].push_back(v);
    }
    size_t words = 0, stash_words = 0;
    bool fork = allow_fork && groups.size() > 1;
    for (auto& kv : groups) {
        PlanGroup g;
        g.count = (int64_t)kv.second.size();
        g.maxn = 0;
        std::vector<int64_t> off(g.count), len(g.count);
        for (int64_t i = 0; i < g.count; i++) {
            int64_t v = kv.second[i];
            off[i] = h_off ? h_off[v] : v * stride;
            len[i] = h_len ? h_len[v] : n;
            g.maxn = std::max(g.maxn, len[i]);
        }
        g.uni_n = g.maxn;
        for (int64_t i = 0; i < g.count; i++)
            if (len[i] != g.maxn) g.uni_n = 0;
        Plan pl;
        make_plan<F>(g.maxn, &pl);
        if (pl.kind == kLarge || pl.kind == kP2R)  // (p2r: its 2^k prefix runs the two-pass plan;
            // chunks are 2^CL words, 2^14 for u64 words past 2^26)
            stash_words = std::max(stash_words, (size_t)std::min<int64_t>(g.count, 65535) << 14);
        if (pl.kind == kP2R) {  // its power tables now, so execute only enqueues
            const int k = pl.l - 1;
            if (!p2r_tables<F>(rh, k, pl.G, p2r_blocks(g.count, 1ll << k, pl.G))) return -1;
        }
        fork &= pl.kind == kSmall || pl.kind == kCluster;
        g.arr_off = words;
        words += 2 * g.count;
        P->host_arrays.insert(P->host_arrays.end(), off.begin(), off.end());
        P->host_arrays.insert(P->host_arrays.end(), len.begin(), len.end());
        P->groups.push_back(g);
    }
    const size_t abytes = std::max<size_t>(words, 1) * sizeof(int64_t);
    if (async) {
        // pageable source: cudaMemcpyAsync returns once it is staged
        CK(cudaMallocAsync(&P->darr, abytes, async_st));
        CK(cudaMemcpyAsync(P->darr, P->host_arrays.data(), words * sizeof(int64_t), cudaMemcpyHostToDevice,
                           async_st));
        if (stash_words) CK(cudaMallocAsync(&P->stash, stash_words * sizeof(W), async_st));
    } else {
        CK(cudaMalloc(&P->darr, abytes));
        CK(cudaMemcpy(P->darr, P->host_arrays.data(), words * sizeof(int64_t), cudaMemcpyHostToDevice));
        if (stash_words) CK(cudaMalloc(&P->stash, stash_words * sizeof(W)));
    }
    if (stash_words) {
        g_aux_cur += (int64_t)(stash_words * sizeof(W));
        g_aux_peak = std::max(g_aux_peak, g_aux_cur);
        g_aux_cur -= (int64_t)(stash_words * sizeof(W));
    }
    P->fork = fork;
    if (fork) {
        const size_t ns = std::min<size_t>(P->groups.size(), kGroupStreams);
        P->side.resize(ns);
        for (auto& s2 : P->side) CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        P->ev_join.resize(P->groups.size());
        for (auto& e : P->ev_join) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return 0;
}

template <class F>
int plan_exec(const PlanImpl* P, void* data, int inverse, const void* pre, cudaStream_t st) {
    using W = typename F::W;
    // Groups are independent vectors.  Tile and cluster groups (no shared
    // stash, no scratch) fork onto the plan's side streams so one launch's
    // tail wave overlaps the next one's start; the join keeps `st` ordered
    // after all (fork/join through the plan's events: graph-capture safe).
    if (P->fork) CK(cudaEventRecord(P->ev_fork, st));
    int rc = 0;
    for (size_t i = 0; i < P->groups.size() && !rc; ++i) {
        const auto& g = P->groups[i];
        const int64_t* d = (const int64_t*)P->darr + g.arr_off;
        VecDesc<W> xd{d, d + g.count, 0, 0};
        cudaStream_t gs = st;
        if (P->fork) {
            gs = P->side[i % P->side.size()];
            CK(cudaStreamWaitEvent(gs, P->ev_fork, 0));
        }
        rc = run_group<F>(P->rh, (W*)data, nullptr, (const W*)pre, g.count, xd, xd, g.maxn, inverse != 0, gs,
                          (W*)P->stash, g.uni_n);
        if (P->fork) CK(cudaEventRecord(P->ev_join[i], gs));
    }
    if (P->fork)
        for (size_t i = 0; i < P->groups.size(); ++i) CK(cudaStreamWaitEvent(st, P->ev_join[i], 0));
    return rc;
}

// Partition a batch by plan (ceil_lg of the length class) and run each group.
// Ragged batches build a temporary plan whose arrays are allocated, filled
// and released stream-ordered on `st`: asynchronous w.r.t. the host.
template <class F>
int run_batch(const RingHost* rh, void* data, const void* in, int64_t count, int64_t n, int64_t stride,
              const int64_t* h_off, const int64_t* h_len, const void* in_data, int64_t in_n,
              int64_t in_stride, const void* pre, bool inverse, cudaStream_t st) {
    using W = typename F::W;
    if (count <= 0) return 0;
    if (!h_off && !h_len) {
        VecDesc<W> xd{nullptr, nullptr, stride, n};
        VecDesc<W> ind{nullptr, nullptr, in_stride, in_n};
        return run_group<F>(rh, (W*)data, (const W*)in_data, (const W*)pre, count, xd, ind, n, inverse, st, nullptr, n);
    }
    (void)in;
    PlanImpl P;
    if (plan_create<F>(rh, count, n, stride, h_off, h_len, &P, st, true)) return -1;
    return plan_exec<F>(&P, data, inverse, pre, st);
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
        if (own.get((size_t)count * r * sizeof(W), st, true)) return -1;
        scratch = own.p;
    }
    // X_v <- TFT_r(a_v || 0), Y_v <- TFT_r(b_v || 0), X_v <- ITFT_r(X_v * Y_v)
    if (run_batch<F>(rh, x, nullptr, count, r, sx, nullptr, nullptr, a, la, sa, nullptr, false, st)) return -1;
    if (run_batch<F>(rh, scratch, nullptr, count, r, r, nullptr, nullptr, b, lb, sb, nullptr, false, st)) return -1;
    if (run_batch<F>(rh, x, nullptr, count, r, sx, nullptr, nullptr, nullptr, 0, 0, scratch, true, st)) return -1;
    return 0;
}


}  // namespace tftb

#define TFTB_INSTANTIATE(F)                                                                                   \
    template int tftb::plan_create<F>(const RingHost*, int64_t, int64_t, int64_t, const int64_t*, const int64_t*, \
                                      PlanImpl*, cudaStream_t, bool, bool);                                                               \
    template int tftb::plan_exec<F>(const PlanImpl*, void*, int, const void*, cudaStream_t);                  \
    template int tftb::dispatch_tft<F>(const RingHost*, void*, int64_t, int64_t, int64_t, const int64_t*,     \
                                       const int64_t*, int, cudaStream_t);                                      \
    template int tftb::dispatch_mul<F>(const RingHost*, const void*, int64_t, int64_t, const void*, int64_t, \
                                       int64_t, void*, int64_t, int64_t, void*, cudaStream_t);
