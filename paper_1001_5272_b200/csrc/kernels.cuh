// TFT / ITFT / product kernels.
//
// Every vector of length n is handled as the first n outputs of the
// zero-padded power-of-two network (the TFT "prefix property",
// reference tests/test_transforms.py:89-98), but only n words of it ever live
// in HBM:
//
//  * n <= 2^t_small: one CTA per vector, whole padded tile in shared memory.
//  * larger n, l = ceil_lg(n) = l0 + l1, C = 2^l1 ("chunk"), R = 2^l0 rows:
//      forward  A  columns c (stride C, R rows, deep stages, untwisted):
//                  full padded column transform in smem; rows < n written
//                  back; the single virtual row K = n>>l1 of columns c >= h
//                  (h = n mod C) goes to a <= C-word stash.
//               B  chunks k (contiguous C words, top stages, block twist k):
//                  the partial last chunk reads its virtual words from the
//                  stash; only positions < n are stored.
//      inverse  1  complete chunks k < K: plain inverse.
//               2  columns c >= h: in-tile ITFT of K rows; their virtual row K
//                  (sum_i x_i omega_K^i) into the stash.
//               3  last chunk (one CTA): h known outputs + C-h stashed inputs,
//                  in-tile generalised ITFT.
//               4  columns c < h: in-tile ITFT of K+1 rows.
// The stash is the only extra device memory besides the per-ring twiddle
// tables (PAPER.md:62 allows O(sqrt n) space for the cache-friendly variant).
#pragma once
#include "tile.cuh"


template <typename W>
struct VecDesc {
    const int64_t* off;  // per-vector word offset, or null -> stride*v
    const int64_t* len;  // per-vector length, or null -> n0
    int64_t stride, n0;
    TFT_DEV int64_t o(int64_t v) const { return off ? off[v] : stride * v; }
    TFT_DEV int64_t n(int64_t v) const { return len ? len[v] : n0; }
};

template <class F>
struct LaunchArgs {
    using W = typename F::W;
    F f;
    RingDev<W> R;
    W* x;                 // data vectors (in place)
    VecDesc<W> xd;
    const W* in;          // forward input (== x for a transform; A or B for a product)
    VecDesc<W> ind;       // in_len <= n; positions >= in_len read as 0
    const W* pre;         // inverse: optional pointwise factor (product: X^ * Y^)
    W* stash;             // per-vector stash, C words each
    int l0, l1, wlog;     // two-pass plan (large kernels)
    int64_t vbase;        // first vector of this launch
    unsigned long long* timing;  // debug: per-CTA phase timestamps (null in production)
    unsigned* done;              // per-vector chunk tickets (fused split inverse), v - vbase
    int dense_cols;              // A/B: dense V^-1 column solves (TFTB_DENSE_COLS)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Phase stamps compile only into the kernels' TIM = true instantiations
// (debug.cu): the volatile timer read is a scheduling barrier that cost the
// production kernels 1-3% when merely guarded at run time (measured).
#define TFTB_STAMP(a, k)                                                                                   \
    do {                                                                                                   \
        if constexpr (TIM) {                                                                               \
            if ((a).timing && threadIdx.x == 0)                                                            \
                (a).timing[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 + (k)] = gtime();             \
        }                                                                                                  \
    } while (0)

// Stamps of the single-CTA tail kernels of a large inverse (k_col1_inv,
// k_last_inv): run-time guarded -- these kernels are latency chains of one
// CTA, the guard costs them nothing (timing is null in production)
#define TFTB_TAIL_STAMP(a, k)                                                                     \
    do {                                                                                          \
        if ((a).timing && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) (a).timing[k] = gtime(); \
    } while (0)

// Hint: bring words [p, p + words) into L2 with TMA bulk prefetches (the
// copy engine streams them while the SM works).  Only the 16-byte-aligned
// inner span, so it never touches bytes outside the range.
template <typename W>
TFT_DEV void l2_prefetch(const W* p, int64_t words) {
    if (words <= 0) return;
    uintptr_t lo = ((uintptr_t)p + 15) & ~(uintptr_t)15;
    const uintptr_t hi = ((uintptr_t)(p + words)) & ~(uintptr_t)15;
    for (; lo < hi; lo += 32768) {
        const uint32_t sz = (uint32_t)min((uintptr_t)32768, hi - lo);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(sz) : "memory");
    }
}

// X^ * Y^ : Montgomery product then * R^2 to undo the R^-1.
template <class F>
TFT_DEV typename F::W pre_mul(const LaunchArgs<F>& a, typename F::W v, typename F::W pw) {
    return a.f.canon(a.f.mont(a.f.red1(a.f.mont(v, pw)), a.R.r2w));
}
template <class F>
TFT_DEV typename F::W load_pre(const LaunchArgs<F>& a, int64_t idx, typename F::W v) {
    if (!a.pre) return v;
    return pre_mul(a, v, a.pre[idx]);
}

// ------------------------------------------------------ tile <-> HBM streaming
// 16-byte vectors of words
template <typename W>
struct Vec16;
template <>
struct Vec16<uint32_t> {
    using T = uint4;
    static constexpr int N = 4;
    TFT_DEV static uint32_t get(const T& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
    TFT_DEV static T make(const uint32_t* e) { return T{e[0], e[1], e[2], e[3]}; }
    TFT_DEV static T zero() { return T{0, 0, 0, 0}; }
};
template <>
struct Vec16<uint64_t> {
    using T = ulonglong2;
    static constexpr int N = 2;
    TFT_DEV static uint64_t get(const T& v, int i) { return i == 0 ? v.x : v.y; }
    TFT_DEV static T make(const uint64_t* e) { return T{e[0], e[1]}; }
    TFT_DEV static T zero() { return T{0, 0}; }
};

template <typename T>
TFT_DEV T ld_stream(const T* p) { return __ldcs(p); }  // read once: evict-first

// S[phys(i)] = xf(i, i < avail ? src[i] : 0) for i < C (phys(i) = i + i/32),
// with 16-byte loads for the aligned body and UNR of them in flight per thread
// (a tile load is one HBM latency, not C/blockDim of them).
template <typename W, int UNR = 8, class XF>
TFT_DEV void tile_load(W* S, const W* src, int64_t avail, uint32_t C, const XF& xf, Lanes ln = cta_lanes()) {
    using V = Vec16<W>;
    constexpr int NV = V::N;
    const uint32_t mis = (uint32_t)(((uintptr_t)src & 15) / sizeof(W));
    const uint32_t head = min(C, (uint32_t)((NV - mis) % NV));
    for (uint32_t i = ln.id; i < head; i += ln.n) S[i + (i >> 5)] = xf(i, (int64_t)i < avail ? src[i] : W(0));
    const uint32_t nq = (C - head) / NV;
    const typename V::T* vs = reinterpret_cast<const typename V::T*>(src + head);
    // quads [0, nfull) lie wholly below avail: no per-word checks there
    const int64_t rest = avail - (int64_t)head;
    const uint32_t nfull = rest <= 0 ? 0u : (uint32_t)min((int64_t)nq, rest / NV);
    for (uint32_t k0 = ln.id; k0 < nfull; k0 += ln.n * UNR) {
        typename V::T buf[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t k = k0 + u * ln.n;
            if (k < nfull) buf[u] = ld_stream(vs + k);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t k = k0 + u * ln.n;
            if (k >= nfull) break;
            const uint32_t i = head + k * NV;
#pragma unroll
            for (int q = 0; q < NV; ++q) S[(i + q) + ((i + q) >> 5)] = xf(i + q, V::get(buf[u], q));
        }
    }
    // the (at most one) partial quad and the zero quads past avail
    for (uint32_t k = nfull + ln.id; k < nq; k += ln.n) {
        const uint32_t i = head + k * NV;
#pragma unroll
        for (int q = 0; q < NV; ++q) S[(i + q) + ((i + q) >> 5)] = xf(i + q, (int64_t)(i + q) < avail ? src[i + q] : W(0));
    }
    for (uint32_t i = head + nq * NV + ln.id; i < C; i += ln.n)
        S[i + (i >> 5)] = xf(i, (int64_t)i < avail ? src[i] : W(0));
}

// tile_load of the pointwise product src[i] * pre[i] (the product's fused
// inverse input): both operands in 16-byte quads, issued together, when
// they share their alignment (the product's two buffers do); else the
// scalar second operand of load_pre.
template <class F, int UNR = 4>
TFT_DEV void tile_load_pre(const LaunchArgs<F>& a, typename F::W* S, const typename F::W* src,
                           const typename F::W* pre, int64_t avail, uint32_t C, Lanes ln = cta_lanes()) {
    using W = typename F::W;
    using V = Vec16<W>;
    constexpr int NV = V::N;
    const uint32_t mis = (uint32_t)(((uintptr_t)src & 15) / sizeof(W));
    if (mis != (uint32_t)(((uintptr_t)pre & 15) / sizeof(W))) {
        tile_load<W>(S, src, avail, C, [&](uint32_t i, W w) { return (int64_t)i < avail ? pre_mul(a, w, pre[i]) : W(0); }, ln);
        return;
    }
    const uint32_t head = min(C, (uint32_t)((NV - mis) % NV));
    auto one = [&](uint32_t i) { S[i + (i >> 5)] = (int64_t)i < avail ? pre_mul(a, src[i], pre[i]) : W(0); };
    for (uint32_t i = ln.id; i < head; i += ln.n) one(i);
    const uint32_t nq = (C - head) / NV;
    const int64_t rest = avail - (int64_t)head;
    const uint32_t nfull = rest <= 0 ? 0u : (uint32_t)min((int64_t)nq, rest / NV);
    const typename V::T* vs = reinterpret_cast<const typename V::T*>(src + head);
    const typename V::T* vp = reinterpret_cast<const typename V::T*>(pre + head);
    for (uint32_t k0 = ln.id; k0 < nfull; k0 += ln.n * UNR) {
        typename V::T bx[UNR], bp[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t k = k0 + u * ln.n;
            if (k < nfull) {
                bx[u] = ld_stream(vs + k);
                bp[u] = ld_stream(vp + k);
            }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t k = k0 + u * ln.n;
            if (k >= nfull) break;
            const uint32_t i = head + k * NV;
#pragma unroll
            for (int q = 0; q < NV; ++q) S[(i + q) + ((i + q) >> 5)] = pre_mul(a, V::get(bx[u], q), V::get(bp[u], q));
        }
    }
    for (uint32_t i = head + nfull * NV + ln.id; i < C; i += ln.n) one(i);
}

// dst[i] = cv(S[phys(i)]) for i < lim, 16-byte stores for the aligned body
template <typename W, class CV, bool STREAM = true>
TFT_DEV void tile_store(W* dst, const W* S, uint32_t lim, const CV& cv, Lanes ln = cta_lanes()) {
    using V = Vec16<W>;
    constexpr int NV = V::N;
    const uint32_t mis = (uint32_t)(((uintptr_t)dst & 15) / sizeof(W));
    const uint32_t head = min(lim, (uint32_t)((NV - mis) % NV));
    for (uint32_t i = ln.id; i < head; i += ln.n) dst[i] = cv(S[i + (i >> 5)]);
    const uint32_t nq = (lim - head) / NV;
    typename V::T* vd = reinterpret_cast<typename V::T*>(dst + head);
    for (uint32_t k = ln.id; k < nq; k += ln.n) {
        const uint32_t i = head + k * NV;
        W e[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) e[q] = cv(S[(i + q) + ((i + q) >> 5)]);
        if constexpr (STREAM) __stcs(vd + k, V::make(e));
        else __stcg(vd + k, V::make(e));  // re-read soon from L2
    }
    for (uint32_t i = head + nq * NV + ln.id; i < lim; i += ln.n) dst[i] = cv(S[i + (i >> 5)]);
}

__device__ __forceinline__ int ceil_lg_dev(int64_t n) {
    return n <= 1 ? 0 : 64 - __clzll((unsigned long long)(n - 1));
}

// ------------------------------------------------------------ helpers
template <typename W>
__global__ void k_u64_to_w(const uint64_t* __restrict__ s, W* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (W)s[i];
}
template <typename W>
__global__ void k_w_to_u64(const W* __restrict__ s, uint64_t* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = (uint64_t)s[i];
}
