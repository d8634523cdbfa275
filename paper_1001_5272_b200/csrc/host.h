// Host-side declarations shared by the libtftb200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "tile.cuh"

namespace tftb {


typedef unsigned __int128 u128;

extern thread_local std::string g_err;
extern thread_local int64_t g_launches;
extern unsigned long long* g_tail_timing;  // debug (debug.cu tftb_debug_tail_timing); null in production
// device bytes a transform allocates beyond its own n words (stash, p2r
// partials, the product's second operand): current and high-water mark of
// this thread's calls -- the footprint audit (tftb_aux_bytes)
extern thread_local int64_t g_aux_cur, g_aux_peak;
// device bytes the host-pointer entry points allocate for the caller's words
// (ring words + conversion staging): current and high-water mark
extern thread_local int64_t g_stage_cur, g_stage_peak;

inline int fail(const std::string& msg) {
    g_err = msg;
    return -1;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return fail(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
inline uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    a %= p;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}
inline int ceil_lg(int64_t n) {
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
W inv_word(W p) {  // p^-1 mod 2^bits (Newton)
    W x = p;
    for (int i = 0; i < 7; i++) x *= (W)2 - p * x;
    return x;
}

template <class F>
F make_field(uint64_t p) {
    F f;
    f.p = (typename F::W)p;
    f.p2 = (typename F::W)(2 * p);
    f.pinv = inv_word<typename F::W>((typename F::W)p);
    if constexpr (std::is_same<F, F30>::value) {
        f.npinv = (uint32_t)(0u - f.pinv);
        f.c32 = (uint32_t)(((unsigned __int128)1 << 32) % p);
        f.c32s = (uint32_t)(((unsigned __int128)f.c32 << 32) / p);
    }
    return f;
}

template <class F>
const RingDev<typename F::W>& ring_dev(const RingHost* rh);
template <>
inline const RingDev<uint32_t>& ring_dev<F30>(const RingHost* rh) { return rh->r32; }
template <>
inline const RingDev<uint32_t>& ring_dev<F32>(const RingHost* rh) { return rh->r32; }
template <>
inline const RingDev<uint64_t>& ring_dev<F62>(const RingHost* rh) { return rh->r64; }

// -------------------------------------------------------------- planning
constexpr int kNT = 256;

template <class F>
struct Limits {
    // log2 words of one CTA's shared-memory chunk (64 KB) and of the column tiles
    static constexpr int CL = sizeof(typename F::W) == 4 ? 14 : 13;
    static constexpr int col_t = sizeof(typename F::W) == 4 ? 14 : 13;
};

enum PlanKind { kSmall = 0, kCluster = 1, kLarge = 2, kP2R = 3 };

// n = 2^k + r with r <= kP2RMax beyond the cluster range runs as the 2^k
// transform plus r dot products (p2r.cuh) instead of a half-empty two-pass plan
constexpr int kP2RMax = 4;

struct Plan {
    PlanKind kind;
    int l, l0, l1, wlog, G;
    // small vectors group by tile size class, cluster ones by chunk count
    // (p2r: n itself, as 2^(l-1) + G)
    int key() const {
        return kind == kSmall ? -100 + l : kind == kCluster ? 1000 + G : kind == kP2R ? 3000 + 8 * l + G : l;
    }
};

template <class F>
int make_plan(int64_t n, Plan* pl, bool p2r_ok = true) {
    const int l = ceil_lg(n);
    pl->l = l;
    pl->l0 = pl->l1 = pl->wlog = 0;
    pl->G = 1;
    const int CL = Limits<F>::CL;
    if (l <= CL) {
        pl->kind = kSmall;
        return 0;
    }
    if (n <= (8ll << CL)) {
        pl->kind = kCluster;
        pl->G = (int)((n + (1ll << CL) - 1) >> CL);
        return 0;
    }
    static const bool no_p2r = getenv("TFTB_NO_P2R") != nullptr;  // A/B knob
    if (p2r_ok && !no_p2r && l - 1 > CL + 3 && n - (1ll << (l - 1)) <= kP2RMax) {
        pl->kind = kP2R;
        pl->G = (int)(n - (1ll << (l - 1)));
        return 0;
    }
    pl->kind = kLarge;
    // chunks are one CTA's shared-memory tile (2^CL words); columns take the
    // rest, as many adjacent columns per CTA as fit a 2^col_t-word tile
    int l1 = CL;
    int l0 = l - l1;
    int col_max = Limits<F>::col_t;
    if (l0 > col_max && CL < 14) {
        // u64 words past 2^26: 2^14-word (128 KB) chunk and column tiles, one
        // CTA per SM -- slower per word, but it reaches 2^28 in two passes
        l1 = 14;
        l0 = l - l1;
        col_max = 14;
    }
    // up to 1024 adjacent columns (a 64 KB tile for 16-row columns)
    int wlog = std::max(0, std::min(10, Limits<F>::col_t - l0));
    if (l0 + wlog > col_max) return fail("transform length too large for the two-pass plan");
    pl->l0 = l0;
    pl->l1 = l1;
    pl->wlog = wlog;
    return 0;
}

template <class K_>
int set_smem(K_ kern, size_t bytes) {
    // one attribute call per (kernel, device) for the largest size seen
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    if (bytes <= 48 * 1024) return 0;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[{(const void*)kern, dev}];
    if (bytes <= cur) return 0;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
    return 0;
}

struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    bool aux = false;
    cudaStream_t s = nullptr;
    // aux: auxiliary space of the algorithm (counted by the footprint audit),
    // as opposed to host-API staging of the caller's own words
    int get(size_t b, cudaStream_t st, bool is_aux = false) {
        s = st;
        if (b == 0) return 0;
        CK(cudaMallocAsync(&p, b, st));
        bytes = b;
        aux = is_aux;
        if (aux) {
            g_aux_cur += (int64_t)b;
            g_aux_peak = std::max(g_aux_peak, g_aux_cur);
        } else {
            g_stage_cur += (int64_t)b;
            g_stage_peak = std::max(g_stage_peak, g_stage_cur);
        }
        return 0;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
        if (p && aux) g_aux_cur -= (int64_t)bytes;
        if (p && !aux) g_stage_cur -= (int64_t)bytes;
    }
};


struct PlanGroup {
    int64_t count, maxn;
    int64_t uni_n = 0;  // the common length when every vector of the group has the same, else 0
    size_t arr_off;  // offsets then lengths, in darr
};

// A plan owns everything its execution touches besides the data: device
// offset/length arrays, the stash, the p2r tables (built at creation) and,
// when its groups fork, its own side streams and fork/join events -- so
// execute only enqueues work (graph-capturable) and two plans never share
// a stream.  A plan is not meant to be executed by two threads at once.
struct PlanImpl {
    const RingHost* rh = nullptr;
    int64_t count = 0;
    std::vector<PlanGroup> groups;
    std::vector<int64_t> host_arrays;
    void* darr = nullptr;
    void* stash = nullptr;
    bool fork = false;
    std::vector<cudaStream_t> side;
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    // temporary plans (tftb_tft_dev with host offsets): arrays allocated and
    // released stream-ordered on this stream, no host synchronisation
    cudaStream_t async_st = nullptr;
    bool async = false;
    ~PlanImpl() {
        if (async) {
            if (darr) cudaFreeAsync(darr, async_st);
            if (stash) cudaFreeAsync(stash, async_st);
        } else {
            if (darr) cudaFree(darr);
            if (stash) cudaFree(stash);
        }
        // (destroying a stream or event with pending work is legal: the
        // resources go once the work completes)
        for (auto e : ev_join) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        for (auto s : side) cudaStreamDestroy(s);
    }
};

template <class F>
int plan_create(const RingHost* rh, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                const int64_t* h_len, PlanImpl* P, cudaStream_t async_st, bool async, bool allow_fork = true);
template <class F>
int plan_exec(const PlanImpl* P, void* data, int inverse, const void* pre, cudaStream_t st);

int get_ring(uint64_t p, uint64_t top, int K, RingHost** out);  // tftb200.cu

// defined per field in inst_f30.cu / inst_f32.cu / inst_f62.cu
template <class F>
int dispatch_tft(const RingHost* rh, void* data, int64_t count, int64_t n, int64_t stride, const int64_t* h_off,
                 const int64_t* h_len, int inverse, cudaStream_t st);
template <class F>
int dispatch_mul(const RingHost* rh, const void* a, int64_t la, int64_t sa, const void* b, int64_t lb, int64_t sb,
                 void* x, int64_t sx, int64_t count, void* scratch, cudaStream_t st);

}  // namespace tftb
