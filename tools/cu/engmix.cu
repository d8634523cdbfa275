// Round-engine arithmetic variants: butterfly formulations
// for the forward and inverse rounds, top (SLO >= 5) and bottom (SLO = 0),
// F30 (p < 2^30, lazy) and F32 (p = 3221225473, canonical), on a resident
// 2^14-word tile, 3 CTAs/SM, 256 threads.  Prints butterflies/clk/SM.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

// ---- F30 forward, single-word Montgomery twiddles, both outputs from hi, u
struct F30M2 : F30 {
    TFT_DEV explicit F30M2(const F30& f) : F30(f) {}
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W ra = red2(x) + p;
        const W hi = __umulhi(y, t.w);
        const W u = __umulhi(y * t.wp, p);
        x = ra + hi - u;
        y = ra - hi + u;
    }
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {  // REDC with the 64-bit sum (negated companion)
        const W s = red2(x + y);
        const W d = x - y + p2;
        x = s;
        const W m = d * (0u - t.wp);
        y = (W)(((uint64_t)d * t.w + (uint64_t)m * p) >> 32);
    }
};
// ---- F30 Shoup with the inverse's product in the REDC-like single-HI form
struct F30S2 : F30 {
    TFT_DEV explicit F30S2(const F30& f) : F30(f) {}
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W ra = red2(x);
        const W q = __umulhi(y, t.wp);
        const W b = y * t.w - q * p;
        x = ra + b;
        y = ra - b + p2;
    }
};
// ---- F32: sum as a - (p - b); inverse likewise
struct F32B : F32 {
    TFT_DEV explicit F32B(const F32& f) : F32(f) {}
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W b = mulw(y, t);
        const W a = x;
        const W nb = p - b;
        const W s = a - nb;
        x = a < nb ? s + p : s;
        const W d = a - b;
        y = a < b ? d + p : d;
    }
    TFT_DEV void inv(W& x, W& y, Tw<W> t) const {
        const W a = x, b = y;
        const W nb = p - b;
        const W s = a - nb;
        x = a < nb ? s + p : s;
        const W d = a - b;
        y = mulw(a < b ? d + p : d, t);
    }
};

template <class FF, int KK, int SLO, bool INV, class TP>
__device__ __forceinline__ void round1(const FF& f, uint32_t* S, const TP& tp, const Tw<uint32_t>* ip) {
    if constexpr (INV) inv_round_units<FF, 14, KK, SLO, 0, false, false>(f, S, tp, ip, 0, cta_lanes());
    else fwd_round_units<FF, 14, KK, SLO, 0, false>(f, S, tp, 0, cta_lanes());
    __syncthreads();
}

// MODE: 0 shipped field, 1 variant field (same twiddle provider kind)
template <class F, class FV, bool INV, int MODE>
__global__ void __launch_bounds__(256, 3) kr(F f, const Tw<uint32_t>* Z, const uint32_t* ZM, uint32_t* out, int reps,
                                             const Tw<uint32_t>* ip) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
    for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) S[i + (i >> 5)] = i * 2654435761u % f.p;
    __syncthreads();
    const TwDirect<F> tp{Z, blockIdx.x & 3, 14, f, ZM};
    const FV fv(f);
    for (int r = 0; r < reps; ++r) {
        // top rounds: pairs (shipped) or the variant field with pairs
        if constexpr (MODE == 0) { round1<F, 5, 9, INV>(f, S, tp, ip); round1<F, 4, 5, INV>(f, S, tp, ip); }
        if constexpr (MODE == 1) { round1<FV, 5, 9, INV>(fv, S, tp, ip); round1<FV, 4, 5, INV>(fv, S, tp, ip); }
        if constexpr (MODE == 2) { round1<FV, 5, 9, INV>(fv, S, tp.mont(), ip); round1<FV, 4, 5, INV>(fv, S, tp.mont(), ip); }
        // bottom round: shipped (bottom_field over words) or variant over words
        if constexpr (MODE == 3) {
            const auto fb = bottom_field(f);
            round1<decltype(fb), 5, 0, INV>(fb, S, tp.mont(), ip);
        }
        if constexpr (MODE == 4) round1<FV, 5, 0, INV>(fv, S, tp.mont(), ip);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
}

template <class F, class FV, bool INV, int MODE>
void run(const char* name, F f, Tw<uint32_t>* Z, uint32_t* ZM, uint32_t* out, const Tw<uint32_t>* ip) {
    size_t smem = (16384 + 512 + 1) * 4;
    auto k = kr<F, FV, INV, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int reps = 40, grid = 148 * 3 * 4;
    float best = 1e9;
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        k<<<grid, 256, smem>>>(f, Z, ZM, out, reps, ip);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it) best = ms < best ? ms : best;
    }
    double stages = MODE <= 2 ? 9 : 5;
    double bf = (double)grid * reps * stages * 8192;
    printf("%-34s %7.3f ms %6.2f bfly/clk/SM (%s)\n", name, best, bf / (best * 1e-3) / 148 / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
}

template <class F>
void tables(F f, uint64_t p, bool shoup, Tw<uint32_t>** Z, uint32_t** ZM, Tw<uint32_t>** ip) {
    std::vector<Tw<uint32_t>> h(1 << 16), hi(64);
    std::vector<uint32_t> hm(1 << 16);
    for (size_t j = 0; j < h.size(); ++j) {
        uint64_t w = (j * 7919ull + 1) % p;
        uint32_t wm = (uint32_t)(((unsigned __int128)w << 32) % p);
        if (shoup) h[j] = {(uint32_t)w, (uint32_t)(((unsigned __int128)w << 32) / p)};
        else h[j] = {wm, wm * (uint32_t)f.pinv};
        hm[j] = wm;
    }
    for (int j = 0; j < 64; ++j) hi[j] = h[j + 5];
    cudaMalloc(Z, h.size() * 8);
    cudaMemcpy(*Z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(ZM, hm.size() * 4);
    cudaMemcpy(*ZM, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(ip, 64 * 8);
    cudaMemcpy(*ip, hi.data(), 64 * 8, cudaMemcpyHostToDevice);
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 148 * 3 * 4 * 256 * 4);
    {
        const uint32_t p = 998244353u;
        F30 f;
        f.p = p;
        f.p2 = 2 * p;
        uint32_t x = p;
        for (int i = 0; i < 6; ++i) x *= 2u - p * x;
        f.pinv = x;
        f.npinv = 0u - x;
        f.c32 = (uint32_t)((1ull << 32) % p);
        f.c32s = (uint32_t)(((unsigned __int128)f.c32 << 32) / p);
        Tw<uint32_t>* Z; uint32_t* ZM; Tw<uint32_t>* ip;
        tables(f, p, true, &Z, &ZM, &ip);
        printf("== F30 forward\n");
        run<F30, F30M2, false, 0>("top  Shoup (shipped)", f, Z, ZM, out, ip);
        run<F30, F30S2, false, 1>("top  Shoup S2", f, Z, ZM, out, ip);
        run<F30, F30M2, false, 2>("top  F30M2 words", f, Z, ZM, out, ip);
        run<F30, F30M2, false, 3>("bot  F30M (shipped)", f, Z, ZM, out, ip);
        run<F30, F30M2, false, 4>("bot  F30M2", f, Z, ZM, out, ip);
        printf("== F30 inverse\n");
        run<F30, F30M2, true, 0>("top  Shoup (shipped)", f, Z, ZM, out, ip);
        run<F30, F30M2, true, 2>("top  F30M2 REDC words", f, Z, ZM, out, ip);
        run<F30, F30M2, true, 3>("bot  F30M (shipped)", f, Z, ZM, out, ip);
        run<F30, F30M2, true, 4>("bot  F30M2 REDC", f, Z, ZM, out, ip);
    }
    {
        const uint32_t p = 3221225473u;
        F32 f;
        f.p = p;
        f.p2 = 0;
        uint32_t x = p;
        for (int i = 0; i < 6; ++i) x *= 2u - p * x;
        f.pinv = x;
        Tw<uint32_t>* Z; uint32_t* ZM; Tw<uint32_t>* ip;
        tables(f, p, false, &Z, &ZM, &ip);
        printf("== F32 forward (canonical = the field outside the rounds; wide = F32W, what the rounds run)\n");
        run<F32, F32W, false, 0>("top  canonical", f, Z, ZM, out, ip);
        run<F32, F32W, false, 1>("top  wide (shipped)", f, Z, ZM, out, ip);
        run<F32, F32B, false, 4>("bot  canonical", f, Z, ZM, out, ip);
        run<F32, F32W, false, 3>("bot  wide (shipped)", f, Z, ZM, out, ip);
        printf("== F32 inverse\n");
        run<F32, F32W, true, 0>("top  canonical", f, Z, ZM, out, ip);
        run<F32, F32W, true, 1>("top  wide (shipped)", f, Z, ZM, out, ip);
        run<F32, F32B, true, 4>("bot  canonical", f, Z, ZM, out, ip);
        run<F32, F32W, true, 3>("bot  wide (shipped)", f, Z, ZM, out, ip);
    }
}
