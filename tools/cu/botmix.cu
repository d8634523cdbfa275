// Bottom-round (SLO = 0, 5 stages, 32-word units) variants on a resident
// 2^14-word tile, 3 CTAs/SM: what limits the bottom round -- twiddle
// loads (L2) or the butterfly arithmetic -- for F30 and F32.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

// single-word twiddles from a 256-entry window (L1-resident; numerically
// meaningless): same instruction stream as TwDirectM without L2 traffic
struct TwSmallM {
    const uint32_t* ZM;
    uint32_t pinv;
    template <int N>
    TFT_DEV void get_many(int, uint32_t J0, Tw<uint32_t>* out) const { ldg_word_run<N>(ZM + (J0 & 255 & ~(N - 1)), pinv, out); }
};
struct TwSmallP {
    const Tw<uint32_t>* Z;
    template <int N>
    TFT_DEV void get_many(int, uint32_t J0, Tw<uint32_t>* out) const { ldg_tw_run<uint32_t, N>(Z + (J0 & 255 & ~(N - 1)), out); }
};

// F30M with both outputs from hi and u directly: x = (ra + p) + hi - u,
// y = (ra + p) - hi + u  (ra = red2(a) in [0, 2p); outputs in [0, 4p))
struct F30M2 : F30 {
    TFT_DEV explicit F30M2(const F30& f) : F30(f) {}
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        const W ra = red2(x) + p;
        const W hi = __umulhi(y, t.w);
        const W u = __umulhi(y * t.wp, p);
        x = ra + hi - u;
        y = ra - hi + u;
    }
};
// F32 butterfly with the sum as a - (p - b) (borrow <=> a + b < p)
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
};

template <class FF, class TP>
__device__ __forceinline__ void bot(const FF& f, uint32_t* S, const TP& tp) {
    fwd_round_units<FF, 14, 5, 0, 0, false>(f, S, tp, 0, cta_lanes());
    __syncthreads();
}

template <class F, int MODE>
__global__ void __launch_bounds__(256, 3) kbot(F f, const Tw<uint32_t>* Z, const uint32_t* ZM, uint32_t* out, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
    for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) S[i + (i >> 5)] = i * 2654435761u % f.p;
    __syncthreads();
    const TwDirect<F> tp{Z, blockIdx.x & 3, 14, f, ZM};
    for (int r = 0; r < reps; ++r) {
        if constexpr (std::is_same<F, F30>::value) {
            if constexpr (MODE == 0) bot(F30M(f), S, tp.mont());                       // shipped
            if constexpr (MODE == 1) bot(F30M(f), S, TwSmallM{ZM, f.pinv});             // L1 twiddles
            if constexpr (MODE == 2) bot(F30M2(f), S, tp.mont());                      // alt butterfly
            if constexpr (MODE == 3) bot(F30M2(f), S, TwSmallM{ZM, f.pinv});
            if constexpr (MODE == 4) bot(f, S, TwSmallP{Z});                           // Shoup, L1 pairs
            if constexpr (MODE == 5) bot(f, S, tp);                                    // Shoup, L2 pairs
        } else {
            if constexpr (MODE == 0) bot(f, S, tp.mont());
            if constexpr (MODE == 1) bot(f, S, TwSmallM{ZM, f.pinv});
            if constexpr (MODE == 2) bot(F32B(f), S, tp.mont());
            if constexpr (MODE == 3) bot(F32B(f), S, TwSmallM{ZM, f.pinv});
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
}

template <class F, int MODE>
void run(const char* name, F f, Tw<uint32_t>* Z, uint32_t* ZM, uint32_t* out) {
    size_t smem = (16384 + 512 + 1) * 4;
    cudaFuncSetAttribute(kbot<F, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int reps = 40, grid = 148 * 3 * 4;
    float best = 1e9;
    for (int k = 0; k < 3; ++k) {
        cudaEventRecord(a);
        kbot<F, MODE><<<grid, 256, smem>>>(f, Z, ZM, out, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (k) best = ms < best ? ms : best;
    }
    double bf = (double)grid * reps * 5 * 8192;
    printf("%-22s %8.3f ms  %6.2f butterflies/clk/SM @1.965GHz  (%s)\n", name, best, bf / (best * 1e-3) / 148 / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
}

template <class F>
void tables(F f, uint64_t p, bool shoup, Tw<uint32_t>** Z, uint32_t** ZM) {
    std::vector<Tw<uint32_t>> h(1 << 16);
    std::vector<uint32_t> hm(1 << 16);
    for (size_t j = 0; j < h.size(); ++j) {
        uint64_t w = (j * 7919ull + 1) % p;
        uint32_t wm = (uint32_t)(((unsigned __int128)w << 32) % p);
        if (shoup) h[j] = {(uint32_t)w, (uint32_t)(((unsigned __int128)w << 32) / p)};
        else h[j] = {wm, wm * (uint32_t)f.pinv};
        hm[j] = wm;
    }
    cudaMalloc(Z, h.size() * 8);
    cudaMemcpy(*Z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(ZM, hm.size() * 4);
    cudaMemcpy(*ZM, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice);
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
        Tw<uint32_t>* Z;
        uint32_t* ZM;
        tables(f, p, true, &Z, &ZM);
        printf("== F30 bottom round\n");
        run<F30, 0>("F30M L2 (shipped)", f, Z, ZM, out);
        run<F30, 1>("F30M L1", f, Z, ZM, out);
        run<F30, 2>("F30M2 L2", f, Z, ZM, out);
        run<F30, 3>("F30M2 L1", f, Z, ZM, out);
        run<F30, 4>("Shoup pairs L1", f, Z, ZM, out);
        run<F30, 5>("Shoup pairs L2", f, Z, ZM, out);
    }
    {
        const uint32_t p = 3221225473u;
        F32 f;
        f.p = p;
        f.p2 = 0;
        uint32_t x = p;
        for (int i = 0; i < 6; ++i) x *= 2u - p * x;
        f.pinv = x;
        Tw<uint32_t>* Z;
        uint32_t* ZM;
        tables(f, p, false, &Z, &ZM);
        printf("== F32 bottom round\n");
        run<F32, 0>("F32 L2 (shipped)", f, Z, ZM, out);
        run<F32, 1>("F32 L1", f, Z, ZM, out);
        run<F32, 2>("F32B L2", f, Z, ZM, out);
        run<F32, 3>("F32B L1", f, Z, ZM, out);
    }
}
