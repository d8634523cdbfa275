// In-smem round throughput by variant (2^14-word tile resident, 3 CTAs/SM,
// 256 threads): which round and which twiddle form limits the tile engine.
//   cur      fwd_rounds_ct as shipped (Shoup top rounds, single-word
//            Montgomery twiddles in the bottom SLO = 0 round)
//   shoup    every round Shoup pairs (8-byte twiddles in the bottom round)
//   top      the two SLO >= 5 rounds only (5 @ 9, 4 @ 5)
//   bot_m / bot_s  the bottom round only, Montgomery words / Shoup pairs
// F32 (p = 3221225473, canonical Montgomery) likewise.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

template <class F>
struct NoMont {  // a TwDirect whose bottom round keeps the pair table
    static constexpr bool kMont = false;
    TwDirect<F> d;
    TFT_DEV Tw<typename F::W> get(int s, uint32_t J) const { return d.get(s, J); }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t J0, Tw<typename F::W>* out) const { d.template get_many<N>(s, J0, out); }
};

template <class F, int MODE>
__global__ void __launch_bounds__(256, 3) kround(F f, const Tw<uint32_t>* Z, const uint32_t* ZM, uint32_t* out, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
    for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) S[i + (i >> 5)] = i * 2654435761u % f.p;
    __syncthreads();
    const TwDirect<F> tp{Z, blockIdx.x & 3, 14, f, ZM};
    const NoMont<F> tn{tp};
    const Lanes ln = cta_lanes();
    for (int r = 0; r < reps; ++r) {
        if constexpr (MODE == 0) fwd_rounds_ct<F, 14, 14>(f, S, tp);
        if constexpr (MODE == 1) fwd_rounds_ct<F, 14, 14>(f, S, tn);
        if constexpr (MODE == 2) {
            fwd_round_ct<F, 14, 5, 9, 0, false>(f, S, tp, 0, ln);
            __syncthreads();
            fwd_round_ct<F, 14, 4, 5, 0, false>(f, S, tp, 0, ln);
            __syncthreads();
        }
        if constexpr (MODE == 3) {
            fwd_round_ct<F, 14, 5, 0, 0, false>(f, S, tp, 0, ln);
            __syncthreads();
        }
        if constexpr (MODE == 4) {
            fwd_round_ct<F, 14, 5, 0, 0, false>(f, S, tn, 0, ln);
            __syncthreads();
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
}

template <class F, int MODE>
void run(const char* name, F f, Tw<uint32_t>* Z, uint32_t* ZM, uint32_t* out) {
    size_t smem = (16384 + 512 + 1) * 4;
    cudaFuncSetAttribute(kround<F, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int reps = 40, grid = 148 * 3 * 4;
    double stages = MODE <= 1 ? 14 : MODE == 2 ? 9 : 5;
    float best = 1e9;
    for (int k = 0; k < 3; ++k) {
        cudaEventRecord(a);
        kround<F, MODE><<<grid, 256, smem>>>(f, Z, ZM, out, reps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (k) best = ms < best ? ms : best;
    }
    double bf = (double)grid * reps * stages * 8192;
    printf("%-10s %8.3f ms  %6.2f butterflies/clk/SM @1.965GHz  (%s)\n", name, best, bf / (best * 1e-3) / 148 / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
}

template <class F>
void all(const char* tag, F f, uint64_t p, bool shoup) {
    std::vector<Tw<uint32_t>> h(1 << 16);
    std::vector<uint32_t> hm(1 << 16);
    uint32_t pinv = f.pinv;
    for (size_t j = 0; j < h.size(); ++j) {
        uint64_t w = (j * 7919ull + 1) % p;
        uint32_t wm = (uint32_t)(((unsigned __int128)w << 32) % p);
        if (shoup) h[j] = {(uint32_t)w, (uint32_t)(((unsigned __int128)w << 32) / p)};
        else h[j] = {wm, wm * pinv};
        hm[j] = wm;
    }
    Tw<uint32_t>* Z;
    uint32_t *ZM, *out;
    cudaMalloc(&Z, h.size() * 8);
    cudaMemcpy(Z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&ZM, hm.size() * 4);
    cudaMemcpy(ZM, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 148 * 3 * 4 * 256 * 4);
    printf("== %s\n", tag);
    run<F, 0>("cur", f, Z, ZM, out);
    run<F, 1>("shoup", f, Z, ZM, out);
    run<F, 2>("top", f, Z, ZM, out);
    run<F, 3>("bot_m", f, Z, ZM, out);
    run<F, 4>("bot_pair", f, Z, ZM, out);
}

int main() {
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
        all<F30>("F30 p=998244353", f, p, true);
    }
    {
        const uint32_t p = 3221225473u;
        F32 f;
        f.p = p;
        f.p2 = 0;
        uint32_t x = p;
        for (int i = 0; i < 6; ++i) x *= 2u - p * x;
        f.pinv = x;
        all<F32>("F32 p=3221225473", f, p, false);
    }
}
