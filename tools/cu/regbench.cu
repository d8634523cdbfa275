// Butterfly throughput with no shared memory: each thread repeats the 5
// layers of a 32-word register unit (reg_fwd, F30 Shoup), twiddles from a
// small L1-resident table.  MINB sets the register budget.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

template <int MINB, int KK>
__global__ void __launch_bounds__(256, MINB) kreg(F30 f, const Tw<uint32_t>* Z, uint32_t* out, int reps) {
    uint32_t v[1 << KK];
#pragma unroll
    for (int i = 0; i < (1 << KK); ++i) v[i] = (threadIdx.x * 2654435761u + i * 40503u) % f.p;
    const TwDirect<F30> tp{Z, 0, 14, f};
    for (int r = 0; r < reps; ++r) reg_fwd<F30, KK, KK - 1>(f, v, (threadIdx.x & 31) << KK, 0, tp);
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < (1 << KK); ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MINB, int KK>
void run(F30 f, Tw<uint32_t>* Z, uint32_t* out) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int reps = 400, grid = 148 * MINB * 4;
    for (int k = 0; k < 3; ++k) {
        cudaEventRecord(a);
        kreg<MINB, KK><<<grid, 256>>>(f, Z, out, reps);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bf = (double)grid * 256 * reps * KK * (1 << (KK - 1));
        if (k) printf("MINB=%d KK=%d: %.3f ms, %.2f butterflies/clk/SM @1.965GHz (%s)\n", MINB, KK, ms,
                      bf / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    const uint32_t p = 998244353u;
    F30 f;
    f.p = p; f.p2 = 2 * p;
    uint32_t x = p; for (int i = 0; i < 6; ++i) x *= 2u - p * x;
    f.pinv = x; f.npinv = 0u - x; f.c32 = (uint32_t)((1ull << 32) % p); f.c32s = (uint32_t)(((unsigned __int128)f.c32 << 32) / p);
    std::vector<Tw<uint32_t>> h(1 << 16);
    for (size_t j = 0; j < h.size(); ++j) { uint32_t w = (uint32_t)((j * 7919ull + 1) % p); h[j] = {w, (uint32_t)(((unsigned __int128)w << 32) / p)}; }
    Tw<uint32_t>* Z; cudaMalloc(&Z, h.size() * 8); cudaMemcpy(Z, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    uint32_t* out; cudaMalloc(&out, 148 * 8 * 4 * 256 * 4);
    run<2, 5>(f, Z, out);
    run<3, 5>(f, Z, out);
    run<4, 5>(f, Z, out);
    run<6, 4>(f, Z, out);
    run<8, 3>(f, Z, out);
}
