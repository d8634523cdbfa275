// Throughput of the in-smem forward rounds alone (2^14-word tile resident,
// rounds repeated), F30 with Shoup twiddles from a synthetic table.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

template <int MINB>
__global__ void __launch_bounds__(256, MINB) kround(F30 f, const Tw<uint32_t>* Z, uint32_t* out, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
    for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) S[i + (i >> 5)] = i * 2654435761u % f.p;
    __syncthreads();
    const TwDirect<F30> tp{Z, blockIdx.x & 3, 14, f};
    for (int r = 0; r < reps; ++r) fwd_rounds_ct<F30, 14, 14>(f, S, tp);
    out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
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
    uint32_t* out; cudaMalloc(&out, 148 * 3 * 4 * 256 * 4);
    size_t smem = (16384 + 512 + 1) * 4;
    cudaFuncSetAttribute(kround<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int reps = 40, grid = 148 * 3 * 4;
    for (int k = 0; k < 2; ++k) {
        cudaEventRecord(a);
        kround<3><<<grid, 256, smem>>>(f, Z, out, reps);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bf = (double)grid * reps * 14 * 8192;
        printf("rounds: %.3f ms, %.2f butterflies/clk/SM @1.9GHz (err %s)\n", ms, bf / (ms * 1e-3) / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
    }
}
