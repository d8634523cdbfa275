// Throughput of modular-multiply formulations on sm_100a (independent chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr uint32_t P = 998244353u;
__device__ __forceinline__ uint32_t redc(uint32_t b, uint32_t w, uint32_t wp) {
    uint32_t m = b * wp; uint64_t t = (uint64_t)b * w + (uint64_t)m * P; return (uint32_t)(t >> 32);
}
__device__ __forceinline__ uint32_t shoup(uint32_t b, uint32_t w, uint32_t ws) {
    uint32_t q = __umulhi(b, ws); return b * w - q * P;
}
template <int V>
__global__ void k(uint32_t* out, uint32_t w, uint32_t wp, int iters) {
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 16 + i + blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (V == 0) x[i] = redc(x[i], w, wp);
            else if (V == 1) x[i] = shoup(x[i], w, wp);
            else if (V == 2) x[i] = x[i] * w + wp;                     // plain IMAD
            else if (V == 3) x[i] = __umulhi(x[i], w) + wp;           // IMAD.HI
            else if (V == 4) { uint64_t t = (uint64_t)x[i] * w; x[i] = (uint32_t)(t >> 32) ^ (uint32_t)t; } // WIDE
            else if (V == 5) { uint32_t a = min(x[i], x[i] - 2 * P); uint32_t b = redc(x[i] ^ it, w, wp); x[i] = a + b; x[i + 0] ^= a - b + 2 * P; } // butterfly-ish
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    const char* names[] = {"redc", "shoup", "imad", "imad.hi", "imad.wide", "bfly"};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 4096;
    for (int v = 0; v < 6; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            switch (v) {
                case 0: k<0><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
                case 1: k<1><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
                case 2: k<2><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
                case 3: k<3><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
                case 4: k<4><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
                case 5: k<5><<<148 * 8, 256>>>(d, 12345, 678, iters); break;
            }
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = 148.0 * 8 * 256 * 16 * iters;
            if (rep) printf("%-10s %.3f ms  %.2f Tops/s  (%.1f ops/clk/SM @1.9GHz)\n", names[v], ms, ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.9e9);
        }
    }
    return 0;
}
