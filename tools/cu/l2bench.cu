// L2 -> SM read bandwidth: every CTA streams (16-byte loads) over a buffer
// small enough to stay L2-resident, many times.  Also the HBM figure for a
// buffer much larger than L2, for comparison.
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(256) kread(const uint4* __restrict__ p, size_t n16, int reps, uint32_t* out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)r * 977; i < n16 + (size_t)r * 977;
             i += stride * 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                size_t j = (i + u * stride) % n16;
                v[u] = __ldcg(p + j);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 4);
    for (size_t mb : {32, 64, 96, 4096}) {
        size_t bytes = mb << 20, n16 = bytes / 16;
        uint4* p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 1, bytes);
        int reps = mb <= 96 ? 20 : 2;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int it = 0; it < 3; ++it) {
            cudaEventRecord(a);
            kread<<<148 * 8, 256>>>(p, n16, reps, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it) printf("%4zu MB x %d: %.1f GB/s\n", mb, reps, (double)bytes * reps / (ms * 1e-3) / 1e9);
        }
        cudaFree(p);
    }
}
