// F32W (field.cuh) against 64-bit reference arithmetic: wide adds, subtracts,
// forward and inverse butterflies on random and edge words, p = 3221225473.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o f32wide f32wide.cu && ./f32wide
#include <cstdio>
#include <cstdlib>
#include "../../paper_1001_5272_b200/csrc/field.cuh"

__global__ void k(F32 f0, const uint32_t* in, int n, unsigned* bad) {
    const F32W f(f0);
    const uint64_t p = f.p;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t a = in[3 * i], bw = in[3 * i + 1], w = in[3 * i + 2] % f.p;
        const uint32_t bc = bw % f.p;
        if (f.addw(a, bc) % p != ((uint64_t)a + bc) % p) atomicAdd(bad + 0, 1);
        if (f.subw(a, bc) % p != ((uint64_t)a % p + p - bc) % p) atomicAdd(bad + 1, 1);
        const Tw<uint32_t> t = f.tw(w);
        // mulw(b, t) = b w R^-1: compare through R: mulw * 2^32 == b w (mod p)
        const uint32_t m = f.mulw(bw, t);
        if (m >= p || (uint64_t)m * (4294967296ull % p) % p != (uint64_t)(bw % p) * w % p) atomicAdd(bad + 2, 1);
        uint32_t x = a, y = bw;
        f.fwd(x, y, t);
        if (x % p != ((uint64_t)a + m) % p || y % p != ((uint64_t)a % p + p - m) % p) atomicAdd(bad + 3, 1);
        x = a, y = bw;
        f.inv(x, y, t);
        const uint32_t d = (uint32_t)(((uint64_t)a % p + p - bc) % p);
        if (x % p != ((uint64_t)a + bc) % p || y != f.mulw(d, t)) atomicAdd(bad + 4, 1);
        if (f.narrow(a) != a % p) atomicAdd(bad + 5, 1);
    }
}

int main() {
    F32 f{};
    f.p = 3221225473u;
    uint32_t inv = 1;
    for (int i = 0; i < 5; ++i) inv *= 2 - f.p * inv;
    f.pinv = inv;
    const int n = 1 << 20;
    uint32_t* h = (uint32_t*)malloc(3 * n * 4);
    const uint32_t edge[] = {0, 1, f.p - 1, f.p, f.p + 1, 0xFFFFFFFFu, 0x80000000u, 1073741823u, 1073741824u};
    srand(1);
    for (int i = 0; i < 3 * n; ++i) h[i] = i < 729 * 3 ? edge[(i % 3 == 0 ? i / 3 : i % 3 == 1 ? i / 27 : i / 243) % 9]
                                                     : ((uint32_t)rand() << 16) ^ rand();
    uint32_t* d; unsigned* bad;
    cudaMalloc(&d, 3 * n * 4); cudaMalloc(&bad, 32); cudaMemset(bad, 0, 32);
    cudaMemcpy(d, h, 3 * n * 4, cudaMemcpyHostToDevice);
    k<<<148, 256>>>(f, d, n, bad);
    unsigned hb[8];
    cudaMemcpy(hb, bad, 32, cudaMemcpyDeviceToHost);
    printf("mismatches addw %u subw %u mulw %u fwd %u inv %u narrow %u (%s)\n", hb[0], hb[1], hb[2], hb[3], hb[4], hb[5],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
