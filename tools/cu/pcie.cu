#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>
int main() {
    size_t B = (size_t)1600 << 20;
    void *h1, *h2, *d1, *d2;
    cudaMallocHost(&h1, B); cudaMallocHost(&h2, B); cudaMalloc(&d1, B); cudaMalloc(&d2, B);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    auto T = [&](auto fn) { cudaDeviceSynchronize(); auto t0 = std::chrono::steady_clock::now(); fn(); cudaDeviceSynchronize();
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
    for (int r = 0; r < 2; r++) {
        double a = T([&]{ cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1); });
        double b = T([&]{ cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2); });
        double c = T([&]{ cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1); cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2); });
        double d = T([&]{ void* p; cudaMallocAsync(&p, B * 2, s1); cudaFreeAsync(p, s1); cudaStreamSynchronize(s1); });
        printf("H2D %.1f ms (%.1f GB/s)  D2H %.1f ms (%.1f GB/s)  both %.1f ms  mallocAsync+free %.2f ms\n", a, B / a / 1e6, b, B / b / 1e6, c, d);
    }
    int v; cudaDeviceGetAttribute(&v, cudaDevAttrAsyncEngineCount, 0); printf("async engines %d\n", v);
}
