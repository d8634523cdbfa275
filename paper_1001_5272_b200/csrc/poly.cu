// Algorithm 3's helper operations of the reference's public polymul API, on
// the device: horner_eval (polymul.py:39-52, _kernels.pyx:401-412 horner_k)
// and fold_twist (polymul.py:55-88, _kernels.pyx:366-398 fold_twist_k).
// The product itself does not need them (it uses three transforms, DESIGN.md
// §3); they are here so the reference's polymul module surface runs on the
// GPU too.  Words are the reference's canonical uint64 residues for every
// ring (p < 2^62): 64-bit Montgomery products (field.cuh F62), values
// canonical at every store.
#include <cuda_runtime.h>

#include "../../include/tftb200.h"
#include "host.h"
#include "kernels.cuh"

namespace {

using tftb::fail;

struct Mont64 {
    F62 f;     // lazy 64-bit Montgomery (R = 2^64)
    uint64_t r2;  // R^2 mod p
    // canonical a * b mod p for canonical a, b
    TFT_DEV uint64_t mul(uint64_t a, uint64_t b) const { return f.red1(f.mont(f.red1(f.mont(a, b)), r2)); }
    TFT_DEV uint64_t add(uint64_t a, uint64_t b) const { return f.red1(a + b); }
    TFT_DEV uint64_t pow(uint64_t b, uint64_t e) const {
        uint64_t r = 1;
        while (e) {
            if (e & 1) r = mul(r, b);
            b = mul(b, b);
            e >>= 1;
        }
        return r;
    }
};

Mont64 make_mont(uint64_t p) {
    Mont64 m;
    m.f = tftb::make_field<F62>(p);
    const unsigned __int128 R = ((unsigned __int128)1 << 64) % p;
    m.r2 = (uint64_t)((R * R) % p);
    return m;
}

constexpr int kHT = 256;  // threads per block

// Block b, thread t owns the contiguous segment [s0, s1) of the coefficients:
// Horner over it (highest first), times x^s0, block-reduced into part[b].
__global__ void k_horner_part(Mont64 m, const uint64_t* __restrict__ poly, int64_t n, uint64_t x, int64_t seg,
                              uint64_t* part) {
    __shared__ uint64_t red[kHT];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t s0 = t * seg, s1 = min(n, s0 + seg);
    uint64_t acc = 0;
    if (s0 < s1) {
        for (int64_t i = s1 - 1; i >= s0; --i) acc = m.add(m.mul(acc, x), poly[i]);
        acc = m.mul(acc, m.pow(x, (uint64_t)s0));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = kHT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] = m.add(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum(Mont64 m, const uint64_t* part, int nb, uint64_t* out) {
    __shared__ uint64_t red[kHT];
    uint64_t acc = 0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc = m.add(acc, part[i]);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = kHT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] = m.add(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// Slot j < L of the block gains sum_k src[j + kL] w^(j + kL): one thread per
// slot, w^j by square-and-multiply, then steps of w^L.
__global__ void k_fold_twist(Mont64 m, const uint64_t* __restrict__ src, int64_t ls, uint64_t* X, int64_t L,
                             uint64_t w, uint64_t wL) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < L; j += (int64_t)gridDim.x * blockDim.x) {
        uint64_t pw = w ? m.pow(w, (uint64_t)j) : 1;
        uint64_t acc = X[j];
        for (int64_t i = j; i < ls; i += L) {
            acc = m.add(acc, w ? m.mul(src[i], pw) : src[i]);
            if (w) pw = m.mul(pw, wL);
        }
        X[j] = acc;
    }
}

struct Stream {
    cudaStream_t s = nullptr;
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
};

}  // namespace

using namespace tftb;

extern "C" {

int tftb_horner_u64(const uint64_t* poly, int64_t n, uint64_t point, uint64_t p, uint64_t* out) {
    if (n <= 0 || !poly || !out) return fail("cannot evaluate an empty polynomial");
    if (p < 3 || !(p & 1) || p >= (1ull << 62) || point >= p) return fail("bad modulus or point");
    Stream st;
    CK(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
    const Mont64 m = make_mont(p);
    // ~16 coefficients per thread at least, at most 8 blocks per SM
    const int64_t threads = std::max<int64_t>(1, std::min<int64_t>((n + 15) / 16, 148 * 8 * kHT));
    const int64_t seg = (n + threads - 1) / threads;
    const int nb = (int)((threads + kHT - 1) / kHT);
    Scratch buf;
    if (buf.get((size_t)(n + nb + 1) * 8, st.s)) return -1;
    uint64_t* dp = (uint64_t*)buf.p;
    uint64_t* part = dp + n;
    CK(cudaMemcpyAsync(dp, poly, (size_t)n * 8, cudaMemcpyHostToDevice, st.s));
    k_horner_part<<<nb, kHT, 0, st.s>>>(m, dp, n, point, seg, part);
    k_sum<<<1, kHT, 0, st.s>>>(m, part, nb, part + nb);
    g_launches += 2;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, part + nb, 8, cudaMemcpyDeviceToHost, st.s));
    CK(cudaStreamSynchronize(st.s));
    return 0;
}

int tftb_fold_twist_u64(const uint64_t* src, int64_t ls, uint64_t* X, int64_t L, uint64_t w, uint64_t p) {
    if (ls < 0 || L <= 0 || !X || (ls && !src)) return fail("bad fold_twist arguments");
    if (p < 3 || !(p & 1) || p >= (1ull << 62) || w >= p) return fail("bad modulus or twist");
    if (ls == 0) return 0;
    Stream st;
    CK(cudaStreamCreateWithFlags(&st.s, cudaStreamNonBlocking));
    const Mont64 m = make_mont(p);
    Scratch buf;
    if (buf.get((size_t)(ls + L) * 8, st.s)) return -1;
    uint64_t* ds = (uint64_t*)buf.p;
    uint64_t* dx = ds + ls;
    CK(cudaMemcpyAsync(ds, src, (size_t)ls * 8, cudaMemcpyHostToDevice, st.s));
    CK(cudaMemcpyAsync(dx, X, (size_t)L * 8, cudaMemcpyHostToDevice, st.s));
    // w^L on the host (one scalar)
    uint64_t wL = 1;
    if (w) wL = powmod(w, (uint64_t)L, p);
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((L + 255) / 256, 148 * 8));
    k_fold_twist<<<nb, 256, 0, st.s>>>(m, ds, ls, dx, L, w == 1 ? 0 : w, wL);
    g_launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(X, dx, (size_t)L * 8, cudaMemcpyDeviceToHost, st.s));
    CK(cudaStreamSynchronize(st.s));
    return 0;
}

}  // extern "C"
