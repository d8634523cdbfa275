// Round throughput vs shared-memory row padding: P = 1 word per 32 (scalar
// accesses everywhere) against P = 4 words (16 B; the SLO = 0 round moves
// its 32-word units with 128-bit LDS/STS).  F30, 2^14-word tile, rounds
// (5 @ 9), (4 @ 5), (5 @ 0) repeated.
#include <cstdio>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/cluster.cuh"

// twiddle provider whose indices stay inside a 64-entry (L1-resident) window:
// same instruction stream, no L2 traffic (numerically meaningless)
struct TwSmall {
    const Tw<uint32_t>* Z;
    TFT_DEV Tw<uint32_t> get(int, uint32_t J) const { return ldg_tw(Z + (J & 63)); }
    template <int N>
    TFT_DEV void get_many(int, uint32_t J0, Tw<uint32_t>* out) const {
        ldg_tw_run<uint32_t, N>(Z + (J0 & 63 & ~(N - 1)), out);
    }
};

struct TwBcast {  // every thread reads the same twiddles (broadcast)
    const Tw<uint32_t>* Z;
    TFT_DEV Tw<uint32_t> get(int, uint32_t J) const { return ldg_tw(Z); }
    template <int N>
    TFT_DEV void get_many(int s, uint32_t, Tw<uint32_t>* out) const { ldg_tw_run<uint32_t, N>(Z + 32 * s, out); }
};

// single-word Montgomery twiddles: the table holds w R mod p (4 B); the
// companion w R p^-1 mod 2^32 is one IMAD; b w = hi(b wR) - hi((b wRp) p) + p
struct F30M : F30 {
    TFT_DEV W mulw(W b, Tw<W> t) const { return __umulhi(b, t.w) - __umulhi(b * t.wp, p) + p; }
    TFT_DEV void fwd(W& x, W& y, Tw<W> t) const {
        W a = red2(x);
        W b = mulw(y, t);
        x = a + b;
        y = a - b + p2;
    }
};
struct TwWord {
    const uint32_t* Zm;
    uint32_t pinv;
    TFT_DEV Tw<uint32_t> get(int, uint32_t J) const { const uint32_t w = __ldg(Zm + J); return Tw<uint32_t>{w, w * pinv}; }
    template <int N>
    TFT_DEV void get_many(int, uint32_t J0, Tw<uint32_t>* out) const {
        if constexpr (N >= 4) {
#pragma unroll
            for (int q = 0; q < N; q += 4) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(Zm + J0 + q));
                out[q] = Tw<uint32_t>{v.x, v.x * pinv}; out[q + 1] = Tw<uint32_t>{v.y, v.y * pinv};
                out[q + 2] = Tw<uint32_t>{v.z, v.z * pinv}; out[q + 3] = Tw<uint32_t>{v.w, v.w * pinv};
            }
        } else {
#pragma unroll
            for (int q = 0; q < N; ++q) out[q] = get(0, J0 + q);
        }
    }
};

template <int P, int KK, int SLO, class TP, class FF = F30>
__device__ __forceinline__ void round_p(const FF& f, uint32_t* S, const TP& tp) {
    constexpr uint32_t NU = 1u << (14 - KK);
    constexpr uint32_t STEP = SLO >= 5 ? (1u << SLO) + (P << (SLO - 5)) : 1u;
    for (uint32_t g = threadIdx.x; g < NU; g += blockDim.x) {
        const uint32_t base = (g & ((1u << SLO) - 1)) | ((g >> SLO) << (SLO + KK));
        uint32_t* pb = S + base + (base >> 5) * P;
        uint32_t v[1 << KK];
        if constexpr (SLO == 0 && KK == 5 && P == 4) {
            const uint4* pv = reinterpret_cast<const uint4*>(pb);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 t = pv[q];
                v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i) v[i] = pb[i * STEP];
        }
        reg_fwd<FF, KK, KK - 1>(f, v, base, SLO, tp);
        if constexpr (SLO == 0 && KK == 5 && P == 4) {
            uint4* pv = reinterpret_cast<uint4*>(pb);
#pragma unroll
            for (int q = 0; q < 8; ++q) pv[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
            for (int i = 0; i < (1 << KK); ++i) pb[i * STEP] = v[i];
        }
    }
}

template <int P, int SMALL>
__global__ void __launch_bounds__(256, 3) kround(F30 f, const Tw<uint32_t>* Z, uint32_t* out, int reps,
                                                 const uint32_t* Zm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* S = reinterpret_cast<uint32_t*>(smem_raw);
    for (uint32_t i = threadIdx.x; i < 16384; i += blockDim.x) S[i + (i >> 5) * P] = i * 2654435761u % f.p;
    __syncthreads();
    const TwDirect<F30> tp{Z, blockIdx.x & 3, 14, f};
    for (int r = 0; r < reps; ++r) {
        round_p<P, 5, 9>(f, S, tp);
        __syncthreads();
        round_p<P, 4, 5>(f, S, tp);
        __syncthreads();
        if constexpr (SMALL == 3) {
            F30M fm;
            static_cast<F30&>(fm) = f;
            round_p<P, 5, 0, TwWord, F30M>(fm, S, TwWord{Zm, f.pinv});
        } else if constexpr (SMALL == 2) round_p<P, 5, 0>(f, S, TwBcast{Z});
        else if constexpr (SMALL == 1) round_p<P, 5, 0>(f, S, TwSmall{Z});
        else round_p<P, 5, 0>(f, S, tp);
        __syncthreads();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = S[threadIdx.x];
}

template <int P, int SMALL>
void run(F30 f, Tw<uint32_t>* Z, uint32_t* out, size_t smem_force = 0, const uint32_t* Zm = nullptr) {
    size_t smem = smem_force ? smem_force : (16384 + 512 * P + P) * 4;
    printf("smem %zu: ", smem);
    cudaFuncSetAttribute(kround<P, SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int reps = 40, grid = 148 * 3 * 4;
    for (int k = 0; k < 3; ++k) {
        cudaEventRecord(a);
        kround<P, SMALL><<<grid, 256, smem>>>(f, Z, out, reps, Zm);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bf = (double)grid * reps * 14 * 8192;
        if (k) printf("small=%d P=%d: %.3f ms, %.2f butterflies/clk/SM @1.965GHz (%s)\n", (int)SMALL, P, ms, bf / (ms * 1e-3) / 148 / 1.965e9,
                      cudaGetErrorString(cudaGetLastError()));
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
    uint32_t* out; cudaMalloc(&out, 148 * 3 * 4 * 256 * 4);
    run<1, 0>(f, Z, out);
    run<1, 1>(f, Z, out);
    run<1, 2>(f, Z, out);
    std::vector<uint32_t> hm(1 << 16);
    for (size_t j = 0; j < hm.size(); ++j) hm[j] = (uint32_t)(((unsigned __int128)h[j].w << 32) % p);
    uint32_t* Zm; cudaMalloc(&Zm, hm.size() * 4); cudaMemcpy(Zm, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice);
    run<1, 3>(f, Z, out, 0, Zm);
}
