// Whole-vector tiles: n <= 2^CL, ceil_lg(n) = T known at compile time.
//
// A vector is the first n outputs of its zero-padded 2^T-point network
// (reference transforms.py:50-63 walks the same tree), so one tile in shared
// memory holds all of it: one HBM read and one HBM write per word.  The
// rounds are the compile-time register rounds of cluster.cuh (<= 5 stages
// per shared-memory pass, conflict-free padded layout); the forward prunes
// units whose outputs are all >= n, the inverse runs the masked in-tile
// solve (complete binary blocks of [0, n), then phases 2/3 of tile.cuh).
//
// Tiles smaller than 2^13 words share a CTA: 2^(T-5) threads per tile (one
// 32-word unit each in a 5-stage round), 256 / that many tiles per CTA, so
// every thread is busy whatever T is.  Barriers stay CTA-wide; tiles of one
// CTA have the same T and walk the same rounds.
#pragma once
#include "cluster.cuh"

template <int T>
struct TileShape {
    static constexpr int NTV = T >= 13 ? 256 : (T >= 5 ? (1 << (T - 5)) : 1);  // threads per tile
    static constexpr int VPB = 256 / NTV;                                     // tiles per CTA
    static constexpr uint32_t WORDS = (1u << T) + ((1u << T) >> 5) + 1;        // padded_words(2^T)
    static constexpr size_t smem(size_t wbytes) { return (size_t)VPB * WORDS * wbytes; }
};

template <class F, int T>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_tile_fwd(LaunchArgs<F> a, int64_t vend) {
    using W = typename F::W;
    using SH = TileShape<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t slot = threadIdx.x / SH::NTV;
    const Lanes ln{threadIdx.x % SH::NTV, (uint32_t)SH::NTV};
    W* S = reinterpret_cast<W*>(smem_raw) + slot * SH::WORDS;
    const int64_t v = a.vbase + (int64_t)blockIdx.x * SH::VPB + slot;
    const bool live = v < vend;
    const F f = a.f;
    int64_t n = 0;
    W* x = nullptr;
    if (live) {
        n = a.xd.n(v);
        x = a.x + a.xd.o(v);
        tile_load<W>(S, a.in + a.ind.o(v), a.ind.n(v), 1u << T, [](uint32_t, W w) { return w; }, ln);
    }
    __syncthreads();
    if constexpr (T > 0) fwd_rounds_ct<F, T, T, 0, true>(f, S, TwDirect<F>{a.R.Zf, 0, T, f, a.R.ZfM}, (uint32_t)n, ln);
    if (live) tile_store<W>(x, S, (uint32_t)n, [&](W w) { return f.canon(w); }, ln);
}

template <class F, int T>
__global__ void __launch_bounds__(256, kern_minb<F>()) k_tile_inv(LaunchArgs<F> a, int64_t vend) {
    using W = typename F::W;
    using SH = TileShape<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t slot = threadIdx.x / SH::NTV;
    const Lanes ln{threadIdx.x % SH::NTV, (uint32_t)SH::NTV};
    W* S = reinterpret_cast<W*>(smem_raw) + slot * SH::WORDS;
    const int64_t v = a.vbase + (int64_t)blockIdx.x * SH::VPB + slot;
    const bool live = v < vend;
    const F f = a.f;
    int64_t n = 0, o = 0;
    if (live) {
        n = a.xd.n(v);
        o = a.xd.o(v);
        if (a.pre)
            tile_load_pre<F>(a, S, a.x + o, a.pre + o, n, 1u << T, ln);
        else
            tile_load<W>(S, a.x + o, n, 1u << T, [](uint32_t, W w) { return w; }, ln);
    }
    __syncthreads();
    // phase 1 (n = 2^T: the plain scaled inverse), then phases 2/3
    const uint32_t h = (uint32_t)n;
    const TwDirect<F> tpi{a.R.Zi, 0, T, f, a.R.ZiM};
    if constexpr (T > 0) {  // (a 1-point transform is the identity)
        inv_rounds_ct<F, T, T, true>(f, S, tpi, a.R.ipow2, h, ln);
        itft_phases23<0>(f, SmemTile<W>{S, T, 0}, h, TwDirect<F>{a.R.Zf, 0, T, f}, tpi, a.R, ln, SH::VPB > 1, true);
    }
    if (live) tile_store<W>(a.x + o, S, h, [&](W w) { return f.canon(w); }, ln);
}
