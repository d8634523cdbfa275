// Internal debug entry points (not part of include/tftb200.h): run one tile
// operation on device data so tools/ can test the tile engine in isolation.
#include "dispatch.cuh"

template <class F>
__global__ void k_dbg_itft_gen(LaunchArgs<F> a, typename F::W* data, int t, int wlog, uint32_t h) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    SmemTile<W> tl{S, t, wlog};
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) tl.at(g) = data[g];
    __syncthreads();
    itft_gen(a.f, tl, h, TwPrefix<F>{a.R.Zf}, TwPrefix<F>{a.R.Zi}, a.R);
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) data[g] = a.f.canon(tl.at(g));
}

template <class F>
__global__ void k_dbg_intt(LaunchArgs<F> a, typename F::W* data, int t) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    SmemTile<W> tl{S, t, 0};
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) tl.at(g) = data[g];
    __syncthreads();
    inv_all<F, false>(a.f, tl, TwPrefix<F>{a.R.Zi}, 1u << t, a.R.ipow2);
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) data[g] = a.f.canon(tl.at(g));
}

extern "C" int tftb_debug_intt_tile(uint64_t p, uint64_t top, int K, void* data, int t) {
    using namespace tftb;
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    LaunchArgs<F30> a{};
    a.f = make_field<F30>(p);
    a.R = rh->r32;
    size_t smem = padded_words(1u << t) * 4;
    if (set_smem(k_dbg_intt<F30>, smem)) return -1;
    k_dbg_intt<F30><<<1, 256, smem>>>(a, (uint32_t*)data, t);
    CK(cudaDeviceSynchronize());
    return 0;
}

extern "C" int tftb_debug_itft_tile(uint64_t p, uint64_t top, int K, void* data, int t, int wlog, uint32_t h) {
    using namespace tftb;
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    if (rh->kind != 0) return fail("debug: F30 only");
    LaunchArgs<F30> a{};
    a.f = make_field<F30>(p);
    a.R = rh->r32;
    size_t smem = padded_words(1u << (t + wlog)) * 4;
    if (set_smem(k_dbg_itft_gen<F30>, smem)) return -1;
    k_dbg_itft_gen<F30><<<1, 256, smem>>>(a, (uint32_t*)data, t, wlog, h);
    CK(cudaDeviceSynchronize());
    return 0;
}
