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

// Phase timestamps of the cluster forward on a uniform batch (count vectors of
// length n): out[cta*8 + k], k = 0 start, 1 loaded, 2 synced, 3 cross done,
// 4 synced, 5 rounds done, 6 stored.
extern "C" int tftb_debug_cluster_timing(uint64_t p, uint64_t top, int K, void* data, int64_t n, int64_t count,
                                         unsigned long long* out, int inverse) {
    using namespace tftb;
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    if (rh->kind != 0) return fail("debug: F30 only");
    Plan pl;
    if (make_plan<F30>(n, &pl) || pl.kind != kCluster) return fail("debug: n must use the cluster plan");
    LaunchArgs<F30> a{};
    a.f = make_field<F30>(p);
    a.R = rh->r32;
    a.x = (uint32_t*)data;
    a.in = a.x;
    a.xd = VecDesc<uint32_t>{nullptr, nullptr, n, n};
    a.ind = a.xd;
    a.timing = out;
    constexpr int CL = Limits<F30>::CL;
    const size_t smem = padded_words(1u << CL) * 4;
    if (set_smem(k_cl_fwd<F30, CL>, smem) || set_smem(k_cl_inv<F30, CL>, smem)) return -1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(pl.G, (unsigned)count, 1);
    lc.blockDim = dim3(256, 1, 1);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (inverse == 2) {  // the no-cluster forward the dispatcher uses
        const int gam = pl.l - CL;
        void (*kg)(LaunchArgs<F30>) = gam == 1 ? k_clg_fwd<F30, CL, 1>
                                     : gam == 2 ? k_clg_fwd<F30, CL, 2> : k_clg_fwd<F30, CL, 3>;
        if (set_smem(kg, smem)) return -1;
        kg<<<dim3(pl.G, (unsigned)count, 1), 256, smem>>>(a);
        CK(cudaGetLastError());
    } else if (inverse) {
        CK(cudaLaunchKernelEx(&lc, k_cl_inv<F30, CL>, a));
    } else {
        CK(cudaLaunchKernelEx(&lc, k_cl_fwd<F30, CL>, a));
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
