// Internal debug entry points (not part of include/tftb200.h): run one tile
// operation on device data so tools/ can test the tile engine in isolation.
#include "dispatch.cuh"

// the production unmasked, scaled in-tile inverse (compile-time rounds of
// cluster.cuh, untwisted twiddles) on one 2^T tile
template <class F, int T>
__global__ void k_dbg_intt(LaunchArgs<F> a, typename F::W* data) {
    using W = typename F::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* S = reinterpret_cast<W*>(smem_raw);
    for (uint32_t g = threadIdx.x; g < (1u << T); g += blockDim.x) S[g + (g >> 5)] = data[g];
    __syncthreads();
    inv_rounds_ct<F, T, T, false>(a.f, S, TwDirect<F>{a.R.Zi, 0, T, a.f, a.R.ZiM}, a.R.ipow2);
    for (uint32_t g = threadIdx.x; g < (1u << T); g += blockDim.x) data[g] = a.f.canon(S[g + (g >> 5)]);
}

template <int T>
int dbg_intt(const tftb::RingHost* rh, LaunchArgs<F30> a, void* data) {
    using namespace tftb;
    const size_t smem = padded_words(1u << T) * 4;
    if (set_smem(k_dbg_intt<F30, T>, smem)) return -1;
    k_dbg_intt<F30, T><<<1, 256, smem>>>(a, (uint32_t*)data);
    CK(cudaDeviceSynchronize());
    return 0;
}

extern "C" int tftb_debug_intt_tile(uint64_t p, uint64_t top, int K, void* data, int t) {
    using namespace tftb;
    RingHost* rh;
    if (get_ring(p, top, K, &rh)) return -1;
    if (rh->kind != 0) return fail("debug: F30 only");
    LaunchArgs<F30> a{};
    a.f = make_field<F30>(p);
    a.R = rh->r32;
    switch (t) {
#define TFTB_DBG(T) \
    case T:         \
        return dbg_intt<T>(rh, a, data);
        TFTB_DBG(1) TFTB_DBG(2) TFTB_DBG(3) TFTB_DBG(4) TFTB_DBG(5) TFTB_DBG(6) TFTB_DBG(7)
        TFTB_DBG(8) TFTB_DBG(9) TFTB_DBG(10) TFTB_DBG(11) TFTB_DBG(12) TFTB_DBG(13) TFTB_DBG(14)
#undef TFTB_DBG
        default: return fail("debug: tile log out of range");
    }
}

// Phase timestamps of the forward cluster-range kernel on a uniform batch
// (count vectors of length n): out[cta*8 + k] from its TFTB_STAMP points.
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
    if (inverse) {  // the fused split inverse: chunk phases, and the last CTA's column work
        if (set_smem(k_cli_chunks<F30, CL>, smem)) return -1;
        Scratch tickets;
        if (tickets.get((size_t)count * 4, nullptr)) return -1;
        CK(cudaMemset(tickets.p, 0, (size_t)count * 4));
        a.done = (unsigned*)tickets.p;
        k_cli_chunks<F30, CL><<<dim3(pl.G, (unsigned)count), 256, smem>>>(a);
        CK(cudaDeviceSynchronize());
        return 0;
    }
    const int gam = pl.l - CL;
    void (*kg)(LaunchArgs<F30>) = gam == 1 ? k_clg_fwd<F30, CL, 1, 2, true>
                                 : gam == 2 ? (pl.G == 3 ? k_clg_fwd<F30, CL, 2, 3, true> : k_clg_fwd<F30, CL, 2, 4, true>)
                                            : k_clg_fwd<F30, CL, 3, 8, true>;
    if (set_smem(kg, smem)) return -1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(pl.G, (unsigned)count, 1);
    lc.blockDim = dim3(256, 1, 1);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    at[1].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
    lc.attrs = at;
    lc.numAttrs = 2;
    CK(cudaLaunchKernelEx(&lc, kg, a));
    CK(cudaDeviceSynchronize());
    return 0;
}

// Device buffer (16 x u64) that receives the phase stamps of the large
// inverse's single-CTA tail kernels (k_col1_inv 0..5, k_last_inv 8..11) on
// later executions; null switches them off.
extern "C" int tftb_debug_tail_timing(unsigned long long* out) {
    tftb::g_tail_timing = out;
    return 0;
}
