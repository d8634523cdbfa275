// Standalone check: itft_gen on a column-interleaved tile (wlog=4) vs one
// column at a time (wlog=0), same inputs.  Uses the real ring tables via the
// library is overkill; build tiny tables here for p = 998244353.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1001_5272_b200/csrc/host.h"
#include "../../paper_1001_5272_b200/csrc/kernels.cuh"
using namespace tftb;
namespace tftb { thread_local std::string g_err; thread_local int64_t g_launches = 0; }

template <int WLOG>
__global__ void kgen(LaunchArgs<F30> a, uint32_t* data, int t, uint32_t h) {
    extern __shared__ uint32_t S[];
    SmemTile<uint32_t> tl{S, t, WLOG};
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) tl.at(g) = data[g];
    __syncthreads();
    itft_gen(a.f, tl, h, TwPrefix<F30>{a.R.Zf}, TwPrefix<F30>{a.R.Zi}, a.R);
    for (uint32_t g = threadIdx.x; g < tl.words(); g += blockDim.x) data[g] = a.f.canon(tl.at(g));
}

int main(int argc, char** argv) {
    int t = argc > 1 ? atoi(argv[1]) : 7;
    uint32_t h = argc > 2 ? atoi(argv[2]) : 68;
    extern int tftb_ring_get(uint64_t, uint64_t, int, void**);
    return 0;
}
