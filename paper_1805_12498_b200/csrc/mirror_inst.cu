// mirror_inst.cu -- instantiates the bit-exact MIRROR kernel for one size S (-DHAFB_S=S).
#include <algorithm>

#include "fast_launch.h"
#include "term_mirror.cuh"

#ifndef HAFB_S
#error "compile with -DHAFB_S=<even size>"
#endif

namespace hafb {

template <int S, bool L>
static cudaError_t launch_one(const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                              cd* terms, int8_t* status, cudaStream_t st, int sms) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int TPB = mirror_tpb<S>();
    constexpr int THREADS = TPB * W;
    const size_t smem = (size_t)TPB * MirrorLayout<S>::TOTAL * sizeof(cd);
    auto kern = mirror_term_kernel<S, L>;
    int occ = 1;
    #ifndef HAFB_MIRROR_CARVEOUT
#define HAFB_MIRROR_CARVEOUT 100
#endif
    cudaError_t e = launch_config((const void*)kern, THREADS, smem, (int)smem, &occ, HAFB_MIRROR_CARVEOUT);
    if (e != cudaSuccess) return e;
    const long long want = (ci.n_items + TPB - 1) / TPB;
    const long long cap_blocks = (long long)sms * std::max(occ, 1);
    const int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, THREADS, smem, st>>>(at, dg, n_half, ci, terms, status);
    return cudaGetLastError();
}

template <>
cudaError_t launch_mirror_S<HAFB_S>(bool loops, const cd* at, const cd* dg, int n_half,
                                    const ClassItems& ci, cd* terms, int8_t* status,
                                    cudaStream_t st, int sms) {
    return loops ? launch_one<HAFB_S, true>(at, dg, n_half, ci, terms, status, st, sms)
                 : launch_one<HAFB_S, false>(at, dg, n_half, ci, terms, status, st, sms);
}

}  // namespace hafb
