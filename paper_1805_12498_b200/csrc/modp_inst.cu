// modp_inst.cu -- instantiates the exact GF(p) term kernel for one size S (-DHAFB_S=S).
#include <algorithm>

#include "fast_launch.h"
#include "term_modp.cuh"

#ifndef HAFB_S
#error "compile with -DHAFB_S=<even size>"
#endif

namespace hafb {

template <int S, bool L>
static cudaError_t launch_one(const uint32_t* at, const uint32_t* dg, int n_half, const ClassItems& ci,
                              uint32_t p, const uint32_t* tab, unsigned long long* total,
                              cudaStream_t st, int sms) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int TPB = kModpThreads / W;
    const size_t smem = (size_t)TPB * ModpLayout<S>::TOTAL * sizeof(uint32_t);
    auto kern = modp_term_kernel<S, L>;
    int occ = 1;
    cudaError_t e = launch_config((const void*)kern, kModpThreads, smem, (int)smem, &occ);
    if (e != cudaSuccess) return e;
    ModP M = make_modp(p);
    const long long want = (ci.n_items + TPB - 1) / TPB;
    const long long cap_blocks = (long long)sms * std::max(occ, 1);
    const int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, kModpThreads, smem, st>>>(at, dg, n_half, ci, M, tab, total);
    return cudaGetLastError();
}

template <>
cudaError_t launch_modp_S<HAFB_S>(bool loops, const uint32_t* at, const uint32_t* dg, int n_half,
                                  const ClassItems& ci, uint32_t p, const uint32_t* tab,
                                  unsigned long long* total, cudaStream_t st, int sms) {
    return loops ? launch_one<HAFB_S, true>(at, dg, n_half, ci, p, tab, total, st, sms)
                 : launch_one<HAFB_S, false>(at, dg, n_half, ci, p, tab, total, st, sms);
}

}  // namespace hafb
