// fast_inst.cu -- instantiates the register kernel for one size S (-DHAFB_S=S).
#include <algorithm>

#include "fast_launch.h"
#include "term_fast.cuh"

#ifndef HAFB_S
#error "compile with -DHAFB_S=<even size>"
#endif

namespace hafb {

// Hessenberg variant per size (measured on B200, tools/micro/phase.cu): the
// shared-memory reduction wins for 18 <= S <= 26 and S >= 34, the register-window
// reduction elsewhere.
constexpr bool smem_hess(int S) { return (S >= 18 && S <= 26) || S >= 34; }

template <int S, bool L>
static cudaError_t launch_one(const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                              cd* terms, int8_t* status, cudaStream_t st, int sms) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int TPB = kFastThreads / W;
    constexpr bool SH = smem_hess(S);
    const size_t smem = (size_t)TPB * FastLayout<S, SH, L>::TOTAL * sizeof(cd) + (kDMax + 1) * sizeof(double);
    auto kern = fast_term_kernel<S, L, SH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFastThreads, smem);
    if (e != cudaSuccess) return e;
    const long long want = (ci.n_items + TPB - 1) / TPB;
    const long long cap_blocks = (long long)sms * std::max(occ, 1);
    const int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, kFastThreads, smem, st>>>(at, dg, n_half, ci, terms, status);
    return cudaGetLastError();
}

template <>
cudaError_t launch_fast_S<HAFB_S>(bool loops, const cd* at, const cd* dg, int n_half,
                                  const ClassItems& ci, cd* terms, int8_t* status, cudaStream_t st,
                                  int sms) {
    return loops ? launch_one<HAFB_S, true>(at, dg, n_half, ci, terms, status, st, sms)
                 : launch_one<HAFB_S, false>(at, dg, n_half, ci, terms, status, st, sms);
}

}  // namespace hafb
