// fast_inst.cu -- instantiates the register kernel for one size S (-DHAFB_S=S).
#include <algorithm>

#include "fast_launch.h"
#include "term_fast.cuh"

#ifndef HAFB_S
#error "compile with -DHAFB_S=<even size>"
#endif

namespace hafb {

// Hessenberg variant per size (measured on B200, tools/class_time.py under ncu): the
// shared-memory reduction wins for 18 <= S <= 24 and S >= 34 (these classes are
// shared-memory-bandwidth bound), the register-window reduction elsewhere.
#ifndef HAFB_SMEM_HI
#define HAFB_SMEM_HI 34
#endif
constexpr bool smem_hess(int S) { return !x2_variant(S) && ((S >= 18 && S <= 24) || S >= HAFB_SMEM_HI); }

// Threads per block.  The register-window kernel for 26 <= S <= 32 runs ONE block of
// 384 threads per SM whose teams are phase-synchronised (__syncthreads between the
// Hessenberg, charpoly and series phases): the SM's instruction cache then holds one
// phase's code at a time, which removed the top stall ("no instruction", 34% of
// stall cycles at S = 30) and cut these classes by ~20%.  The shared-memory classes
// are L1-bound and gain nothing from it (measured), so they keep 128-thread blocks.
#ifndef HAFB_REG_THREADS
#define HAFB_REG_THREADS 384
#endif
constexpr int threads_for(int S) {
    return !smem_hess(S) && (S >= 26 || x2_variant(S)) ? (S > 32 ? 256 : HAFB_REG_THREADS)
           : S > 32 ? 64  // 64-lane teams: one team per block (register-limited: 5 teams/SM, not 4)
           : smem_hess(S) ? 32  // one team per block: the register file packs one more team
           : kFastThreads;
}

template <int S, bool L>
static cudaError_t launch_one(const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                              cd* terms, int8_t* status, cudaStream_t st, int sms) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int NT = threads_for(S);
    constexpr int TPB = NT / W;
    constexpr bool SH = smem_hess(S);
    const size_t base_smem = (size_t)TPB * FastLayout<S, SH, L, !SH && x2_variant(S)>::TOTAL * sizeof(cd) + (kDMax + 1) * sizeof(double);
    // the one-block-per-SM register classes stage Atilde in shared memory when it fits
    const int n = 2 * n_half;
    const size_t a_bytes = (size_t)n * (n + 1) * sizeof(cd);
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int stage = (NT > kFastThreads && !SH && base_smem + a_bytes <= (size_t)optin) ? 1 : 0;
    const size_t smem = base_smem + (stage ? a_bytes : 0);
    auto kern = fast_term_kernel<S, L, SH, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    const long long want = (ci.n_items + TPB - 1) / TPB;
    const long long cap_blocks = (long long)sms * std::max(occ, 1);
    const int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, NT, smem, st>>>(at, dg, n_half, ci, terms, status, stage);
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
