// fast_inst.cu -- instantiates the register kernel for one size S (-DHAFB_S=S).
#include <algorithm>

#include "fast_launch.h"
#include "term_fast.cuh"

#ifndef HAFB_S
#error "compile with -DHAFB_S=<even size>"
#endif

namespace hafb {

// Hessenberg variant per size (measured on B200, tools/micro/phase.cu and
// tools/class_time.py under ncu):
//   18 <= S <= 32  static-column register reduction (ns_hessenberg, one warp per subset);
//   S = 34, 36     (no loops) one warp with the extra rows held column-wise (nsx_hessenberg);
//   S >= 34        shared-memory reduction over 64-lane teams (smem_hessenberg: a two-warp
//                  static-column team measured 7-11 % slower -- its second warp carries
//                  2..8 rows but issues the whole instruction stream);
//   10 <= S <= 16  the same static-column kernel on 16-lane teams (two subsets per warp);
//   S <= 8         register-window reduction (fast_hessenberg, 2..8-lane teams).
#ifndef HAFB_SMEM_HI
#define HAFB_SMEM_HI 34
#endif
constexpr bool smem_hess(int S) { return !ns_variant(S) && ((S >= 18 && S <= 24) || S >= HAFB_SMEM_HI); }
// the FAST spectral backend runs where the kernel keeps the packed Hessenberg form
constexpr bool fast_spectral_ok(int S, bool loops) {
    return (nsx_variant(S) && !loops) || !smem_hess(S);
}

// Threads per block.  The register classes run ONE block per SM whose teams are
// phase-synchronised (__syncthreads between the Hessenberg, charpoly and series phases):
// the SM's instruction cache then holds one phase's code at a time (this removed the
// "no instruction" stall, 34% of stall cycles at S = 30), and the block stages Atilde in
// shared memory for the gathers.  512 threads (16 teams, <= 128 registers) for S <= 22,
// 384 (12 teams, <= 168 registers) up to S = 32.  The shared-memory classes are L1-bound
// and gain nothing from phase sync (measured), so they keep small blocks.
#ifndef HAFB_NS_WIDE_THREADS
#define HAFB_NS_WIDE_THREADS 64
#endif
#ifndef HAFB_NS_SMALL_THREADS
#define HAFB_NS_SMALL_THREADS 512
#endif
#ifndef HAFB_REG_THREADS
#define HAFB_REG_THREADS 384
#endif
// Split rows (term_fast.cuh, ns_split_k): the no-loop static-column classes S = 24..28
// keep part of each row in shared memory and run 16 teams per SM.
#ifndef HAFB_SPLIT_HI
#define HAFB_SPLIT_HI 28
#endif
constexpr int threads_for(int S, bool loops) {
    return ns_variant(S) ? (S > 32 ? HAFB_NS_WIDE_THREADS : S <= 16 ? kFastThreads : S <= 22 ? HAFB_NS_SMALL_THREADS
                            : (!loops && S >= HAFB_NS_SPLIT_LO && S <= HAFB_SPLIT_HI) ? 512 : HAFB_REG_THREADS)
           : !smem_hess(S) && S >= 26 ? (S > 32 ? 256 : HAFB_REG_THREADS)
           : S > 32 ? 64  // 64-lane teams: one team per block (register-limited: 5 teams/SM, not 4)
           : smem_hess(S) ? 32  // one team per block: the register file packs one more team
           : kFastThreads;
}

#ifndef HAFB_NSX_THREADS
#define HAFB_NSX_THREADS 256
#endif

// NSX classes with split rows (term_fast.cuh, nsx_split_k): blocks of 11-12 teams at <= 168
// registers, tried from the largest down until the workspaces and the staged Atilde fit one
// SM's shared memory: S = 34 runs 12 teams up to n = 52 (167.7 -> 146.0 ms at n = 52) and 11
// up to n = 60 (-4 % at n = 56); S = 36 runs 11 teams up to n = 52 (-6 %; 10 teams measured
// 2 % slower than the unsplit kernel).  The unsplit 256-thread kernel (8 teams) is the last
// level and the FAST spectral configuration.
constexpr int nsx_threads(int S, bool spec, int level) {
    if (spec || S == 38 || nsx_split_k(S, 384) <= 2) return HAFB_NSX_THREADS;
    return level == 0 ? 384 : level == 1 ? 352 : HAFB_NSX_THREADS;
}

// (S = 30, 32 with the triangular staging fit 16 / 14 split-row teams; measured -0.8 % and
// +4.7 % against their 12 unsplit teams, so they stay at 384 threads.)
template <int S, bool L, bool SPEC = false, int LEVEL = 0>
static cudaError_t launch_one(const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                              cd* terms, int8_t* status, cudaStream_t st, int sms, int cap = 0) {
    // S = 34, 36 without loops: one-warp teams with the extra rows held column-wise
    constexpr bool NSX = nsx_variant(S) && !L;
    constexpr bool SH = smem_hess(S) && !NSX;
    constexpr int W = FastTeam<S, L, SH>::W;
    constexpr int NT = NSX ? nsx_threads(S, SPEC, LEVEL) : threads_for(S, L);
    constexpr int TPB = NT / W;
    const size_t base_smem = (size_t)TPB * FastLayout<S, SH, L>::TOTAL * sizeof(cd) + kInvSlots * sizeof(double);
    // the one-block-per-SM register classes stage Atilde in shared memory when it fits
    const int n = 2 * n_half;
    const size_t a_bytes = (size_t)n * (n + 1) * sizeof(cd);
    const int optin = device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin);
    // stage 1: the full Atilde (row stride n+1); stage 2 (one problem, no loops, S >= 30): the
    // lower triangle of the symmetric A it was built from -- half the bytes, verified by every
    // block while it stages (term_fast.cuh)
    const size_t tri_bytes = (size_t)n * (n + 1) / 2 * sizeof(cd);
    const bool tri_ok = !L && !SH && S >= 30 && ci.n_items == ci.per_problem;
    const int stage = !(NT > kFastThreads && !SH)                ? 0
                      : base_smem + a_bytes <= (size_t)optin      ? 1
                      : tri_ok && base_smem + tri_bytes <= (size_t)optin ? 2
                                                                         : 0;
    if constexpr (NSX && NT != HAFB_NSX_THREADS) {
        if (!stage) return launch_one<S, L, SPEC, LEVEL + 1>(at, dg, n_half, ci, terms, status, st, sms, cap);
    }
    const size_t smem = base_smem + (stage == 1 ? a_bytes : stage == 2 ? tri_bytes : 0);
    // 64-lane shared-memory classes that fill the GPU: the register-capped instantiation
    // (6 teams per SM instead of 5)
    void (*kern)(const cd*, const cd*, int, ClassItems, cd*, int8_t*, int, int) = fast_term_kernel<S, L, SH, NT, SPEC>;
    if constexpr (sh_capped_ok(S, SH, NT) && !SPEC) {
        if (ci.n_items >= 4LL * HAFB_SH_MINB * sms) kern = fast_term_kernel<S, L, SH, NT, SPEC, HAFB_SH_MINB>;
    }
    // smem depends on n (the staged Atilde): the attribute is the size-independent
    // opt-in maximum, so host threads launching different n never race on it
    int occ = 1;
    cudaError_t e = launch_config((const void*)kern, NT, smem, optin, &occ);
    if (e != cudaSuccess) return e;
    const long long want = (ci.n_items + TPB - 1) / TPB;
    const long long cap_blocks = (long long)sms * std::max(occ, 1);
    const int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, NT, smem, st>>>(at, dg, n_half, ci, terms, status, stage, cap);
    return cudaGetLastError();
}

template <>
cudaError_t launch_fast_S<HAFB_S>(bool loops, const cd* at, const cd* dg, int n_half,
                                  const ClassItems& ci, cd* terms, int8_t* status, cudaStream_t st,
                                  int sms, bool spectral, int cap) {
    if (spectral) {
        // the FAST spectral backend needs the packed Hessenberg form (not the 64-lane
        // shared-memory classes: the caller routes those to the bit-exact kernel)
        if constexpr (fast_spectral_ok(HAFB_S, true)) {
            if (loops) return launch_one<HAFB_S, true, true>(at, dg, n_half, ci, terms, status, st, sms, cap);
        }
        if constexpr (fast_spectral_ok(HAFB_S, false)) {
            if (!loops) return launch_one<HAFB_S, false, true>(at, dg, n_half, ci, terms, status, st, sms, cap);
        }
        return cudaErrorNotSupported;  // the caller runs the bit-exact spectral kernel
    }
    return loops ? launch_one<HAFB_S, true>(at, dg, n_half, ci, terms, status, st, sms)
                 : launch_one<HAFB_S, false>(at, dg, n_half, ci, terms, status, st, sms);
}

}  // namespace hafb
