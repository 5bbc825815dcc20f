// fast_launch.h -- host launchers of the register kernels, one translation unit
// per size S (fast_inst.cu compiled with -DHAFB_S=S) so they build in parallel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cplx.cuh"
#include "enumerate.cuh"

namespace hafb {

constexpr int kFastSMax = 48;  // sizes above run in the shared-memory kernel

// launch fast_term_kernel<S, loops> over the items of one popcount class
template <int S>
cudaError_t launch_fast_S(bool loops, const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                          cd* terms, int8_t* status, cudaStream_t st, int sms);

// launch mirror_term_kernel<S, loops> (bit-exact charpoly backend), S = 2..62
template <int S>
cudaError_t launch_mirror_S(bool loops, const cd* at, const cd* dg, int n_half,
                            const ClassItems& ci, cd* terms, int8_t* status, cudaStream_t st,
                            int sms);

// launch modp_term_kernel<S, loops> (exact GF(p) terms, summed into *total), S = 2..62
template <int S>
cudaError_t launch_modp_S(bool loops, const uint32_t* at, const uint32_t* dg, int n_half,
                          const ClassItems& ci, uint32_t p, const uint32_t* inv,
                          unsigned long long* total, cudaStream_t st, int sms);

}  // namespace hafb
