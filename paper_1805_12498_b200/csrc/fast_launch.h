// fast_launch.h -- host launchers of the register kernels, one translation unit
// per size S (fast_inst.cu compiled with -DHAFB_S=S) so they build in parallel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <utility>
#include <vector>

#include "cplx.cuh"
#include "enumerate.cuh"

namespace hafb {

// Per-(kernel, device, block size, smem) launch configuration, computed once: the max
// dynamic shared memory attribute (set to `smem_attr`, a size-independent value, so
// concurrent host threads never race on it) and the occupancy.  The two runtime
// queries cost tens of microseconds per launch, which dominated small problems (a
// hafnian of n = 20 is ~12 launches of a few microseconds each).
// carveout >= 0: the kernel's preferred shared-memory carveout (percent of the unified
// L1/shared array); the small-block shared-memory kernels ask for the maximum, else the
// driver may pick a smaller shared-memory configuration and cap their teams per SM
inline cudaError_t launch_config(const void* kern, int threads, size_t smem, int smem_attr,
                                 int* occ, int carveout = -1) {
    struct Entry {
        const void* k;
        int dev, threads;
        size_t smem;
        int occ;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> g(mu);
        for (const Entry& x : cache)
            if (x.k == kern && x.dev == dev && x.threads == threads && x.smem == smem) {
                *occ = x.occ;
                return cudaSuccess;
            }
    }
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_attr);
    if (e != cudaSuccess) return e;
    if (carveout >= 0) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        if (e != cudaSuccess) return e;
    }
    int o = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    cache.push_back(Entry{kern, dev, threads, smem, o});
    *occ = o;
    return cudaSuccess;
}

// Device attributes, cached per device.
inline int device_attr(cudaDeviceAttr a) {
    static std::mutex mu;
    static std::vector<std::pair<long long, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const long long key = (long long)dev * 1000 + (long long)a;
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto& x : cache)
            if (x.first == key) return x.second;
    }
    int v = 0;
    cudaDeviceGetAttribute(&v, a, dev);
    std::lock_guard<std::mutex> g(mu);
    cache.emplace_back(key, v);
    return v;
}

constexpr int kFastSMax = 48;  // sizes above run in the shared-memory kernel

// launch fast_term_kernel<S, loops> over the items of one popcount class; spectral: the
// FAST spectral backend (QR on the Hessenberg form, sweeps capped at cap * S) --
// fast_spectral_ok(S, loops) says where it exists
template <int S>
cudaError_t launch_fast_S(bool loops, const cd* at, const cd* dg, int n_half, const ClassItems& ci,
                          cd* terms, int8_t* status, cudaStream_t st, int sms, bool spectral = false,
                          int cap = 0);

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
