// reduce.cuh -- the reference's reduction contract on the device.
//
// _numba.py:373-383: each fixed range of masks is Kahan-summed in mask order;
// engine.py:87-97: the range partials are combined by a fixed pairwise tree.
// Both are order-defined, so they are reproduced exactly: one thread walks one
// range sequentially (the only reduction order that is bit-identical to the
// reference), and the tree is the same pairwise tree.
#pragma once

#include "cplx.cuh"

namespace hafb {

// Sequential Kahan state (the reference's compensated sum, _numba.py:373-383).
struct Kahan {
    double sre = 0.0, sim = 0.0, cre = 0.0, cim = 0.0;
    long long fail = 0;
    __device__ __forceinline__ void add(cd t, int st) {
        if (st != 0) fail = st;
        double yre = __dsub_rn(t.re, cre), yim = __dsub_rn(t.im, cim);
        double tre = __dadd_rn(sre, yre), tim = __dadd_rn(sim, yim);
        cre = __dsub_rn(__dsub_rn(tre, sre), yre);
        cim = __dsub_rn(__dsub_rn(tim, sim), yim);
        sre = tre;
        sim = tim;
    }
};

// One WARP walks terms[q0 .. q0+count) in order for a Kahan chain held by lane 0:
// the warp loads chunks of kChunk terms with coalesced 16-byte loads (the next chunk's
// loads in flight while lane 0 runs the current one from shared memory).  The chain
// itself stays strictly sequential: the order, and so every bit, is the reference's.
constexpr int kKahanChunk = 128;
struct KahanStage {
    double2 v[kKahanChunk];
    int8_t s[kKahanChunk];
};

__device__ __forceinline__ void warp_kahan_run(const cd* __restrict__ terms,
                                               const int8_t* __restrict__ status, uint64_t q0,
                                               uint64_t count, Kahan& k, KahanStage& st) {
    constexpr int PER = kKahanChunk / 32;
    const int lane = threadIdx.x & 31;
    double2 v[PER];
    int8_t sv[PER];
    auto load = [&](uint64_t base) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint64_t idx = base + (uint64_t)(j * 32 + lane);
            if (idx < count) {
                v[j] = __ldg(reinterpret_cast<const double2*>(terms + q0 + idx));
                sv[j] = __ldg(reinterpret_cast<const signed char*>(status) + q0 + idx);
            } else {
                v[j] = make_double2(0.0, 0.0);
                sv[j] = 0;
            }
        }
    };
    if (count == 0) return;
    load(0);
    for (uint64_t base = 0; base < count; base += kKahanChunk) {
        __syncwarp();
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            st.v[j * 32 + lane] = v[j];
            st.s[j * 32 + lane] = sv[j];
        }
        __syncwarp();
        if (base + kKahanChunk < count) load(base + kKahanChunk);
        if (lane == 0) {
            const int n = (int)(count - base < (uint64_t)kKahanChunk ? count - base : kKahanChunk);
#pragma unroll 8
            for (int i = 0; i < n; ++i) k.add(mk(st.v[i].x, st.v[i].y), st.s[i]);
        }
    }
}

// FAST arithmetic: the same range sum with the chain split over the warp's lanes (lane l
// Kahan-sums terms l, l+32, ... with coalesced loads; the 32 compensated partials are
// combined by a fixed butterfly), so a range costs count/32 chain steps instead of
// count.  Deterministic for any rank count (a function of the range alone).  `fail`
// keeps the reference's semantics: the status of the last failing term in mask order.
__device__ __forceinline__ void warp_par_run(const cd* __restrict__ terms,
                                             const int8_t* __restrict__ status, uint64_t q0,
                                             uint64_t count, Kahan& k) {
    const int lane = threadIdx.x & 31;
    Kahan mine;
    long long last = -1;
    int last_st = 0;
    for (uint64_t i = lane; i < count; i += 32) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(terms + q0 + i));
        const int st = __ldg(reinterpret_cast<const signed char*>(status) + q0 + i);
        mine.add(mk(v.x, v.y), 0);
        if (st != 0) {
            last = (long long)i;
            last_st = st;
        }
    }
    double re = mine.sre - mine.cre, im = mine.sim - mine.cim;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, off);
        im += __shfl_xor_sync(0xffffffffu, im, off);
        const long long ol = __shfl_xor_sync(0xffffffffu, last, off);
        const int os = __shfl_xor_sync(0xffffffffu, last_st, off);
        if (ol > last) {
            last = ol;
            last_st = os;
        }
    }
    k.sre = re;
    k.sim = im;
    k.cre = k.cim = 0.0;
    k.fail = last_st;
}

// Batched over `batch` problems whose terms are `per` apart.
// Kahan per chunk over masks [lo + r*width, min(lo + (r+1)*width, hi)); terms are
// indexed by mask - lo.  Mask 0 is skipped.  fails[r] keeps the reference's
// "last nonzero status in the range" semantics.
template <bool PAR = false>
__global__ void __launch_bounds__(128) range_kahan_kernel(const cd* __restrict__ terms,
                                                          const int8_t* __restrict__ status,
                                                          uint64_t lo, uint64_t hi, uint64_t width,
                                                          int n_chunks, int batch, long long per,
                                                          cd* __restrict__ partials,
                                                          long long* __restrict__ fails) {
    __shared__ KahanStage stage[4];
    const int g = blockIdx.x * 4 + (threadIdx.x >> 5);  // one warp per chunk
    if (g >= n_chunks * batch) return;
    int bq = g / n_chunks, r = g - bq * n_chunks;
    terms += (size_t)bq * per;
    status += (size_t)bq * per;
    uint64_t a = lo + (uint64_t)r * width, b = a + width;
    if (a > hi) a = hi;
    if (b > hi) b = hi;
    if (a == 0 && b > 0) a = 1;  // mask 0 is skipped
    Kahan k;
    if (b > a) {
        if constexpr (PAR) warp_par_run(terms, status, a - lo, b - a, k);
        else warp_kahan_run(terms, status, a - lo, b - a, k, stage[threadIdx.x >> 5]);
    }
    if ((threadIdx.x & 31) == 0) {
        partials[g] = mk(k.sre, k.sim);
        fails[g] = k.fail;
    }
}

// _numba.py:387-412 sum_subsets_fast: worker w runs ONE Kahan chain over the masks of
// ranges w, w+W, w+2W, ... in order (ranges [1 + r*width, ...) as in sum_subsets_det).
__global__ void __launch_bounds__(128) worker_kahan_kernel(const cd* __restrict__ terms,
                                                           const int8_t* __restrict__ status,
                                                           uint64_t total, uint64_t width, int n_ranges,
                                                           int workers, cd* __restrict__ wsums,
                                                           long long* __restrict__ wfails) {
    __shared__ KahanStage stage[4];
    const int w = blockIdx.x * 4 + (threadIdx.x >> 5);  // one warp per worker
    if (w >= workers) return;
    Kahan k;
    for (int r = w; r < n_ranges; r += workers) {
        uint64_t a = 1 + (uint64_t)r * width, b = a + width;
        if (b > total) b = total;
        if (b > a) warp_kahan_run(terms, status, a - 1, b - a, k, stage[threadIdx.x >> 5]);
    }
    if ((threadIdx.x & 31) == 0) {
        wsums[w] = mk(k.sre, k.sim);
        wfails[w] = k.fail;
    }
}

// Range-list mode: partial p sums terms [p*width, (p+1)*width) of the buffer, whose
// masks are 1 + ranges[p]*width + offset; masks >= total are padding.
template <bool PAR = false>
__global__ void __launch_bounds__(128) list_kahan_kernel(const cd* __restrict__ terms,
                                                         const int8_t* __restrict__ status,
                                                         const int32_t* __restrict__ ranges, int count,
                                                         uint64_t width, uint64_t total,
                                                         cd* __restrict__ partials,
                                                         long long* __restrict__ fails) {
    __shared__ KahanStage stage[4];
    const int p = blockIdx.x * 4 + (threadIdx.x >> 5);  // one warp per listed range
    if (p >= count) return;
    uint64_t first = 1 + (uint64_t)ranges[p] * width;
    const uint64_t n = first >= total ? 0 : (total - first < width ? total - first : width);
    Kahan k;
    if constexpr (PAR) warp_par_run(terms, status, (uint64_t)p * width, n, k);
    else warp_kahan_run(terms, status, (uint64_t)p * width, n, k, stage[threadIdx.x >> 5]);
    if ((threadIdx.x & 31) == 0) {
        partials[p] = mk(k.sre, k.sim);
        fails[p] = k.fail;
    }
}

// engine.py:87-97 tree_reduce over `n` partials of each of `batch` problems
// (batched hafnians); one thread per problem, in-place on a scratch copy.
__global__ void tree_reduce_kernel(cd* __restrict__ vals, int n, int batch, cd* __restrict__ out) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    cd* v = vals + (size_t)b * n;
    int len = n;
    if (len <= 0) { out[b] = mk(0.0, 0.0); return; }
    while (len > 1) {
        int nn = 0;
        for (int i = 0; i + 1 < len; i += 2) v[nn++] = m_add(v[i], v[i + 1]);
        if (len & 1) v[nn++] = v[len - 1];
        len = nn;
    }
    out[b] = v[0];
}

}  // namespace hafb
