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

// Batched over `batch` problems whose terms are `per` apart.
// Kahan per chunk over masks [lo + r*width, min(lo + (r+1)*width, hi)); terms are
// indexed by mask - lo.  Mask 0 is skipped.  fails[r] keeps the reference's
// "last nonzero status in the range" semantics.
__global__ void __launch_bounds__(128) range_kahan_kernel(const cd* __restrict__ terms,
                                                          const int8_t* __restrict__ status,
                                                          uint64_t lo, uint64_t hi, uint64_t width,
                                                          int n_chunks, int batch, long long per,
                                                          cd* __restrict__ partials,
                                                          long long* __restrict__ fails) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_chunks * batch) return;
    int bq = g / n_chunks, r = g - bq * n_chunks;
    terms += (size_t)bq * per;
    status += (size_t)bq * per;
    uint64_t a = lo + (uint64_t)r * width, b = a + width;
    if (a > hi) a = hi;
    if (b > hi) b = hi;
    double sre = 0.0, sim = 0.0, cre = 0.0, cim = 0.0;
    long long fail = 0;
    for (uint64_t mask = a; mask < b; ++mask) {
        if (mask == 0) continue;
        uint64_t q = mask - lo;
        cd t = terms[q];
        int st = status[q];
        if (st != 0) fail = st;
        double yre = __dsub_rn(t.re, cre), yim = __dsub_rn(t.im, cim);
        double tre = __dadd_rn(sre, yre), tim = __dadd_rn(sim, yim);
        cre = __dsub_rn(__dsub_rn(tre, sre), yre);
        cim = __dsub_rn(__dsub_rn(tim, sim), yim);
        sre = tre;
        sim = tim;
    }
    partials[g] = mk(sre, sim);
    fails[g] = fail;
}

// _numba.py:387-412 sum_subsets_fast: worker w runs ONE Kahan chain over the masks of
// ranges w, w+W, w+2W, ... in order (ranges [1 + r*width, ...) as in sum_subsets_det).
__global__ void worker_kahan_kernel(const cd* __restrict__ terms, const int8_t* __restrict__ status,
                                    uint64_t total, uint64_t width, int n_ranges, int workers,
                                    cd* __restrict__ wsums, long long* __restrict__ wfails) {
    int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= workers) return;
    double sre = 0.0, sim = 0.0, cre = 0.0, cim = 0.0;
    long long fail = 0;
    for (int r = w; r < n_ranges; r += workers) {
        uint64_t a = 1 + (uint64_t)r * width, b = a + width;
        if (b > total) b = total;
        for (uint64_t mask = a; mask < b; ++mask) {
            uint64_t q = mask - 1;
            cd t = terms[q];
            int st = status[q];
            if (st != 0) fail = st;
            double yre = __dsub_rn(t.re, cre), yim = __dsub_rn(t.im, cim);
            double tre = __dadd_rn(sre, yre), tim = __dadd_rn(sim, yim);
            cre = __dsub_rn(__dsub_rn(tre, sre), yre);
            cim = __dsub_rn(__dsub_rn(tim, sim), yim);
            sre = tre;
            sim = tim;
        }
    }
    wsums[w] = mk(sre, sim);
    wfails[w] = fail;
}

// Range-list mode: partial p sums terms [p*width, (p+1)*width) of the buffer, whose
// masks are 1 + ranges[p]*width + offset; masks >= total are padding.
__global__ void list_kahan_kernel(const cd* __restrict__ terms, const int8_t* __restrict__ status,
                                  const int32_t* __restrict__ ranges, int count, uint64_t width,
                                  uint64_t total, cd* __restrict__ partials,
                                  long long* __restrict__ fails) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    uint64_t first = 1 + (uint64_t)ranges[p] * width;
    double sre = 0.0, sim = 0.0, cre = 0.0, cim = 0.0;
    long long fail = 0;
    for (uint64_t off = 0; off < width && first + off < total; ++off) {
        uint64_t q = (uint64_t)p * width + off;
        cd t = terms[q];
        int st = status[q];
        if (st != 0) fail = st;
        double yre = __dsub_rn(t.re, cre), yim = __dsub_rn(t.im, cim);
        double tre = __dadd_rn(sre, yre), tim = __dadd_rn(sim, yim);
        cre = __dsub_rn(__dsub_rn(tre, sre), yre);
        cim = __dsub_rn(__dsub_rn(tim, sim), yim);
        sre = tre;
        sim = tim;
    }
    partials[p] = mk(sre, sim);
    fails[p] = fail;
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
