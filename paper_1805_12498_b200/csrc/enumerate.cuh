// enumerate.cuh -- size-class enumeration of pair subsets.
//
// The reference walks masks in numeric order (_numba.py:375); the cost of a
// mask grows like popcount^3, so a warp that mixes popcounts diverges and a
// fixed range split is unbalanced (SURVEY.md H2 / finding 5).  Here every
// kernel launch handles ONE popcount class m: item rho of the class maps to
// the rho-th mask of popcount m inside a list of mask segments, by colex
// unranking (combinatorial number system).  Terms are written to the buffer
// slot of their mask, so the order-defined reduction afterwards is unchanged.
#pragma once

#include <stdint.h>

namespace hafb {

struct Seg {
    unsigned long long lo, hi;  // masks [lo, hi)
    long long out_off;          // buffer index of mask x is out_off + (x - lo)
};

// Items of one popcount class over a segment list (and over `batch` problems).
struct ClassItems {
    unsigned long long c_top;           // C(D-1, m): the unranking's first binomial
    const Seg* segs;
    const long long* prefix;            // nseg+1: # class-m masks before segment s
    const unsigned long long* base;     // nseg: # class-m integers below segs[s].lo
    int nseg;
    int m;
    int D;
    long long per_problem;              // = prefix[nseg]
    long long n_items;                  // = batch * per_problem
    long long term_stride;              // buffer offset between problems
    long long at_stride, dg_stride;     // input offsets between problems (in cd)
    const uint32_t* mlist;              // explicit-mask mode: the class's masks ...
    const long long* mout;              // ... and their buffer indices (else null)
    Seg seg0;                           // nseg == 1: the segment and its base by value
    unsigned long long base0;           // (no dependent loads for the first item)
    unsigned long long* ctr = nullptr;  // zeroed work counter: dynamic chunks (FAST kernels)
};

// the r-th (0-based) integer with popcount m, bits below D (combinatorial number
// system).  The binomials are stepped arithmetically from c_top = C(D-1, m):
//   C(b-1, m) = C(b, m) (b - m) / b,   C(b-1, m-1) = C(b, m) m / b,
// exact in double (every value is an integer < 2^36 and the quotient is exact), so
// unranking issues no memory loads: a table lookup per bit is a chain of ~D dependent
// global-memory round trips, which made the first item of every launch cost ~15 us.
__device__ __forceinline__ uint32_t unrank_mask(unsigned long long r, int m, int D,
                                                unsigned long long c_top) {
    uint32_t mask = 0;
    double c = (double)c_top;  // C(b, m) for the current b
    for (int b = D - 1; b >= 0 && m > 0; --b) {
        if ((double)r >= c) {
            mask |= 1u << b;
            r -= (unsigned long long)c;
            c = b > 0 ? (c * (double)m) / (double)b : 0.0;
            --m;
        } else {
            c = b > 0 ? (c * (double)(b - m)) / (double)b : 0.0;
        }
    }
    return mask;
}

// Dynamic work distribution of the class kernels (ClassItems::ctr): blocks take chunks
// of at most HAFB_DYN_CHUNK items per team, at least HAFB_DYN_PER chunks per team.
#ifndef HAFB_DYN
#define HAFB_DYN 1
#endif
#ifndef HAFB_DYN_CHUNK
#define HAFB_DYN_CHUNK 16
#endif
#ifndef HAFB_DYN_PER
#define HAFB_DYN_PER 8
#endif

struct ItemRef {
    uint32_t mask;
    long long problem;
    long long out;  // buffer index (including the problem offset)
};

__device__ __forceinline__ ItemRef resolve_item(const ClassItems& ci, long long item) {
    ItemRef r;
    r.problem = item / ci.per_problem;
    long long rho = item - r.problem * ci.per_problem;
    if (ci.mlist) {
        r.mask = ci.mlist[rho];
        r.out = r.problem * ci.term_stride + ci.mout[rho];
        return r;
    }
    if (ci.nseg == 1) {
        r.mask = unrank_mask(ci.base0 + (unsigned long long)rho, ci.m, ci.D, ci.c_top);
        r.out = r.problem * ci.term_stride + ci.seg0.out_off + (long long)(r.mask - ci.seg0.lo);
        return r;
    }
    int lo = 0, hi = ci.nseg - 1;
    while (lo < hi) {  // last s with prefix[s] <= rho
        int mid = (lo + hi + 1) >> 1;
        if (ci.prefix[mid] <= rho) lo = mid;
        else hi = mid - 1;
    }
    const Seg sg = ci.segs[lo];
    r.mask = unrank_mask(ci.base[lo] + (unsigned long long)(rho - ci.prefix[lo]), ci.m, ci.D, ci.c_top);
    r.out = r.problem * ci.term_stride + sg.out_off + (long long)(r.mask - sg.lo);
    return r;
}

// Sequential walk over consecutive items of a class.  Inside one segment of one
// problem, class rank rho+1 is the next larger integer of popcount m (colex order),
// obtained from the current mask by Gosper's step; the full unranking (~D dependent
// double divisions) runs only at the first item and at segment/problem edges.
struct ItemCursor {
    long long next = -1;      // the item that continues the walk
    long long item_end = -1;  // first item outside the current segment (or problem)
    long long delta = 0;      // out - mask inside the current segment
    ItemRef ref;
};

__device__ __forceinline__ uint32_t next_same_popcount(uint32_t x) {
    const uint32_t c = x & (0u - x);
    const uint32_t r = x + c;
    return (((r ^ x) >> 2) >> (__ffs(x) - 1)) | r;
}

__device__ __forceinline__ ItemRef cursor_item(const ClassItems& ci, long long item, ItemCursor& cur) {
    if (!ci.mlist && item == cur.next && item < cur.item_end) {
        cur.next = item + 1;
        cur.ref.mask = next_same_popcount(cur.ref.mask);
        cur.ref.out = (long long)cur.ref.mask + cur.delta;
        return cur.ref;
    }
    cur.next = item + 1;
    cur.ref = resolve_item(ci, item);
    if (!ci.mlist) {
        const long long p0 = cur.ref.problem * ci.per_problem;
        if (ci.nseg == 1) {
            cur.item_end = p0 + ci.per_problem;
            cur.delta = cur.ref.out - (long long)cur.ref.mask;
            return cur.ref;
        }
        const long long rho = item - p0;
        int lo = 0, hi = ci.nseg - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (ci.prefix[mid] <= rho) lo = mid;
            else hi = mid - 1;
        }
        cur.item_end = p0 + ci.prefix[lo + 1];
        cur.delta = cur.ref.out - (long long)cur.ref.mask;
    }
    return cur.ref;
}

}  // namespace hafb
