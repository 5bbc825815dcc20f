// qr_fast.cuh -- FAST spectral backend: eigenvalues of the packed upper-Hessenberg form
// by the reference's implicit single-shift QR (_numba.py:70-188), then power sums
// (_numba.py:191-200), in FMA arithmetic on one team (W = 16 or 32 lanes).
//
// Same algorithm and control flow as the reference -- the deflation test
// |h(l,l-1)| <= 1e-14 (|h(l,l)| + |h(l-1,l-1)|) scanned from the bottom of the active
// block, 1x1 and 2x2 deflations (the 2x2 eigenvalue pair by the reference's formulas),
// the Wilkinson-type shift with an exceptional shift every tenth stagnant sweep, the
// Givens convention [[c, s], [-conj(s), c]] and the sweep cap cap_mult * S (status 1)
// -- with these exact-arithmetic substitutions: |z| = sqrt(re^2 + im^2) (no hypot
// scaling), divisions through a reciprocal, the deflation scan done by all lanes at
// once (each lane tests one position; the first hit from the bottom wins, as in the
// sequential scan), and the power sums lambda_i^k by binary powering (lane = k).
//
// Storage: column c of the packed form holds rows 0..c+1 at c(c+3)/2 (term_fast.cuh).
// The bulge of the chase (row k+2 of column k, below the subdiagonal) never goes to
// memory: every lane carries it in a register from one rotation to the next.
#pragma once

#include "cplx.cuh"

namespace hafb {

__device__ __forceinline__ int pk_idx(int r, int c) { return (c * (c + 3)) / 2 + r; }

__device__ __forceinline__ double q_abs(cd z) { return sqrt(fma(z.re, z.re, z.im * z.im)); }
__device__ __forceinline__ cd q_conj(cd z) { return mk(z.re, -z.im); }
__device__ __forceinline__ cd q_scale(cd z, double a) { return mk(z.re * a, z.im * a); }
__device__ __forceinline__ cd q_sub(cd a, cd b) { return mk(a.re - b.re, a.im - b.im); }
// x / y
__device__ __forceinline__ cd q_div(cd x, cd y) {
    const double r = 1.0 / fma(y.re, y.re, y.im * y.im);
    return q_scale(f_mul(x, q_conj(y)), r);
}
// principal square root
__device__ __forceinline__ cd q_sqrt(cd z) {
    const double r = q_abs(z);
    if (r == 0.0) return mk(0.0, 0.0);
    if (z.re >= 0.0) {
        const double t = sqrt(0.5 * (r + z.re));
        return mk(t, z.im / (2.0 * t));
    }
    const double t = sqrt(0.5 * (r - z.re));
    return mk(fabs(z.im) / (2.0 * t), copysign(t, z.im));
}

// 1/sqrt(d), finite d > 0: hardware estimate + two Newton steps
__device__ __forceinline__ double q_rsqrt(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double h = 0.5 * d;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// _numba.py:70-82: c real, s complex with [[c, s], [-conj(s), c]] (x, y) = (r, 0).
// With nx = |x|^2, ny = |y|^2 and q = 1/sqrt(nx (nx + ny)): c = nx q = |x|/r and
// s = x conj(y) q = (x/|x|)(conj(y)/r) -- one reciprocal square root on the chain.
__device__ __forceinline__ void q_givens(cd x, cd y, double& c, cd& s) {
    const double nx = fma(x.re, x.re, x.im * x.im), ny = fma(y.re, y.re, y.im * y.im);
    if (ny == 0.0) {
        c = 1.0;
        s = mk(0.0, 0.0);
    } else if (nx == 0.0) {
        c = 0.0;
        s = q_scale(q_conj(y), q_rsqrt(ny));
    } else {
        const double q = q_rsqrt(nx * (nx + ny));
        c = nx * q;
        s = q_scale(f_mul(x, q_conj(y)), q);
    }
}

// One implicit single-shift bulge chase on the active block [lo, hi] (_numba.py:85-112).
template <int W, class Sync>
__device__ __forceinline__ void q_sweep(cd* Hs, int lo, int hi, cd shift, int lane, Sync&& sync) {
    cd bulge = mk(0.0, 0.0);  // h(k+1, k-1) entering step k (k > lo)
    for (int k = lo; k < hi; ++k) {
        cd x, y;
        if (k == lo) {
            x = q_sub(Hs[pk_idx(lo, lo)], shift);
            y = Hs[pk_idx(lo + 1, lo)];
        } else {
            x = Hs[pk_idx(k, k - 1)];
            y = bulge;
        }
        double c;
        cd s;
        q_givens(x, y, c, s);
        const cd sc = q_conj(s);
        // h(k+2, k+1) before the column rotation touches it: the next bulge is conj(s) * it
        const bool more = k + 2 <= hi;
        const cd h21 = more ? Hs[pk_idx(k + 2, k + 1)] : mk(0.0, 0.0);
        sync();  // every lane has read x, y and h21 before the rotations overwrite them
        // row rotation, columns col0..hi (lane = column); the bulge column k-1 rotates
        // (x, y) in registers and drops its row k+1 entry (reference: set to 0) -- selects
        // and predicated stores, no divergent region
        const int col0 = k == lo ? lo : k - 1;
        for (int col = col0 + lane; col <= hi; col += W) {
            const bool bc = col == k - 1;
            const int b = (col * (col + 3)) / 2;
            const cd l1 = Hs[b + k], l2 = Hs[b + k + 1];
            const cd t1 = bc ? x : l1, t2 = bc ? y : l2;
            Hs[b + k] = f_cma(q_scale(t1, c), s, t2);
            if (!bc) Hs[b + k + 1] = f_cms(q_scale(t2, c), sc, t1);
        }
        sync();
        // column rotation, rows lo..min(k+2, hi) (lane = row); row k+2 of column k is the
        // new bulge (zero before, conj(s) h21 after: kept in a register), its column k+1
        // entry becomes c h21
        const int re = more ? k + 2 : hi;
        const int b0 = (k * (k + 3)) / 2, b1 = b0 + k + 2;  // columns k, k+1
        for (int row = lo + lane; row <= re; row += W) {
            const bool br = row == k + 2;
            const cd l1 = Hs[b0 + row], t2 = Hs[b1 + row];
            const cd t1 = br ? mk(0.0, 0.0) : l1;
            if (!br) Hs[b0 + row] = f_cma(q_scale(t1, c), sc, t2);
            Hs[b1 + row] = f_cms(q_scale(t2, c), s, t1);
        }
        bulge = f_mul(sc, h21);
        sync();
    }
}

// Eigenvalues of the packed S x S Hessenberg form into eig[0..S) (_numba.py:115-188).
// Returns converged; `sweeps` = sweeps used.  Destroys Hs.
template <int S, int W, class Sync>
__device__ __forceinline__ bool q_eigvals(cd* Hs, cd* eig, int cap_mult, int lane, int& sweeps,
                                          Sync&& sync) {
    constexpr double kRtol = 1e-14;  // DEFLATION_RTOL, _numba.py:32
    const int cap = cap_mult * S;
    int total = 0, stagnation = 0;
    int hi = S - 1;
    bool conv = true;
    HT_DECL
    while (hi >= 0) {
        if (hi == 0) {
            if (lane == 0) eig[0] = Hs[pk_idx(0, 0)];
            break;
        }
        // deflation scan: positions p = hi, hi-1, ..., 1; the first small subdiagonal
        // from the bottom wins (lane l tests p = hi - l, W positions per round)
        int lo = 0;
        for (int base = hi; base >= 1; base -= W) {
            const int p = base - lane;
            bool small = false;
            if (p >= 1) {
                const double sd = q_abs(Hs[pk_idx(p, p - 1)]);
                small = sd <= kRtol * (q_abs(Hs[pk_idx(p, p)]) + q_abs(Hs[pk_idx(p - 1, p - 1)]));
            }
            const unsigned b = __ballot_sync(W < 32 ? (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)))
                                                    : 0xffffffffu,
                                             small);
            const unsigned mine = W < 32 ? (b >> ((threadIdx.x & 31) & ~(W - 1))) & ((1u << W) - 1u) : b;
            if (mine) {
                lo = base - (__ffs(mine) - 1);
                break;
            }
        }
        sync();
        HT_MARK(5);
        if (lo > 0 && lane == 0) Hs[pk_idx(lo, lo - 1)] = mk(0.0, 0.0);
        if (lo == hi) {
            if (lane == 0) eig[hi] = Hs[pk_idx(hi, hi)];
            sync();
            hi -= 1;
            stagnation = 0;
            continue;
        }
        if (lo == hi - 1) {
            const cd a = Hs[pk_idx(lo, lo)], b = Hs[pk_idx(lo, hi)], cc = Hs[pk_idx(hi, lo)],
                     d = Hs[pk_idx(hi, hi)];
            const cd half = q_scale(f_add(a, d), 0.5);
            const cd det = f_cms(f_mul(a, d), b, cc);
            const cd disc = q_sqrt(f_cms(f_mul(half, half), mk(1.0, 0.0), det));
            const cd e1 = f_add(half, disc), e2 = q_sub(half, disc);
            if (lane == 0) {
                const double a1 = q_abs(e1), a2 = q_abs(e2);
                if (a1 >= a2) {
                    eig[hi] = e1;
                    eig[lo] = a1 > 0.0 ? q_div(det, e1) : e2;
                } else {
                    eig[hi] = e2;
                    eig[lo] = a2 > 0.0 ? q_div(det, e2) : e1;
                }
            }
            sync();
            hi -= 2;
            stagnation = 0;
            continue;
        }
        if (total >= cap) {
            conv = false;
            break;
        }
        stagnation += 1;
        cd shift;
        if (stagnation % 10 == 0) {
            shift = f_add(Hs[pk_idx(hi, hi)], mk(0.75 * q_abs(Hs[pk_idx(hi, hi - 1)]), 0.0));
        } else {
            const cd a = Hs[pk_idx(hi - 1, hi - 1)], b = Hs[pk_idx(hi - 1, hi)],
                     cc = Hs[pk_idx(hi, hi - 1)], d = Hs[pk_idx(hi, hi)];
            const cd delta = q_scale(q_sub(a, d), 0.5);
            const cd bc = f_mul(b, cc);
            const cd disc = q_sqrt(f_cma(bc, delta, delta));
            const cd d1 = f_add(delta, disc), d2 = q_sub(delta, disc);
            const cd den = q_abs(d1) >= q_abs(d2) ? d1 : d2;
            shift = (den.re == 0.0 && den.im == 0.0) ? d : q_sub(d, q_div(bc, den));
        }
        HT_MARK(6);
        q_sweep<W>(Hs, lo, hi, shift, lane, sync);
        HT_MARK(7);
        total += 1;
    }
    sync();
    sweeps = total;
    return conv;
}

// t_k = sum_i lambda_i^k, k = 1..D, into T[1..D] (_numba.py:191-200; lane k-1 owns t_k;
// the power by binary powering, the squarings shared by every lane)
template <int S, int W>
__device__ __forceinline__ void q_power_sums(const cd* eig, cd* T, int D, int lane) {
    constexpr int R = (32 + W - 1) / W;
    cd acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = mk(0.0, 0.0);
    for (int i = 0; i < S; ++i) {
        cd base = eig[i];
        cd res[R];
#pragma unroll
        for (int r = 0; r < R; ++r) res[r] = mk(1.0, 0.0);
#pragma unroll
        for (int bit = 0; bit < 6; ++bit) {  // k <= 32 < 2^6
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = lane + 1 + W * r;
                if ((k >> bit) & 1) res[r] = f_mul(res[r], base);
            }
            base = f_mul(base, base);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = f_add(acc[r], res[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int k = lane + 1 + W * r;
        if (k <= D) T[k] = acc[r];
    }
}

}  // namespace hafb
