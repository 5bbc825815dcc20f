// term_smem.cuh -- general subset-term kernel: one warp per subset, the subset
// matrix staged in shared memory.  Handles every size s = 2|Z| <= 64, both
// backends (charpoly / spectral), with and without loop terms, in MIRROR
// arithmetic (bit-identical to the reference).  The register-resident kernels
// (term_fast.cuh for FAST, term_mirror.cuh for the bit-exact charpoly backend)
// take over the FLOP-heavy sizes; this kernel covers the rest
// and is the parity baseline for them.
//
// Reference: pkg/src/hafnium/kernels/_numba.py
//   subset_term        :297-351   (gather, dispatch, series, loops, exp, sign)
//   _hessenberg        :36-67     (pivoted elementary similarity)
//   _charpoly          :203-225   (leading-minor recurrence)
//   _traces_from_charpoly :228-250
//   _hess_eigvals/_qr_sweep/_givens :70-188, _power_sums :191-200
//   _loop_chain        :253-273,  _exp_top :276-294
//
// Parallelisation never reorders a floating-point reduction: every sum the
// reference computes sequentially is computed sequentially by one lane, and
// lanes only split loops whose iterations are independent in the reference.
#pragma once

#include "cplx.cuh"
#include "enumerate.cuh"

namespace hafb {

constexpr int kMaxHalf = 32;  // masks are 32-bit on the device: n <= 64, s <= 64
constexpr double kDeflationRtol = 1e-14;  // _numba.py:32

// shared-memory footprint (in cd elements) of one warp's workspace for subset
// matrices up to size S with K = n/2 power traces (S = n when the warp may see any
// subset; S = 2m for a one-class launch)
__host__ __device__ inline int smem_warp_elems(int S, int K) {
    int hreg = S * S > S * K ? S * S : S * K;  // H doubles as the power-sum scratch
    int pt = (S + 1) * (S + 2) / 2;            // triangular charpoly table
    return hreg + pt + 6 * (S + 2) + 3 * (K + 2);
}
__host__ __device__ inline int smem_warp_elems(int n) { return smem_warp_elems(n, n / 2); }
// the spectral class kernel's compact workspace: the S x S matrix, five S+2 vectors
// (loop vectors, the vertex list, eigenvalues) and three K+2 series vectors -- no
// charpoly table, and the power sums need no S x K scratch (lane k recomputes the
// reference's power chain, see subset_term_smem).  At S = 20, n = 52: 9.5 KB per warp
// instead of 15.5 KB, two 8-warp blocks per SM instead of one.
__host__ __device__ inline int smem_warp_elems_spec(int S, int K) { return S * S + 5 * (S + 2) + 3 * (K + 2); }

struct WarpWs {
    cd* H;    // s*s, row-major, ld = s (also the s*K power-sum scratch)
    cd* P;    // triangular: row k at k(k+1)/2, length k+1
    cd* vec;  // misc vectors, each S+2
    cd* mu;
    cd* v;
    cd* xv;
    cd* u;
    cd* unew;
    cd* eig;
    cd* t;    // K+2
    cd* s;    // K+2
    cd* E;    // K+2
};

__device__ inline WarpWs carve(cd* base, int S, int K) {
    WarpWs w;
    int hreg = S * S > S * K ? S * S : S * K;
    w.H = base;
    w.P = w.H + hreg;
    cd* q = w.P + (S + 1) * (S + 2) / 2;
    w.mu = q; q += S + 2;
    w.v = q; q += S + 2;
    w.xv = q; q += S + 2;
    w.u = q; q += S + 2;
    w.unew = q; q += S + 2;
    w.eig = q; q += S + 2;
    w.t = q; q += K + 2;
    w.s = q; q += K + 2;
    w.E = q; q += K + 2;
    w.vec = nullptr;
    return w;
}
__device__ inline WarpWs carve(cd* base, int n) { return carve(base, n, n / 2); }
__device__ inline WarpWs carve_spec(cd* base, int S, int K) {
    WarpWs w;
    w.H = base;
    w.P = nullptr;
    cd* q = w.H + S * S;
    w.mu = nullptr;
    w.v = q; q += S + 2;
    w.xv = q; q += S + 2;
    w.u = q; q += S + 2;
    w.unew = q; q += S + 2;
    w.eig = q; q += S + 2;
    w.t = q; q += K + 2;
    w.s = q; q += K + 2;
    w.E = q; q += K + 2;
    w.vec = nullptr;
    return w;
}

// ------------------------------------------------------------------ Hessenberg
// _numba.py:36-67.  The i-loop is sequential (each i's row op then column op);
// within one row op / column op the k iterations are independent -> lanes.
__device__ inline void hess_smem(cd* H, int m, int lane) {
#define HH(r, c) H[(r) * m + (c)]
    for (int j = 0; j < m - 2; ++j) {
        // pivot: first index attaining the max of hypot(h[i,j]), i >= j+1 (strict '>' scan)
        double best = -1.0;
        int bi = 0x7fffffff;
        for (int i = j + 1 + lane; i < m; i += 32) {
            double a = m_abs(HH(i, j));
            if (a > best) { best = a; bi = i; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            double ob = __shfl_xor_sync(0xffffffffu, best, off);
            int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        double big0 = m_abs(HH(j + 1, j));
        int piv = bi;
        double big = best;
        if (isnan(big0) || bi == 0x7fffffff) { piv = j + 1; big = big0; }
        if (big == 0.0) continue;
        if (piv != j + 1) {
            for (int k = j + lane; k < m; k += 32) {
                cd t = HH(piv, k); HH(piv, k) = HH(j + 1, k); HH(j + 1, k) = t;
            }
            __syncwarp();
            for (int k = lane; k < m; k += 32) {
                cd t = HH(k, piv); HH(k, piv) = HH(k, j + 1); HH(k, j + 1) = t;
            }
            __syncwarp();
        }
        cd p = HH(j + 1, j);
        for (int i = j + 2; i < m; ++i) {
            cd mu = m_div(HH(i, j), p);  // column j is untouched inside step j
            __syncwarp();
            if (m_nz(mu)) {
                for (int k = j + 1 + lane; k < m; k += 32)
                    HH(i, k) = m_sub(HH(i, k), m_mul(mu, HH(j + 1, k)));
                __syncwarp();
                for (int k = lane; k < m; k += 32)
                    HH(k, j + 1) = m_add(HH(k, j + 1), m_mul(mu, HH(k, i)));
                __syncwarp();
            }
            if (lane == 0) HH(i, j) = mk(0.0, 0.0);
        }
        __syncwarp();
    }
#undef HH
}

// ------------------------------------------------------------------ charpoly
// _numba.py:203-225 on a triangular table; lane d owns coefficient d.
__device__ inline void charpoly_smem(const cd* H, int m, cd* P, int lane) {
#define HH(r, c) H[(r) * m + (c)]
#define PR(k) (P + (k) * ((k) + 1) / 2)
    if (lane == 0) P[0] = mk(1.0, 0.0);
    __syncwarp();
    for (int k = 1; k <= m; ++k) {
        cd* Pk = PR(k);
        const cd* Pk1 = PR(k - 1);
        cd hk = HH(k - 1, k - 1);
        for (int d = lane; d <= k; d += 32) {
            cd v;
            if (d == k) {
                v = Pk1[k - 1];
            } else {
                cd base = d >= 1 ? Pk1[d - 1] : mk(0.0, 0.0);
                v = m_sub(base, m_mul(hk, Pk1[d]));
            }
            // prod chain is uniform across lanes; each lane applies the i-terms to its d
            cd prod = mk(1.0, 0.0);
            for (int i = k - 1; i > 0; --i) {
                prod = m_mul(prod, HH(i, i - 1));
                if (!m_nz(prod)) break;
                cd coef = m_mul(HH(i - 1, k - 1), prod);
                if (m_nz(coef) && d < i) v = m_sub(v, m_mul(coef, PR(i - 1)[d]));
            }
            Pk[d] = v;
        }
        __syncwarp();
    }
#undef HH
#undef PR
}

// _numba.py:228-250 (sequential; lane 0).  returns ok
__device__ inline bool traces_from_charpoly_seq(const cd* a, int m, int K, cd* t) {
    for (int k = 0; k < K; ++k) t[k] = mk(0.0, 0.0);
    int kmax = K < m ? K : m;
    for (int k = 1; k <= kmax; ++k) {
        cd acc = m_mul(mk((double)(-k), 0.0), a[m - k]);
        for (int j = 1; j < k; ++j) acc = m_sub(acc, m_mul(a[m - j], t[k - j - 1]));
        t[k - 1] = acc;
    }
    if (m >= 1) {
        for (int k = m + 1; k <= K; ++k) {
            cd acc = mk(0.0, 0.0);
            for (int j = 0; j < m; ++j) acc = m_sub(acc, m_mul(a[j], t[k - m + j - 1]));
            t[k - 1] = acc;
        }
    }
    bool ok = true;
    for (int k = 0; k < K; ++k)
        if (!m_finite(t[k])) ok = false;
    return ok;
}

// ------------------------------------------------------------------ spectral
// _numba.py:70-82
__device__ inline void givens_m(cd x, cd y, double& c, cd& s) {
    double ax = m_abs(x), ay = m_abs(y);
    if (ay == 0.0) { c = 1.0; s = mk(0.0, 0.0); return; }
    if (ax == 0.0) { c = 0.0; s = m_rdiv(mk(y.re, -y.im), ay); return; }
    double r = m_hypot(ax, ay);
    c = r_div(ax, r);
    s = m_mul(m_rdiv(x, ax), m_rdiv(mk(y.re, -y.im), r));
}

// _numba.py:85-112; rotations of one sweep step are lane-parallel over columns/rows
__device__ inline void qr_sweep_smem(cd* H, int m, int lo, int hi, cd shift, int lane) {
#define HH(r, c) H[(r) * m + (c)]
    for (int k = lo; k < hi; ++k) {
        cd x, y;
        if (k == lo) { x = m_sub(HH(lo, lo), shift); y = HH(lo + 1, lo); }
        else { x = HH(k, k - 1); y = HH(k + 1, k - 1); }
        double c; cd s;
        givens_m(x, y, c, s);
        cd sc = mk(s.re, -s.im);
        __syncwarp();
        int col0 = (k == lo) ? lo : k - 1;
        for (int col = col0 + lane; col <= hi; col += 32) {
            cd t1 = HH(k, col), t2 = HH(k + 1, col);
            HH(k, col) = m_add(m_rmul(c, t1), m_mul(s, t2));
            // col == k-1 (k > lo): the reference rotates, then sets h[k+1, k-1] = 0
            // (_numba.py:102-103) -- store the final 0 directly
            HH(k + 1, col) = col == k - 1 ? mk(0.0, 0.0) : m_add(m_mul(m_neg(sc), t1), m_rmul(c, t2));
        }
        __syncwarp();
        int row_end = k + 2;
        if (row_end > hi) row_end = hi;
        for (int row = lo + lane; row <= row_end; row += 32) {
            cd t1 = HH(row, k), t2 = HH(row, k + 1);
            HH(row, k) = m_add(m_rmul(c, t1), m_mul(sc, t2));
            HH(row, k + 1) = m_add(m_mul(m_neg(s), t1), m_rmul(c, t2));
        }
        __syncwarp();
    }
#undef HH
}

// _numba.py:115-188 after the Hessenberg reduction. returns converged; eig[] filled
__device__ inline bool hess_eigvals_smem(cd* H, int m, int cap_mult, cd* eig, int lane,
                                         long long* sweeps_out = nullptr) {
#define HH(r, c) H[(r) * m + (c)]
    for (int i = lane; i < m; i += 32) eig[i] = mk(0.0, 0.0);
    __syncwarp();
    if (m == 0) return true;
    hess_smem(H, m, lane);
    long long total = 0;
    long long cap = (long long)cap_mult * m;
    int hi = m - 1;
    long long stagnation = 0;
    while (hi >= 0) {
        if (hi == 0) {
            if (lane == 0) eig[0] = HH(0, 0);
            break;
        }
        // deflation scan (_numba.py:132-138): positions lo = hi, hi-1, ..., 1, the first
        // small subdiagonal from the bottom wins.  Each lane evaluates the reference's test
        // for one position (the same operations, so the same decisions) and a ballot picks
        // the first hit: one round of three hypots instead of up to hi sequential ones.
        int lo = 0;
        for (int base = hi; base >= 1; base -= 32) {
            const int p = base - lane;
            bool small = false;
            if (p >= 1) {
                const double sd = m_abs(HH(p, p - 1));
                small = sd <= r_mul(kDeflationRtol, r_add(m_abs(HH(p, p)), m_abs(HH(p - 1, p - 1))));
            }
            const unsigned b = __ballot_sync(0xffffffffu, small);
            if (b) {
                lo = base - (__ffs(b) - 1);
                break;
            }
        }
        if (lo > 0) {
            __syncwarp();
            if (lane == 0) HH(lo, lo - 1) = mk(0.0, 0.0);
            __syncwarp();
        }
        if (lo == hi) {
            if (lane == 0) eig[hi] = HH(hi, hi);
            hi -= 1;
            stagnation = 0;
            continue;
        }
        if (lo == hi - 1) {
            cd a = HH(lo, lo), b = HH(lo, hi), cc = HH(hi, lo), d = HH(hi, hi);
            cd half = m_rmul(0.5, m_add(a, d));
            cd det = m_sub(m_mul(a, d), m_mul(b, cc));
            cd disc = m_sqrt(m_sub(m_mul(half, half), det));
            cd e1 = m_add(half, disc), e2 = m_sub(half, disc);
            if (lane == 0) {
                if (m_abs(e1) >= m_abs(e2)) {
                    eig[hi] = e1;
                    eig[lo] = (m_abs(e1) > 0.0) ? m_div(det, e1) : e2;
                } else {
                    eig[hi] = e2;
                    eig[lo] = (m_abs(e2) > 0.0) ? m_div(det, e2) : e1;
                }
            }
            hi -= 2;
            stagnation = 0;
            continue;
        }
        if (total >= cap) {
            if (sweeps_out) *sweeps_out = total;
            return false;
        }
        stagnation += 1;
        cd shift;
        if (stagnation % 10 == 0) {
            shift = m_add(HH(hi, hi), mk(r_mul(0.75, m_abs(HH(hi, hi - 1))), 0.0));
        } else {
            cd a = HH(hi - 1, hi - 1), b = HH(hi - 1, hi), cc = HH(hi, hi - 1), d = HH(hi, hi);
            cd delta = m_rmul(0.5, m_sub(a, d));
            cd bc = m_mul(b, cc);
            cd disc = m_sqrt(m_add(m_mul(delta, delta), bc));
            cd d1 = m_add(delta, disc), d2 = m_sub(delta, disc);
            cd den = (m_abs(d1) >= m_abs(d2)) ? d1 : d2;
            if (!m_nz(den)) shift = d;
            else shift = m_sub(d, m_div(bc, den));
        }
        qr_sweep_smem(H, m, lo, hi, shift, lane);
        total += 1;
    }
    __syncwarp();
    if (sweeps_out) *sweeps_out = total;
    return true;
#undef HH
}

// ------------------------------------------------------------------ the term
// One warp evaluates subset `mask` (32-bit, nonzero).  BACKEND 1 = charpoly,
// 0 = spectral.  Returns (via lane 0) term and status.
template <int BACKEND, bool LOOPS>
__device__ inline void subset_term_smem(const cd* __restrict__ atilde, const cd* __restrict__ diag,
                                        int n_half, uint32_t mask, int cap_mult, WarpWs& w,
                                        int lane, cd& term_out, int& status_out) {
    const int n = 2 * n_half;
    const int K = n_half;
    const int m = __popc(mask);
    const int size = 2 * m;
    // vertex list: pair p -> (2*bit, 2*bit+1); stored as ints in w.unew scratch
    int* idx = reinterpret_cast<int*>(w.unew);
    if (lane < m) {
        int bit = __fns(mask, 0, lane + 1);
        idx[2 * lane] = 2 * bit;
        idx[2 * lane + 1] = 2 * bit + 1;
    }
    __syncwarp();
    for (int e = lane; e < size * size; e += 32) {
        int r = e / size, c = e - r * size;
        w.H[e] = atilde[idx[r] * n + idx[c]];
    }
    if (LOOPS) {
        for (int r = lane; r < size; r += 32) w.v[r] = diag[idx[r]];
    }
    __syncwarp();
    int status = 0;
    if (BACKEND == 1) {
        hess_smem(w.H, size, lane);
        charpoly_smem(w.H, size, w.P, lane);
        const cd* a = w.P + size * (size + 1) / 2;
        int ok = 1;
        if (lane == 0) ok = traces_from_charpoly_seq(a, size, K, w.t) ? 1 : 0;
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) status = 2;
    } else {
        bool conv = hess_eigvals_smem(w.H, size, cap_mult, w.eig, lane);
        if (!conv) {
            status = 1;
        } else {
            // _power_sums (_numba.py:191-200): t[k] += p over eigenvalues i in order, with
            // p = lam^(k+1) from the reference's chain p = lam, p *= lam, ...  Lane k replays
            // that chain for its own k (the same k multiplications per eigenvalue, so the
            // same bits) and accumulates over i in order: no S x K scratch.
            __syncwarp();
            for (int k = lane; k < K; k += 32) {
                cd acc = mk(0.0, 0.0);
                for (int i = 0; i < size; ++i) {
                    const cd lam = w.eig[i];
                    cd p = lam;
                    for (int j = 0; j < k; ++j) p = m_mul(p, lam);
                    acc = m_add(acc, p);
                }
                w.t[k] = acc;
            }
        }
    }
    __syncwarp();
    if (status != 0) {
        term_out = mk(0.0, 0.0);
        status_out = status;
        return;
    }
    // series s_k = t_k / (2k)   (_numba.py:334-336)
    for (int k = lane; k <= K; k += 32)
        w.s[k] = (k == 0) ? mk(0.0, 0.0) : m_rdiv(w.t[k - 1], r_mul(2.0, (double)k));
    __syncwarp();
    if (LOOPS) {
        // Xv swaps v within each pair; _loop_chain over the UN-reduced gathered B
        for (int r = lane; r < size; r += 32) {
            w.xv[r] = w.v[r ^ 1];
            w.u[r] = w.v[r];
        }
        __syncwarp();
        for (int k = 0; k < K; ++k) {
            if (lane == 0) {
                cd acc = mk(0.0, 0.0);
                for (int i = 0; i < size; ++i) acc = m_add(acc, m_mul(w.u[i], w.xv[i]));
                // s[k+1] += 0.5 * ell[k]
                w.s[k + 1] = m_add(w.s[k + 1], m_rmul(0.5, acc));
            }
            if (k < K - 1) {
                cd un[2];
                for (int q = 0; q < 2; ++q) {
                    int j = lane + 32 * q;
                    if (j < size) {
                        cd acc = mk(0.0, 0.0);
                        for (int i = 0; i < size; ++i)
                            acc = m_add(acc, m_mul(w.u[i], atilde[idx[i] * n + idx[j]]));
                        un[q] = acc;
                    }
                }
                __syncwarp();
                for (int q = 0; q < 2; ++q) {
                    int j = lane + 32 * q;
                    if (j < size) w.u[j] = un[q];
                }
            }
            __syncwarp();
        }
    }
    // _exp_top (_numba.py:276-294): lane d owns E[d] (and E[d + 32]: D = 32 needs 33
    // coefficients); each F[d] is a sequential sum
    const int D = K;
    for (int d = lane; d <= D; d += 32) w.E[d] = (d == 0) ? mk(1.0, 0.0) : mk(0.0, 0.0);
    __syncwarp();
    // (only E[D] is returned: at step j the coefficients d > D - j + 1 never reach it and
    // are skipped; the computed ones keep their operation sequences)
    for (int j = D; j > 0; --j) {
        double inv = r_div(1.0, (double)j);
        const int dmax = D - j + 1;
        cd f[2] = {mk(0.0, 0.0), mk(0.0, 0.0)};
        for (int q = 0; q < 2; ++q) {
            const int d = lane + 32 * q;
            if (d <= dmax) {
                cd acc = mk(0.0, 0.0);
                for (int tt = 1; tt <= d; ++tt) acc = m_add(acc, m_mul(w.E[d - tt], w.s[tt]));
                f[q] = m_rmul(inv, acc);
                if (d == 0) f[q] = m_add(f[q], mk(1.0, 0.0));
            }
        }
        __syncwarp();
        for (int q = 0; q < 2; ++q)
            if (lane + 32 * q <= dmax) w.E[lane + 32 * q] = f[q];
        __syncwarp();
    }
    cd coeff = w.E[D];
    term_out = ((n_half - m) & 1) ? m_neg(coeff) : coeff;
    status_out = 0;
}

// Where item q of a problem takes its mask from (term buffers are indexed by q).
struct MaskMap {
    uint64_t lo;                 // plain mode: mask = lo + q
    const uint32_t* mask_list;   // explicit masks
    const int32_t* range_list;   // range mode: q -> range range_list[q / width], offset q % width
    uint64_t width;
    uint64_t total;              // 2^n_half; range-mode masks >= total are padding (skipped)
    __device__ __forceinline__ uint32_t operator()(long long q) const {
        if (mask_list) return mask_list[q];
        if (range_list) {
            long long p = q / (long long)width, off = q - p * (long long)width;
            uint64_t m = 1 + (uint64_t)range_list[p] * width + (uint64_t)off;
            return m < total ? (uint32_t)m : 0u;
        }
        return (uint32_t)(lo + (uint64_t)q);
    }
};

// Terms for item it in [0, total_items): problem b = it / per, q = it % per, mask = map(q);
// problem b reads atilde + b*at_stride, diag + b*dg_stride.
// Mask 0 yields term 0 / status 0 (the drivers skip it).
template <int BACKEND, bool LOOPS>
__global__ void __launch_bounds__(256) terms_smem_kernel(
    const cd* __restrict__ atilde, const cd* __restrict__ diag, int n_half, MaskMap map,
    long long per, long long total_items, int cap_mult, long long at_stride, long long dg_stride,
    cd* __restrict__ terms, int8_t* __restrict__ status) {
    extern __shared__ cd smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int n = 2 * n_half;
    WarpWs w = carve(smem + (size_t)wib * smem_warp_elems(n), n);
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long it = (long long)blockIdx.x * (blockDim.x >> 5) + wib; it < total_items; it += nwarps) {
        long long b = it / per, q = it - b * per;
        uint32_t mask = map(q);
        cd t = mk(0.0, 0.0);
        int st = 0;
        if (mask != 0)
            subset_term_smem<BACKEND, LOOPS>(atilde + b * at_stride, diag + b * dg_stride, n_half,
                                             mask, cap_mult, w, lane, t, st);
        if (lane == 0) {
            terms[it] = t;
            if (st) status[it] = (int8_t)st;  // the buffer is zeroed by the host
        }
        __syncwarp();
    }
}

}  // namespace hafb

namespace hafb {
// Class-enumerated variant (one popcount class per launch, see enumerate.cuh);
// used for the sizes the register kernels do not cover.
template <int BACKEND, bool LOOPS>
__global__ void __launch_bounds__(256) terms_smem_class_kernel(
    const cd* __restrict__ atilde, const cd* __restrict__ diag, int n_half, ClassItems ci,
    int cap_mult, cd* __restrict__ terms, int8_t* __restrict__ status) {
    extern __shared__ cd smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int S = 2 * ci.m;  // one class per launch: size the workspace for it
    WarpWs w = BACKEND == 0 ? carve_spec(smem + (size_t)wib * smem_warp_elems_spec(S, n_half), S, n_half)
                            : carve(smem + (size_t)wib * smem_warp_elems(S, n_half), S, n_half);
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    // items one at a time: from the class's counter when set (per-subset QR times vary by
    // the sweep count, so a static interleave leaves warps idle at the end), else strided
    const bool dyn = HAFB_DYN && ci.ctr != nullptr;
    long long it = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    for (;;) {
        if (dyn) {
            unsigned long long g = 0;
            if (lane == 0) g = atomicAdd(ci.ctr, 1ull);
            it = (long long)__shfl_sync(0xffffffffu, g, 0);
        }
        if (it >= ci.n_items) break;
        const ItemRef ir = resolve_item(ci, it);
        cd t = mk(0.0, 0.0);
        int st = 0;
        subset_term_smem<BACKEND, LOOPS>(atilde + ir.problem * ci.at_stride,
                                         diag + ir.problem * ci.dg_stride, n_half, ir.mask,
                                         cap_mult, w, lane, t, st);
        if (lane == 0) {
            terms[ir.out] = t;
            if (st) status[ir.out] = (int8_t)st;  // the buffer is zeroed by the host
        }
        __syncwarp();
        if (!dyn) it += nwarps;
    }
}
}  // namespace hafb
