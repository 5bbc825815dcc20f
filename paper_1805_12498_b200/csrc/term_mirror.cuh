// term_mirror.cuh -- bit-exact (MIRROR) subset-term kernel for the charpoly backend.
//
// Same launch structure as the FAST kernel (one popcount class per launch, a team
// of W lanes per subset, lane r owns row r, the subset matrix in shared memory),
// but every floating-point value is produced by the same IEEE operations, on the
// same operands, in the same order as the reference (pkg/src/hafnium/kernels/
// _numba.py), using the m_* operations of cplx.cuh (no FMA contraction, Smith
// division, glibc hypot).  Lanes only ever split loops whose iterations are
// independent in the reference; every sequential reduction of the reference
// stays sequential.  Terms are bit-identical to _numba.subset_term(backend=1).
//
//   Hessenberg (_numba.py:36-67): the i-loop of step j is sequential.  Lane r
//     walks i = j+2..m-1 and applies, for its own row, exactly the updates the
//     reference applies to row r at iteration i: the deferred row operation of row
//     r on column i (value before/after it chosen by i >= r), the row operation on
//     column j+1 at i == r (against the pivot row's running h[j+1][j+1], which
//     every lane replays bit-identically), and the column operation.
//   charpoly (_numba.py:203-225): the prod/coef chains of all k run in parallel
//     (lane k-1 walks its own chain in the reference's order, with the break);
//     then P_k is built over k with lane d owning coefficient d and applying the
//     i-terms in the reference's descending order.
//   Newton / Cayley-Hamilton (_numba.py:228-250), series (:334-347) and the
//     Horner exp coefficient (_numba.py:276-294, O(D^3), lane-parallel over d).
#pragma once

#include "cplx.cuh"
#include "enumerate.cuh"
#include "term_fast.cuh"

namespace hafb {

constexpr int kMirrorThreads = 64;
#ifndef MIRROR_CP_UNROLL
#define MIRROR_CP_UNROLL 4
#endif
#ifndef MIRROR_HS_UNROLL
#define MIRROR_HS_UNROLL 1
#endif
// minimum resident 64-thread blocks per SM the register allocation must allow: 8 caps
// the kernel at 128 registers (16 warps/SM); left free, ptxas spent 255 at S = 28..32
// and registers, not shared memory, capped the teams per SM
#ifndef HAFB_MIRROR_MINB
#define HAFB_MIRROR_MINB 8
#endif
template <int S>
constexpr int mirror_minb() {
    return TeamWidth<S>::W >= 32 ? HAFB_MIRROR_MINB : 1;  // 16-lane teams spill at 128
}
constexpr int kMirrorCpUnroll = MIRROR_CP_UNROLL;  // charpoly i-loop unroll
constexpr int kMirrorHsUnroll = MIRROR_HS_UNROLL;  // Hessenberg column-loop unroll

// teams per block: one team per block from W = 32 up (the kernel is latency-bound and
// shared-memory-limited, so single-team blocks let leftover shared memory host one
// more team per SM); small teams share 64-thread blocks
template <int S>
constexpr int mirror_tpb() {
    return TeamWidth<S>::W >= 32 ? 1 : kMirrorThreads / TeamWidth<S>::W;
}

template <int S>
struct MirrorLayout {
    static constexpr int LD = S + 1;                     // odd column stride: conflict-free
    static constexpr int HSN = (S - 1) * (S + 2) / 2 + S;  // packed upper-Hessenberg entries
    // Region A holds, in turn (shared memory limits this kernel's teams per SM, so
    // nothing is kept twice):
    //   * the S x S subset matrix (column-major, stride LD) during the reduction;
    //   * the packed upper-Hessenberg form, column c at c(c+3)/2, packed IN PLACE column by
    //     column (column c's packed slot ends below column c's own source for S <= 52);
    //   * in the charpoly, the coefficients coef_{k,i} in place of h(i-1, k-1), and P_k
    //     (coefficients 0..k-1; P_k[k] = 1 is implicit) in the slot of column k-2, dead
    //     once P_{k-1} is built (it has exactly k entries); the final P_S goes to A;
    //   * after the charpoly, the monic charpoly A and the series scratch T, SS, E, beyond
    //     the packed region.
    // (S > 52: the packed form goes to its own region after the matrix)
    static constexpr bool INPLACE = S <= 52;
    static constexpr int H = 0;
    static constexpr int HS = INPLACE ? 0 : S * LD;
    static constexpr int A = HS + HSN;                   // [S+1] monic charpoly, ascending
    static constexpr int T = A + S + 1;                  // [kDMax+2] traces
    static constexpr int SS = T + kDMax + 2;             // [kDMax+2] series
    static constexpr int E = SS + kDMax + 2;             // [kDMax+2] exp Horner state
    static constexpr int AREA = S * LD > E + kDMax + 2 ? S * LD : E + kDMax + 2;
    static constexpr int U = AREA;                       // [2][S] loop-chain vector (before the reduction)
    static constexpr int MU = U + 2 * S;                 // [S+2] multipliers by logical row
    static constexpr int ELL = MU + S + 2;               // [kDMax+2] loop corrections
    static constexpr int RED = ELL + kDMax + 2;          // [8] cross-warp exchange (W = 64)
    static constexpr int P1 = RED + 8;                   // [1] P_1[0]
    static constexpr int INTS = P1 + 2;                  // int area (in cd slots)
    static constexpr int LMN = (2 * S + 3 * (S + 2) + 3) / 4 + 1;  // lm[2][S], stop[S+2], misc
    static constexpr int INVT = INTS + LMN;              // [kDMax+1] doubles: 1/j (_exp_top)
    static constexpr int TOTAL = INVT + (kDMax + 2) / 2;
};

// first-strict-max argmax over (key, row): larger key wins, ties -> smaller row; NaN
// keys never win (a > b and a == b are false for NaN), as in the reference's scan
template <int W>
__device__ __forceinline__ void team_argmax_exact(const TeamCtx<W>& tc, cd* red, double& key,
                                                  int& row, int& lane_of) {
    constexpr int WW = W < 32 ? W : 32;
#pragma unroll
    for (int off = WW / 2; off > 0; off >>= 1) {
        const double ok = tshfl_xor<W>(key, off);
        const int orow = tshfl_xor<W>(row, off);
        const int olane = tshfl_xor<W>(lane_of, off);
        if (ok > key || (ok == key && orow < row)) {
            key = ok;
            row = orow;
            lane_of = olane;
        }
    }
    if constexpr (W > 32) {
        const int w = tc.lane >> 5;
        if ((tc.lane & 31) == 0) {
            red[w] = mk(key, (double)row);
            red[2 + w] = mk((double)lane_of, 0.0);
        }
        tc.sync();
        const cd a0 = red[0], a1 = red[1];
        const bool second = a1.re > a0.re || (a1.re == a0.re && a1.im < a0.im);
        key = second ? a1.re : a0.re;
        row = (int)(second ? a1.im : a0.im);
        lane_of = (int)(second ? red[3].re : red[2].re);
        tc.sync();
    }
}

template <int W>
__device__ __forceinline__ cd team_bcast(const TeamCtx<W>& tc, cd* red, cd v, int src_lane) {
    if constexpr (W <= 32) {
        const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + src_lane;
        cd r;
        r.re = __shfl_sync(tc.wmask, v.re, src);
        r.im = __shfl_sync(tc.wmask, v.im, src);
        return r;
    } else {
        if (tc.lane == src_lane) red[4] = v;
        tc.sync();
        const cd r = red[4];
        tc.sync();
        return r;
    }
}

template <int S, bool LOOPS>
__global__ void __launch_bounds__(kMirrorThreads, mirror_minb<S>()) mirror_term_kernel(
    const cd* __restrict__ atilde, const cd* __restrict__ diag, int n_half, ClassItems ci,
    cd* __restrict__ terms, int8_t* __restrict__ status) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int TPB = mirror_tpb<S>();
    constexpr int M = S / 2;
    using L = MirrorLayout<S>;
    constexpr int LD = L::LD;
    extern __shared__ cd smem[];
    TeamCtx<W> tc;
    tc.tib = threadIdx.x / W;
    tc.lane = threadIdx.x % W;
    if constexpr (W < 32) {
        tc.wmask = ((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1));
    } else {
        tc.wmask = 0xffffffffu;
    }
    const int lane = tc.lane;
    cd* ws = smem + (size_t)tc.tib * L::TOTAL;
    cd* H = ws + L::H;
    cd* MU = ws + L::MU;
    cd* T = ws + L::T;
    cd* SSr = ws + L::SS;
    cd* E = ws + L::E;
    cd* ELL = ws + L::ELL;
    cd* RED = ws + L::RED;
    int* ints = reinterpret_cast<int*>(ws + L::INTS);
    int* LM0 = ints;            // [2][S] logical row -> lane
    int* STOP = ints + 2 * S;   // [S+2] smallest i of coef chain k (k = 1..S)
    const int n = 2 * n_half;
    const int D = n_half;
    // each team walks a contiguous run of the class's items (successive masks by Gosper's
    // step, ItemCursor): which team computes which subset changes, no arithmetic does
    const long long n_teams = (long long)gridDim.x * TPB;
    // work distribution as in the FAST kernel: dynamic block chunks from the class's
    // counter (every problem of a batch alike: this kernel stages nothing per block)
    const bool dyn = HAFB_DYN && ci.ctr != nullptr;
    long long ch = (ci.n_items + n_teams - 1) / n_teams;
    if (dyn) {
        ch = ci.n_items / (n_teams * HAFB_DYN_PER);
        ch = ch < 1 ? 1 : (ch > HAFB_DYN_CHUNK ? HAFB_DYN_CHUNK : ch);
    }
    const long long chunk = ch;
    long long first = ((long long)blockIdx.x * TPB + tc.tib) * chunk;
    ItemCursor cur;
    // _exp_top's 1/j for every j: the same correctly rounded quotients, computed once per
    // team instead of once per subset (D divisions on the chain of every term)
    double* INVJ = reinterpret_cast<double*>(ws + L::INVT);
    for (int j = lane; j <= kDMax; j += W) INVJ[j] = j ? r_div(1.0, (double)j) : 0.0;
    tc.sync();

    // block-shared: the spare slot of team 0's 1/j table
    long long* dyn_base = reinterpret_cast<long long*>(reinterpret_cast<double*>(smem + L::INVT) + kDMax + 1);
    for (;;) {
    if (dyn) {
        __syncthreads();
        if (threadIdx.x == 0) *dyn_base = (long long)atomicAdd(ci.ctr, (unsigned long long)(TPB * chunk));
        __syncthreads();
        const long long b0 = *dyn_base;
        if (b0 >= ci.n_items) break;
        first = b0 + (long long)tc.tib * chunk;
    }
    for (long long it = 0; it < chunk; ++it) {
        const long long item = first + it;
        const bool valid = item < ci.n_items;
        const ItemRef ir = cursor_item(ci, valid ? item : 0, cur);
        const cd* at = atilde + ir.problem * ci.at_stride;
        const cd* dg = diag + ir.problem * ci.dg_stride;
        int vbit[M];
        {
            uint32_t mm = ir.mask;
#pragma unroll
            for (int q = 0; q < M; ++q) {
                vbit[q] = __ffs(mm) - 1;
                mm &= mm - 1;
            }
        }
        const int mybit = lane < S ? (int)__fns(ir.mask, 0, (lane >> 1) + 1) : 0;
        const int vr = 2 * mybit + (lane & 1);
        HT_DECL
        // ------------------------------------------------ gather b = Atilde[idx][:, idx]
        if (lane < S) {
#pragma unroll
            for (int c = 0; c < S; ++c) H[c * LD + lane] = at[vr * n + 2 * vbit[c >> 1] + (c & 1)];
        }
        tc.sync();
        // ------------------------------------------------ loop chain (_numba.py:253-273)
        if constexpr (LOOPS) {
            cd* U = ws + L::U;
            // v = diag[idx], xv = pair-swapped v; u = v
            if (lane < S) U[lane] = dg[vr];
            tc.sync();
            for (int k = 0; k < D; ++k) {
                cd* u = U + (k & 1) * S;
                cd* un = U + ((k + 1) & 1) * S;
                // ell[k] = sum_i u[i]*xv[i] in order (every lane replays it; lane 0 stores)
                cd acc = mk(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < S; ++i) acc = m_add(acc, m_mul(u[i], dg[2 * vbit[i >> 1] + ((i & 1) ^ 1)]));
                if (lane == 0) ELL[k] = acc;
                if (k < D - 1) {
                    // unew[j] = sum_i u[i]*b[i][j], lane j, i in order
                    if (lane < S) {
                        cd s = mk(0.0, 0.0);
                        for (int i = 0; i < S; ++i) s = m_add(s, m_mul(u[i], H[lane * LD + i]));
                        un[lane] = s;
                    }
                }
                tc.sync();
            }
        }
        HT_MARK(0);
        // ------------------------------------------------ Hessenberg (_numba.py:36-67)
        int myrow = lane;
        if (lane < S) LM0[lane] = lane;
        tc.sync();
#pragma unroll 1
        for (int j = 0; j < S - 2; ++j) {
            const int B = j & 1;
            const int* lm = LM0 + B * S;
            int* lmn = LM0 + (1 - B) * S;
            const cd x = lane < S ? H[j * LD + lane] : mk(0.0, 0.0);
            double key = (myrow >= j + 1 && myrow < S) ? m_abs(x) : -1.0;
            const double mykey = key;
            int brow = myrow < S ? myrow : 0x3fffffff, blane = lane;
            team_argmax_exact<W>(tc, RED, key, brow, blane);
            const int l_j1 = lm[j + 1];
            double big0;
            if constexpr (W <= 32) {
                big0 = __shfl_sync(tc.wmask, mykey, ((int)(threadIdx.x & 31) & ~(W - 1)) + l_j1);
            } else {
                if (lane == l_j1) RED[5] = mk(mykey, 0.0);
                tc.sync();
                big0 = RED[5].re;
                tc.sync();
            }
            int piv = brow, plane = blane;
            double big = key;
            if (isnan(big0) || key < 0.0) {  // reference: nothing beats a NaN start
                piv = j + 1;
                plane = l_j1;
                big = big0;
            }
            if (big == 0.0) {  // `if big == 0.0: continue`
                if (lane < S) lmn[lane] = lm[lane];
                tc.sync();
                continue;
            }
            // swap rows piv <-> j+1 (relabel) and columns piv <-> j+1 (own elements)
            if (lane < S) lmn[lane] = lane == j + 1 ? plane : (lane == piv ? l_j1 : lm[lane]);
            if (myrow == piv) myrow = j + 1;
            else if (myrow == j + 1) myrow = piv;
            cd acc = lane < S ? H[(j + 1) * LD + lane] : mk(0.0, 0.0);  // my h[.][j+1]
            if (piv != j + 1 && lane < S) {
                const cd xb = H[piv * LD + lane];
                H[piv * LD + lane] = acc;
                acc = xb;
            }
            const int lp = plane;  // lane of the pivot row (logical j+1)
            const cd p = team_bcast<W>(tc, RED, x, lp);          // h[j+1][j]
            cd P = team_bcast<W>(tc, RED, acc, lp);              // h[j+1][j+1]
            const bool elim = myrow >= j + 2 && myrow < S;
            const cd mu = elim ? m_div(x, p) : mk(0.0, 0.0);    // h[i][j] / p
            const bool mnz = elim && m_nz(mu);
            if (elim) MU[myrow] = mu;
            tc.sync();
            const cd* prow = H + lp;  // the pivot row in place: h[j+1][i] = prow[i*LD]
#pragma unroll kMirrorHsUnroll
            for (int i = j + 2; i < S; ++i) {
                const cd mi = MU[i];
                const cd hri = lane < S ? H[i * LD + lane] : mk(0.0, 0.0);
                const cd pri = prow[i * LD];
                // deferred row operation of my row on column i (applied at iteration myrow)
                const cd xn = mnz ? m_sub(hri, m_mul(mu, pri)) : hri;
                if (m_nz(mi)) {
                    // row op on column j+1 (lane myrow == i): computed by every lane and
                    // selected, so no divergent region (same IEEE result for that lane)
                    const cd ra = m_sub(acc, m_mul(mu, P));
                    if (myrow == i) acc = ra;
                    const cd v = (elim && myrow <= i) ? xn : hri;
                    acc = m_add(acc, m_mul(mi, v));                   // column op
                    P = m_add(P, m_mul(mi, pri));                     // pivot row's column op
                }
                if (mnz) H[i * LD + lane] = xn;
            }
            if (lane < S) H[(j + 1) * LD + lane] = acc;
            tc.sync();
        }
        const int* lmf = LM0 + ((S - 2) & 1) * S;  // final logical row -> lane
        // pack the reduced (upper Hessenberg) form in place: logical row i, columns
        // c >= i-1.  Column c's packed slot ends below its own source and overlaps only
        // the sources of columns < c, which are read already (c(c+3)/2 + c + 2 <= c(S+1)
        // for S <= 52; larger S pack into a separate region).
        cd* HSp = ws + L::HS;
#pragma unroll 1
        for (int c = 0; c < S; ++c) {
            const bool on = lane < S && lane <= c + 1;
            const cd v = on ? H[c * LD + lmf[lane]] : mk(0.0, 0.0);
            tc.sync();
            if (on) HSp[(c * (c + 3)) / 2 + lane] = v;
        }
        tc.sync();
        auto h = [&](int i, int c) -> cd { return HSp[(c * (c + 3)) / 2 + i]; };
        // P_m[d] for d < m (m >= 1; slot of column m-2, P_1 in its own cell)
        auto pslot = [&](int m) -> cd* { return m >= 2 ? HSp + ((m - 2) * (m + 1)) / 2 : ws + L::P1; };
        cd* Af = ws + L::A;
        HT_MARK(1);
        // ------------------------------------------------ charpoly (_numba.py:203-225)
        // (1) coefficient chains: lane k-1 walks prod/coef of P_k, i = k-1 .. 1; coef_{k,i}
        //     replaces h(i-1, k-1) (read only by this lane; the chains read subdiagonals)
        if (lane < S) {
            const int k = lane + 1;
            cd prod = mk(1.0, 0.0);
            int stop = k;
            for (int i = k - 1; i > 0; --i) {
                prod = m_mul(prod, h(i, i - 1));
                if (!m_nz(prod)) break;
                cd* cp = HSp + ((k - 1) * (k + 2)) / 2 + (i - 1);
                *cp = m_mul(*cp, prod);
                stop = i;
            }
            STOP[k] = stop;
        }
        tc.sync();
        // (2) P_k over k; lane d owns coefficient d
        for (int k = 1; k <= S; ++k) {
            const cd hk = h(k - 1, k - 1);
            const cd* Pk1 = pslot(k >= 2 ? k - 1 : 1);  // P_{k-1}[d], d < k-1 (unused for k = 1)
            cd* Pk = k < S ? pslot(k) : Af;
            const int stop = STOP[k];
            const cd* coefs = HSp + ((k - 1) * (k + 2)) / 2;  // coef_{k,i} at i-1
            for (int d = lane; d <= k; d += W) {
                // P_{k-1}[e] with the implicit leading 1 (P_0 = 1)
                auto pk1 = [&](int e) -> cd { return e == k - 1 ? mk(1.0, 0.0) : Pk1[e]; };
                cd v;
                if (d == k) {
                    v = mk(1.0, 0.0);  // P_{k-1}[k-1]
                } else {
                    const cd base0 = d >= 1 ? pk1(d - 1) : mk(0.0, 0.0);
                    v = m_sub(base0, m_mul(hk, pk1(d)));
                }
#pragma unroll kMirrorCpUnroll
                for (int i = k - 1; i >= stop && i > 0; --i) {
                    const cd coef = coefs[i - 1];
                    // every lane computes, d < i selects (no divergent region; the read for
                    // d >= i - 1 is replaced by the implicit 1 or lands on a finite entry of
                    // the shared table and is discarded)
                    const cd* pim = pslot(i >= 2 ? i - 1 : 1);  // (P_0: only the implicit 1 is used)
                    const cd pv = d == i - 1 ? mk(1.0, 0.0) : pim[d < i ? d : 0];
                    const cd t = m_sub(v, m_mul(coef, pv));
                    if (m_nz(coef) && d < i) v = t;
                }
                if (k == S || d < k) Pk[d] = v;
            }
            tc.sync();
        }
        const cd* a = Af;  // monic charpoly, ascending, a[S] = 1
        HT_MARK(2);
        // ------------------------------------------------ Newton + Cayley-Hamilton (_numba.py:228-250)
        // sequential; every lane replays it (lane 0 stores)
        int bad = 0;
        {
            const int K = D, m = S;
            const int kmax = K < m ? K : m;
            for (int k = 1; k <= kmax; ++k) {
                cd acc = m_mul(mk((double)(-k), 0.0), a[m - k]);
                for (int jj = 1; jj < k; ++jj) acc = m_sub(acc, m_mul(a[m - jj], T[k - jj - 1]));
                if (lane == 0) T[k - 1] = acc;
                tc.sync();
            }
            for (int k = m + 1; k <= K; ++k) {
                cd acc = mk(0.0, 0.0);
                for (int jj = 0; jj < m; ++jj) acc = m_sub(acc, m_mul(a[jj], T[k - m + jj - 1]));
                if (lane == 0) T[k - 1] = acc;
                tc.sync();
            }
            for (int k = 0; k < K; ++k)
                if (!m_finite(T[k])) bad = 1;
        }
        // ------------------------------------------------ series (_numba.py:334-347)
        for (int k = lane; k <= D; k += W) {
            cd sk = k == 0 ? mk(0.0, 0.0) : m_rdiv(T[k - 1], r_mul(2.0, (double)k));
            if constexpr (LOOPS) {
                if (k >= 1) sk = m_add(sk, m_rmul(0.5, ELL[k - 1]));
            }
            SSr[k] = sk;
            E[k] = k == 0 ? mk(1.0, 0.0) : mk(0.0, 0.0);
        }
        tc.sync();
        HT_MARK(3);
        // ------------------------------------------------ _exp_top (_numba.py:276-294), Horner
        // Only E[D] is returned, and F[d] reads E[0..d-1]: at step jj the coefficients
        // d > D - jj + 1 never reach E[D], so they are not computed (the ones that are
        // computed are the same operation sequences: bit-identical, half the chain).
        for (int jj = D; jj > 0; --jj) {
            const double inv = INVJ[jj];  // = r_div(1.0, jj)
            const int dmax = D - jj + 1;
            cd f[(kDMax + W) / W];
#pragma unroll
            for (int r = 0; r < (kDMax + W) / W; ++r) {
                const int d = lane + W * r;
                f[r] = mk(0.0, 0.0);
                if (d <= dmax) {
                    cd acc = mk(0.0, 0.0);
                    for (int tt = 1; tt <= d; ++tt) acc = m_add(acc, m_mul(E[d - tt], SSr[tt]));
                    f[r] = m_rmul(inv, acc);
                    if (d == 0) f[r] = m_add(f[r], mk(1.0, 0.0));
                }
            }
            tc.sync();
#pragma unroll
            for (int r = 0; r < (kDMax + W) / W; ++r) {
                const int d = lane + W * r;
                if (d <= dmax) E[d] = f[r];
            }
            tc.sync();
        }
        if (valid && lane == 0) {
            const cd coeff = E[D];
            const bool neg = ((D - M) & 1) != 0;
            terms[ir.out] = bad ? mk(0.0, 0.0) : (neg ? m_neg(coeff) : coeff);
            if (bad) status[ir.out] = 2;  // the buffer is zeroed by the host
        }
        tc.sync();
        HT_MARK(4);
    }
    if (!dyn) break;
    }
}

}  // namespace hafb
