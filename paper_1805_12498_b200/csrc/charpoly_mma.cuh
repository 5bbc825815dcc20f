// charpoly_mma.cuh -- blocked characteristic polynomial of the packed upper-Hessenberg
// form on the FP64 tensor cores (mma.sync.m8n8k4.f64), one warp per subset (FAST).
//
// The reference's leading-minor recurrence (_numba.py:203-225) is
//   P_0 = 1,  P_k(x) = x P_{k-1}(x) - sum_{m=0}^{k-1} C[k][m] P_m(x),
//   C[k][m] = h(m, k-1) * prod_{j=m+1}^{k-1} h(j, j-1)   (C[k][k-1] = h(k-1, k-1)),
// evaluated in term_fast.cuh with lane d owning coefficient d of every P_k.  That
// mapping spends S^2/2 warp steps on S^3/6 useful complex multiply-adds (lane d idles
// while m < d).  Here the k range is cut into blocks of 8; for a block starting at K
// the part of the sum over the OLD polynomials (m < K) is one small complex GEMM
//   T[j][d] = sum_{m<K} C[K+j][m] P_m[d]      (8 x K times K x K, P_m[d] = 0 for d > m)
// run as four real m8n8k4 DMMAs per (k-step, n-tile), skipping the all-zero tiles of
// the triangular P; only the in-block terms (m >= K) stay on the lane-per-coefficient
// recurrence (<= 7 per k instead of k).  The DMMA reaches the FP64 peak from a single
// warp (tools/micro/dmma.cu), so the GEMM part costs a fraction of the issue slots of
// the equivalent DFMA loop.
//
// Shared-memory reuse (no extra allocation):
//   * the C[k][m] replace the Hessenberg entries in place (column k-1 of the packed
//     store, rows 0..k-2; the diagonal and subdiagonal stay) -- one pass, no barriers;
//   * P_m (coefficients 0..m-1; P_m[m] = 1) is stored in the packed slot of column m-2,
//     which is dead once P_{m-1} is built and has exactly m entries; P_1 sits in RED;
//   * T is staged in the pivot-row / multiplier / charpoly-coefficient scratch (dead
//     after the Hessenberg reduction), row stride K+1 (conflict-free fragment stores).
// A tail of R rows after the last full block runs as its own GEMM block only when the
// DMMA work (t(t+1) tiles, t = K/8) is below the DFMA work it replaces (R t); otherwise
// it is merged into the previous block, whose rows past the eighth take their old part
// from a DFMA loop over the stored P_m.
// Exact-arithmetic identity only: results agree with the sequential recurrence to
// rounding (FAST).
#pragma once

#include "cplx.cuh"

namespace hafb {

#ifndef HAFB_CP_MMA
#define HAFB_CP_MMA 1
#endif
// a tail block of at least this many rows always runs as a GEMM block
#ifndef HAFB_CP_TAIL_MIN
#define HAFB_CP_TAIL_MIN 99
#endif

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

// packed upper-Hessenberg index: column c starts at c(c+3)/2
__host__ __device__ constexpr int pk_at(int c, int r) { return (c * (c + 3)) / 2 + r; }

// block plan: blocks start at 0, 8, 16, ...; the tail of R = (S+1) mod 8 rows after
// the last full block is a GEMM block iff t + 1 < R (t = its start / 8), else merged
template <int S>
struct CpPlan {
    static constexpr int NFULL = (S + 1) / 8;
    static constexpr int REM = (S + 1) - 8 * NFULL;
    static constexpr bool TAIL = REM > 0 && NFULL >= 1 && (NFULL + 1 < REM || REM >= HAFB_CP_TAIL_MIN);
    static constexpr int NB = NFULL + (TAIL ? 1 : 0);
    static constexpr int start(int b) { return 8 * b; }
    static constexpr int rows(int b) {
        return b < NFULL - 1 ? 8 : b == NFULL - 1 ? (TAIL ? 8 : 8 + REM) : REM;
    }
    static constexpr int KLAST = 8 * (NB - 1);  // P_m with m >= KLAST stay in registers
    static constexpr int TB_NEED(int b) { return (rows(b) < 8 ? rows(b) : 8) * (start(b) + 1); }
    static constexpr int tb_max() {
        int mx = 0;
        for (int b = 1; b < NB; ++b) mx = TB_NEED(b) > mx ? TB_NEED(b) : mx;
        return mx;
    }
};

// P_m[d] from the in-place store (m < KLAST), with the implicit zeros and the monic 1
template <int S, class L>
__device__ __forceinline__ cd cp_pval(const cd* ws, int m, int d) {
    const int addr = m >= 2 ? L::HS + ((m - 2) * (m + 1)) / 2 + d : L::RED;
    const bool ld = d < m;
    const cd v = ws[ld ? addr : L::HS];
    return mk(ld ? v.re : (d == m ? 1.0 : 0.0), ld ? v.im : 0.0);
}

// Coefficients of P_S into ws[L::A + 0..S] (A[S] = 1).  One full warp (W = 32, S <= 32).
template <int S, class L>
__device__ __forceinline__ void charpoly_mma(cd* ws, const int lane) {
    // lane d owns coefficient d; for S > 32 (the NSX classes) lanes < E = S - 32 also own
    // coefficient 32 + lane (non-zero only in P_k, k >= 32: the last block's rows)
    static_assert(S <= 40, "at most two coefficients per lane");
    constexpr int E = S > 32 ? S - 32 : 0;
    using PL = CpPlan<S>;
    static_assert(PL::tb_max() <= L::RED - L::PR, "T staging exceeds the dead scratch");
    cd* Hs = ws + L::HS;
    cd* TB = ws + L::PR;
    cd* A = ws + L::A;
    HT_DECL
    // ---- in place: C[k][m] = h(m, k-1) * prod_{j=m+1}^{k-1} h(j, j-1), m = lane <= k-2
    {
        // the subdiagonal h(j, j-1) first (independent broadcasts, off the product chain)
        cd bt[S];
        static_for<1, S>([&](auto jj) {
            constexpr int j = decltype(jj)::value;
            bt[j] = Hs[pk_at(j - 1, j)];
            return true;
        });
        cd prodl = mk(1.0, 0.0);
        static_for<2, S + 1>([&](auto kk) {
            constexpr int k = decltype(kk)::value;
            const cd beta = bt[k - 1];
            const bool on = lane <= k - 2;
            const cd np = f_mul(lane == k - 2 ? mk(1.0, 0.0) : prodl, beta);
            prodl = mk(on ? np.re : prodl.re, on ? np.im : prodl.im);
            cd* p = Hs + pk_at(k - 1, on ? lane : 0);
            const cd h = *p;
            const cd c = f_mul(h, prodl);
            if (on) *p = c;
            return true;
        });
        if constexpr (E > 0) {  // rows m = 32 + lane
            cd prodx = mk(1.0, 0.0);
            static_for<34, S + 1>([&](auto kk) {
                constexpr int k = decltype(kk)::value;
                const bool on = lane < E && 32 + lane <= k - 2;
                const cd np = f_mul(32 + lane == k - 2 ? mk(1.0, 0.0) : prodx, bt[k - 1]);
                prodx = mk(on ? np.re : prodx.re, on ? np.im : prodx.im);
                cd* p = Hs + pk_at(k - 1, on ? 32 + lane : 0);
                const cd h = *p;
                const cd c = f_mul(h, prodx);
                if (on) *p = c;
                return true;
            });
        }
    }
    __syncwarp();
    HT_MARK(5);
    const int lm = lane & 3, lr = lane >> 2;
    cd Pprev = mk(0.0, 0.0);  // P_{K-1}[lane] entering a block
    static_for<0, PL::NB>([&](auto bb) {
        constexpr int b = decltype(bb)::value;
        constexpr int K = PL::start(b);
        constexpr int R = PL::rows(b);
        constexpr int M0 = R < 8 ? R : 8;
        constexpr int T = K / 8;  // n-tiles (d < K) and half the k-steps
        // ---- old part of the first M0 rows on the tensor cores
        if constexpr (K > 0) {
            double tre[T][2], tim[T][2];
#pragma unroll
            for (int nt = 0; nt < T; ++nt) tre[nt][0] = tre[nt][1] = tim[nt][0] = tim[nt][1] = 0.0;
            const bool rowok = lr < M0;
            static_for<0, 2 * T>([&](auto kss) {
                constexpr int ks = decltype(kss)::value;
                const int m = 4 * ks + lm;
                const cd a = Hs[pk_at(K + (rowok ? lr : 0) - 1, m)];
                const double are = rowok ? a.re : 0.0, aim = rowok ? a.im : 0.0;
                const double anim = -aim;
                static_for<0, T>([&](auto ntt) {
                    constexpr int nt = decltype(ntt)::value;
                    if constexpr (ks >= 2 * nt) {  // tiles with every d > every m are zero
                        const cd bv = cp_pval<S, L>(ws, m, 8 * nt + lr);
                        dmma884(tre[nt], are, bv.re);
                        dmma884(tre[nt], anim, bv.im);
                        dmma884(tim[nt], are, bv.im);
                        dmma884(tim[nt], aim, bv.re);
                    }
                    return true;
                });
                return true;
            });
            if (rowok) {
#pragma unroll
                for (int nt = 0; nt < T; ++nt) {
                    cd* t = TB + lr * (K + 1) + 8 * nt + 2 * lm;
                    t[0] = mk(tre[nt][0], tim[nt][0]);
                    t[1] = mk(tre[nt][1], tim[nt][1]);
                }
            }
            __syncwarp();
        }
        HT_MARK(6);
        // ---- the block's rows, lane d = coefficient d
        cd Pb[R];
        cd Pb2[E > 0 ? R : 1];  // coefficient 32 + lane (lanes < E)
        static_for<0, R>([&](auto jj) {
            constexpr int j = decltype(jj)::value;
            constexpr int k = K + j;
            if constexpr (k == 0) {
                Pb[0] = mk(lane == 0 ? 1.0 : 0.0, 0.0);
            } else {
                const cd pk1 = j == 0 ? Pprev : Pb[j == 0 ? 0 : j - 1];
                cd acc;
                acc.re = __shfl_up_sync(0xffffffffu, pk1.re, 1);
                acc.im = __shfl_up_sync(0xffffffffu, pk1.im, 1);
                if (lane == 0) acc = mk(0.0, 0.0);
                cd acc2 = mk(0.0, 0.0);
                if constexpr (K > 0) {
                    if constexpr (j < 8) {
                        const cd t = TB[j * (K + 1) + (lane < K ? lane : 0)];
                        acc2 = mk(lane < K ? -t.re : 0.0, lane < K ? -t.im : 0.0);
                    } else {
                        // rows past the eighth of a merged block: old part by DFMA
                        static_for<0, K>([&](auto mm) {
                            constexpr int m = decltype(mm)::value;
                            const cd c = Hs[pk_at(k - 1, m)];
                            const cd p = cp_pval<S, L>(ws, m, lane);
                            if constexpr (m & 1) acc2 = f_cms(acc2, c, p);
                            else acc = f_cms(acc, c, p);
                            return true;
                        });
                    }
                }
                // in-block part, m = K .. k-1 (P_m in registers)
                static_for<K, k>([&](auto mm) {
                    constexpr int m = decltype(mm)::value;
                    const cd c = Hs[pk_at(k - 1, m)];
                    if constexpr (m & 1) acc2 = f_cms(acc2, c, Pb[m - K]);
                    else acc = f_cms(acc, c, Pb[m - K]);
                    return true;
                });
                acc = f_add(acc, acc2);
                Pb[j] = acc;
                if constexpr (k == S) {
                    if (lane < S) A[lane] = acc;
                }
                if constexpr (E > 0) {
                    // P_k[32 + lane]: zero below k = 32; no old part (P_m[d] = 0 for m < K <= 32 <= d)
                    if constexpr (k < 32) {
                        Pb2[j] = mk(0.0, 0.0);
                    } else {
                        const cd pk2 = j == 0 ? mk(0.0, 0.0) : Pb2[j == 0 ? 0 : j - 1];
                        cd q, w31;
                        q.re = __shfl_up_sync(0xffffffffu, pk2.re, 1);
                        q.im = __shfl_up_sync(0xffffffffu, pk2.im, 1);
                        w31.re = __shfl_sync(0xffffffffu, pk1.re, 31);
                        w31.im = __shfl_sync(0xffffffffu, pk1.im, 31);
                        if (lane == 0) q = w31;  // P_{k-1}[31]
                        constexpr int M2 = K > 32 ? K : 32;
                        static_for<M2, k>([&](auto mm) {
                            constexpr int m = decltype(mm)::value;
                            q = f_cms(q, Hs[pk_at(k - 1, m)], Pb2[m - K]);
                            return true;
                        });
                        Pb2[j] = q;
                        if constexpr (k == S) {
                            if (lane < E) A[32 + lane] = q;
                        }
                    }
                }
            }
            return true;
        });
        // store the block's P_k for the later blocks' GEMMs (column k-2 is dead by now);
        // after the rows, so no store sits between the rows' shared-memory loads
        if constexpr (K < PL::KLAST) {
            static_for<0, R>([&](auto jj) {
                constexpr int k = K + decltype(jj)::value;
                if constexpr (k == 1) {
                    if (lane == 0) ws[L::RED] = Pb[1];
                } else if constexpr (k >= 2) {
                    if (lane < k) Hs[((k - 2) * (k + 1)) / 2 + lane] = Pb[k - K];
                }
                return true;
            });
        }
        Pprev = Pb[R - 1];
        __syncwarp();
        HT_MARK(7);
        return true;
    });
    if (lane == 0) A[S] = mk(1.0, 0.0);
    __syncwarp();
}

}  // namespace hafb
