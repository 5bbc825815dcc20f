// term_fast.cuh -- register-resident FAST subset-term kernel (charpoly backend).
//
// One TEAM of W lanes evaluates one pair subset of size S = 2m (W = S rounded
// up to a power of two, 2..64; W = 64 spans two warps).  Lane r of the team
// owns row r of the subset matrix B = X.A_Z in registers, so the two O(S^3)
// parts of the Hessenberg reduction (_numba.py:36-67) are lane-local:
//   rank-1 row update  h[i,k] -= mu_i h[p,k]     (pivot row broadcast from smem)
//   column gemv        h[k,p] += sum_i mu_i h[k,i] (mu broadcast from smem)
// and they are fused into one pass over the columns with FMA-contracted
// complex multiply-adds.  Exact-arithmetic identities used (results agree with
// the reference to rounding, not bit for bit -- MIRROR mode is term_smem.cuh):
//   * L^{-1} H L is applied as (L^{-1} H) L instead of interleaving each i;
//   * pivot choice by |re|+|im| (the reference uses hypot);
//   * the row swap of the pivoting is a relabelling of which lane holds which
//     logical row (no data movement); the column swap is a register swap;
//   * Newton's identities and the exp-series coefficient use the O(D^2)
//     recurrences (e' = s' e), parallel over the coefficient index;
//   * the charpoly leading-minor recurrence (_numba.py:203-225) is evaluated
//     with lane d owning coefficient d of every P_k.
// Columns retire into shared memory as the reduction advances (column j is
// final after step j), so the register window shifts left every two steps and
// the step body has static register indices without unrolling over j.
#pragma once

#include <type_traits>

#include "cplx.cuh"
#include "enumerate.cuh"

namespace hafb {

// Compile-time loop: f(std::integral_constant<int, I>) for I = B, B+STEP, ... < E,
// stopping early when f returns false.  Guarantees static register indices
// (a #pragma unroll loop with an early exit is not always fully unrolled, and a
// partially unrolled register array is demoted to local memory).
template <int I>
using ic = std::integral_constant<int, I>;

template <int B, int E, int STEP = 1, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        if (f(ic<B>{})) static_for<B + STEP, E, STEP>(f);
    }
}

#ifdef HAFB_TIMING
__device__ unsigned long long g_phase[16];
__device__ unsigned long long g_phase_cnt[16];
#define HT_DECL long long ht_prev = clock64();
#define HT_MARK(k)                                                    \
    do {                                                              \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                    \
            long long ht_now = clock64();                             \
            atomicAdd(&g_phase[k], (unsigned long long)(ht_now - ht_prev)); \
            atomicAdd(&g_phase_cnt[k], 1ull);                         \
            ht_prev = ht_now;                                         \
        }                                                             \
    } while (0)
#else
#define HT_DECL
#define HT_MARK(k)
#endif

template <int S>
struct TeamWidth {
    static constexpr int W = S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : S <= 32 ? 32 : 64;
};

constexpr int kFastThreads = 128;
constexpr int kGroup = 2;
// threshold partial pivoting: the natural pivot is kept when |h[J+1][J]| >= tau * max
// (|multipliers| <= 1/tau); 1.0 = classic partial pivoting
#ifndef HAFB_PIVOT_TAU
#define HAFB_PIVOT_TAU 1.0f
#endif
constexpr float kPivotThreshold = HAFB_PIVOT_TAU;  // columns per uniform branch in the Hessenberg sweep
constexpr int kDMax = 32;  // D = n/2 <= 32
// doubles reserved for the 1/k table in front of the staged Atilde: an even count keeps
// Atilde 16-byte aligned (an 8-byte-aligned complex array loses LDS.128 and, at S = 28,
// cost 300 B of register spills and 13 % of the step)
constexpr int kInvSlots = (kDMax + 2) & ~1;
#ifndef HAFB_SHFL_PIVOT
#define HAFB_SHFL_PIVOT 1
#endif
// static-column ("no shift") Hessenberg for the register classes (ns_hessenberg)
#ifndef HAFB_NS
#define HAFB_NS 1
#endif
#ifndef HAFB_NS_LO
#define HAFB_NS_LO 10
#endif
#ifndef NS_SPECINV
#define NS_SPECINV 1
#endif
#ifndef NS_HIKEY
#define NS_HIKEY 1
#endif
#ifndef NS_BRANCHLESS
#define NS_BRANCHLESS 1
#endif
#ifndef HAFB_PSYNC
#define HAFB_PSYNC 1
#endif
#ifndef HAFB_QSERIES
#define HAFB_QSERIES 1
#endif
#ifndef HAFB_QS_FOLD
#define HAFB_QS_FOLD 0
#endif
#ifndef HAFB_NS_HI
#define HAFB_NS_HI 32
#endif
constexpr bool ns_variant(int S) { return HAFB_NS && S >= HAFB_NS_LO && S <= HAFB_NS_HI; }

// packed upper-Hessenberg storage, column-major: column c holds rows 0..min(c+1, S-1)
// and starts at c(c+3)/2.
__host__ __device__ constexpr int hs_elems(int S) { return (S - 1) * (S + 2) / 2 + S; }

template <int S, bool SH = false, bool LOOPS = true>
struct FastLayout {
    static constexpr int HS = 0;                      // packed Hessenberg, or (SH) the S x S matrix
    static constexpr int SP = S + 12;                  // padded pivot-row / multiplier length
    static constexpr int PR = HS + (SH ? S * S : hs_elems(S));  // [2][SP] pivot rows (register variant)
    // [2][SP] multipliers (the window variant for S >= 26 shuffles the pivot row: no PR)
    // S = 28 (static-column kernel, one pivot-row and one multiplier buffer): single
    // buffers, so 16 teams and the staged Atilde of n <= 56 fit one SM's shared memory
    static constexpr bool TRIM = !SH && S == 28 && HAFB_NS;
    // S = 34, 36 (NSX with split rows, 12 teams): one pivot-row buffer; the second multiplier
    // buffer stays (the tensor-core charpoly stages T in this scratch and needs the room)
    static constexpr bool TRIM_PR = TRIM || (!SH && !LOOPS && (S == 34 || S == 36) && HAFB_NS);
    static constexpr int MU = PR + ((SH || (HAFB_SHFL_PIVOT && S >= 26 && !HAFB_NS)) ? 0 : TRIM_PR ? SP : 2 * SP);
    static constexpr int CF = MU + (TRIM ? SP : 2 * SP);  // [2][S] charpoly coefs
    static constexpr int RED = CF + 2 * S;            // [2][2][2] argmax exchange (W = 64)
    static constexpr int A = RED + 8;                 // [S+1] charpoly coefficients
    static constexpr int U = A + S + 1;               // [2][S] loop-chain vector (LOOPS)
    static constexpr int PX = U + (LOOPS ? 2 * S : 0);  // [S] cross-warp exchange (W = 64)
    static constexpr int T = PX + ((S > 32 && (SH || LOOPS)) ? S : 4);  // [kDMax+2] traces / exp broadcast (PX: two-warp teams only)
    static constexpr int G = T + kDMax + 2;           // [kDMax+2] g_j = j s_j
    static constexpr int FLAG = G + kDMax + 2;        // [1]
    static constexpr int SIGN = (S + 3) / 4 + 1;      // cd slots holding S ints
    static constexpr int SIG = FLAG + 2;              // [2][S] int: logical row -> lane (SH)
    static constexpr int CRN = SIG + (SH ? 2 * SIGN : 0);  // NSX: the extra rows' columns >= 32 ([E][E])
    static constexpr int TOTAL = CRN + (S > 32 ? (S - 32) * (S - 32) : 0);
};

template <int W>
struct TeamCtx {
    int lane;  // rank within the team
    int tib;   // team index within the block
    unsigned wmask;
    __device__ __forceinline__ void sync() const {
        if constexpr (W <= 32) {
            __syncwarp(wmask);
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + tib), "r"(W) : "memory");
        }
    }
};

template <int W>
__device__ __forceinline__ bool lane_is(const TeamCtx<W>& tc, int r) {
    return tc.lane == r;
}

template <int W>
__device__ __forceinline__ double tshfl_xor(double v, int off) {
    return __shfl_xor_sync(0xffffffffu, v, off, W < 32 ? W : 32);
}
template <int W>
__device__ __forceinline__ int tshfl_xor(int v, int off) {
    return __shfl_xor_sync(0xffffffffu, v, off, W < 32 ? W : 32);
}
template <int W>
__device__ __forceinline__ double tshfl(double v, int src) {
    return __shfl_sync(0xffffffffu, v, src, W < 32 ? W : 32);
}
template <int W>
__device__ __forceinline__ double tshfl_up(double v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d, W < 32 ? W : 32);
}

__device__ __forceinline__ cd f_add(cd a, cd b) { return mk(a.re + b.re, a.im + b.im); }
// 1/d for finite d > 0: hardware reciprocal estimate + two Newton steps (full
// double precision without the IEEE division's special-case path)
__device__ __forceinline__ double f_rcp(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ cd f_inv(cd p) {
    const double r = f_rcp(fma(p.re, p.re, p.im * p.im));
    return mk(p.re * r, -p.im * r);
}

// team argmax over (key, row): larger key wins, ties -> smaller row; returns the
// winner's key, row and its column-j value p.
template <int W>
__device__ __forceinline__ void team_argmax(const TeamCtx<W>& tc, cd* red, double& key, int& row,
                                            cd& pv) {
    constexpr int WW = W < 32 ? W : 32;
#pragma unroll
    for (int off = WW / 2; off > 0; off >>= 1) {
        double ok = tshfl_xor<W>(key, off);
        int orow = tshfl_xor<W>(row, off);
        double opr = tshfl_xor<W>(pv.re, off);
        double opi = tshfl_xor<W>(pv.im, off);
        if (ok > key || (ok == key && orow < row)) {
            key = ok;
            row = orow;
            pv = mk(opr, opi);
        }
    }
    if constexpr (W > 32) {
        const int w = tc.lane >> 5;
        if ((tc.lane & 31) == 0) {
            red[2 * w] = mk(key, (double)row);
            red[2 * w + 1] = pv;
        }
        tc.sync();
        cd a0 = red[0], p0 = red[1], a1 = red[2], p1 = red[3];
        if (a1.re > a0.re || (a1.re == a0.re && a1.im < a0.im)) {
            a0 = a1;
            p0 = p1;
        }
        key = a0.re;
        row = (int)a0.im;
        pv = p0;
    }
}

// Register moves that the compiler may not if-convert into selects: with them the
// column swap below stays a short uniform branch tree (~5 compares + 8 moves)
// instead of an 8-FSEL-per-candidate select chain.
__device__ __forceinline__ void vmov(double& d, double s) {
    asm volatile("mov.b64 %0, %1;" : "=d"(d) : "d"(s));
}

// swap hr[A] <-> hr[b] for a team-uniform runtime b in [LO, HI) (binary branch tree)
template <int S, int LO, int HI>
__device__ __forceinline__ void swap_bs(cd (&hr)[S], int A, int b) {
    if constexpr (HI - LO == 1) {
        const cd t = hr[A];
        vmov(hr[A].re, hr[LO].re);
        vmov(hr[A].im, hr[LO].im);
        vmov(hr[LO].re, t.re);
        vmov(hr[LO].im, t.im);
    } else if constexpr (HI > LO) {
        constexpr int MID = (LO + HI) / 2;
        if (b < MID) swap_bs<S, LO, MID>(hr, A, b);
        else swap_bs<S, MID, HI>(hr, A, b);
    }
}

// Team argmax of a nonnegative pivot key: the key is rounded to float, its low 6
// mantissa bits replaced by (63 - lane) and the packed words max-reduced with one
// redux.sync per warp.  Returns the winning lane (ties -> lowest lane) and the
// winning float key bits (0 if every key is 0).
template <int W>
__device__ __forceinline__ int team_argmax_lane(const TeamCtx<W>& tc, cd* red, double key,
                                                unsigned& kbits) {
    const unsigned kb = key > 0.0 ? __float_as_uint(__double2float_ru(key)) : 0u;
    unsigned packed = (kb & ~63u) | (unsigned)(63 - tc.lane);
    unsigned mx;
    if constexpr (W <= 32) {
        mx = __reduce_max_sync(tc.wmask, packed);
    } else {
        mx = __reduce_max_sync(0xffffffffu, packed);
        unsigned* r = reinterpret_cast<unsigned*>(red);
        if ((tc.lane & 31) == 0) r[tc.lane >> 5] = mx;
        tc.sync();
        const unsigned a0 = r[0], a1 = r[1];
        mx = a0 > a1 ? a0 : a1;
    }
    kbits = mx & ~63u;
    return 63 - (int)(mx & 63u);
}

// One Hessenberg step J = J0 + OFF on the shifting register window w[c] = logical
// column J0 + c of the lane's row (positions c < live = S - J0 are live).
template <int S, int W, int OFF>
__device__ __forceinline__ void fast_hess_step(cd (&w)[S], const int J0, int& myrow,
                                               const TeamCtx<W>& tc, cd* ws) {
    using L = FastLayout<S>;
    cd* Hs = ws + L::HS;
    HT_DECL
    const int J = J0 + OFF;
    const int live = S - J0;
    const cd hj = w[OFF];
    const double key = (myrow > J && myrow < S) ? fabs(hj.re) + fabs(hj.im) : 0.0;
    unsigned kbits;
    int wl = team_argmax_lane<W>(tc, ws + L::RED + 4 * OFF, key, kbits);
    if constexpr (kPivotThreshold < 1.0f && W <= 32) {
        // threshold pivoting: keep the natural pivot row J+1 when its key is within
        // kPivotThreshold of the column maximum (no column swap needed then)
        const unsigned nb = __reduce_max_sync(
            tc.wmask, myrow == J + 1 ? __float_as_uint(__double2float_ru(key)) : 0u);
        const unsigned nat_lane = __reduce_max_sync(tc.wmask, myrow == J + 1 ? (unsigned)tc.lane : 0u);
        if (kbits != 0u && __uint_as_float(nb) >= kPivotThreshold * __uint_as_float(kbits))
            wl = (int)nat_lane;
    }
    HT_MARK(8);
    const int CS = (J * (J + 3)) / 2;  // start of column J in the packed store
    if (kbits == 0u) {  // nothing to eliminate below the subdiagonal
        if (myrow <= J + 1) Hs[CS + myrow] = hj;
        return;
    }
    int brow;
    cd p;
    if constexpr (W <= 32) {
        const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + wl;
        brow = __shfl_sync(tc.wmask, myrow, src);
        p.re = __shfl_sync(tc.wmask, hj.re, src);
        p.im = __shfl_sync(tc.wmask, hj.im, src);
    } else {
        cd* r = ws + L::RED + 4 * OFF + 2;
        if (tc.lane == wl) {
            r[0] = hj;
            r[1] = mk((double)myrow, 0.0);
        }
        tc.sync();
        p = r[0];
        brow = (int)r[1].re;
    }
    // the reciprocal's dependent DFMA chain is issued before the relabel and the column
    // swap's branch tree, which then run under its latency
    const cd ip = f_inv(p);
    HT_MARK(5);
    HT_MARK(13);
    if (myrow == brow) myrow = J + 1;
    else if (myrow == J + 1) myrow = brow;
    if (myrow <= J + 1) Hs[CS + myrow] = hj;
    HT_MARK(6);
    if (brow != J + 1) swap_bs<S, OFF + 2, S>(w, OFF + 1, brow - J0);
    HT_MARK(9);
    const bool elim = myrow >= J + 2 && myrow < S;
    const cd mu = elim ? f_mul(hj, ip) : mk(0.0, 0.0);
    HT_MARK(7);
    if constexpr (HAFB_SHFL_PIVOT && S >= 26) {
        // the pivot row stays in the pivot lane's registers: every lane reads its entries
        // with register shuffles inside the sweep (no serial publish through shared memory)
        cd* mus = ws + L::MU + OFF * L::SP;
        if (myrow == J + 1) {
#pragma unroll
            for (int z = 0; z < kGroup; ++z) mus[live + z] = mk(0.0, 0.0);  // pipelined over-read
        }
        if (elim) mus[myrow - J0] = mu;
        tc.sync();
        HT_MARK(10);
        const int psrc = ((int)(threadIdx.x & 31) & ~(W - 1)) + wl;
        auto pbc = [&](const cd& v) -> cd {
            cd r;
            r.re = __shfl_sync(tc.wmask, v.re, psrc);
            r.im = __shfl_sync(tc.wmask, v.im, psrc);
            return r;
        };
        const cd hj1 = f_cms(w[OFF + 1], mu, pbc(w[OFF + 1]));
        cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
        static_assert(kGroup == 2, "the pipelined sweep is written for pairs");
        cd ma = mus[OFF + 2], mb = mus[OFF + 3];
        static_for<OFF + 2, S, 2>([&](auto gg) {
            constexpr int c = decltype(gg)::value;
            if (c < live) {
                const cd ma2 = mus[c + 2], mb2 = mus[c + 3];
                const cd pa = pbc(w[c]);
                w[c] = f_cms(w[c], mu, pa);
                acc0 = f_cma(acc0, ma, w[c]);
                if constexpr (c + 1 < S) {
                    const cd pb = pbc(w[c + 1]);
                    w[c + 1] = f_cms(w[c + 1], mu, pb);
                    acc1 = f_cma(acc1, mb, w[c + 1]);
                }
                ma = ma2;
                mb = mb2;
            }
            return true;
        });
        w[OFF + 1] = f_add(hj1, f_add(acc0, acc1));
    } else {
        cd* pr = ws + L::PR + OFF * L::SP;
        cd* mus = ws + L::MU + OFF * L::SP;
        if (myrow == J + 1) {
            pr[OFF + 1] = w[OFF + 1];
            static_for<OFF + 2, S, kGroup>([&](auto gg) {
                constexpr int c0 = decltype(gg)::value;
                if (c0 < live) {
                    static_for<c0, (c0 + kGroup < S ? c0 + kGroup : S)>([&](auto c) {
                        pr[c()] = w[c()];
                        return true;
                    });
                }
                return true;
            });
#pragma unroll
            for (int z = 0; z < kGroup; ++z) {  // zero padding past the live edge
                pr[live + z] = mk(0.0, 0.0);
                mus[live + z] = mk(0.0, 0.0);
            }
        }
        if (elim) mus[myrow - J0] = mu;
        tc.sync();
        HT_MARK(10);
        const cd hj1 = f_cms(w[OFF + 1], mu, pr[OFF + 1]);
        cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
        // pairs of columns under one uniform guard; the next pair's broadcasts are
        // loaded before the current pair's multiply-adds (software pipelining across
        // the guard; the padded buffers make the over-read harmless)
        static_assert(kGroup == 2, "the pipelined sweep is written for pairs");
        cd pa = pr[OFF + 2], ma = mus[OFF + 2], pb = pr[OFF + 3], mb = mus[OFF + 3];
        static_for<OFF + 2, S, 2>([&](auto gg) {
            constexpr int c = decltype(gg)::value;
            if (c < live) {
                const cd pa2 = pr[c + 2], ma2 = mus[c + 2], pb2 = pr[c + 3], mb2 = mus[c + 3];
                w[c] = f_cms(w[c], mu, pa);
                acc0 = f_cma(acc0, ma, w[c]);
                if constexpr (c + 1 < S) {
                    w[c + 1] = f_cms(w[c + 1], mu, pb);
                    acc1 = f_cma(acc1, mb, w[c + 1]);
                }
                pa = pa2;
                ma = ma2;
                pb = pb2;
                mb = mb2;
            }
            return true;
        });
        w[OFF + 1] = f_add(hj1, f_add(acc0, acc1));
    }
    HT_MARK(11);
}

// Hessenberg reduction (_numba.py:36-67) as a ROLLED loop over pairs of steps on a
// shifting register window: at the pair starting at J0, w[c] holds logical column
// J0 + c of the lane's row.  Both steps of the pair use static register offsets
// (0 and 1); trailing columns run in groups under a warp-uniform guard against
// the live edge; the window shifts left by two per pair.  Every register index is
// static while the code stays two step bodies long (a fully unrolled reduction is
// ~20K instructions and misses in the i-cache).  Rows are relabelled (lane <->
// logical row `myrow`); the pivot column swap is a uniform branch tree.
template <int S, int W>
__device__ __forceinline__ void fast_hessenberg(cd (&w)[S], int& myrow, const TeamCtx<W>& tc,
                                                cd* ws) {
    using L = FastLayout<S>;
#pragma unroll 1
    for (int J0 = 0; J0 < S - 2; J0 += 2) {
        fast_hess_step<S, W, 0>(w, J0, myrow, tc, ws);
        fast_hess_step<S, W, 1>(w, J0, myrow, tc, ws);
        HT_DECL
        const int live = S - J0;
        static_for<0, S - 2>([&](auto c) {
            if (c() + 2 < live) w[c()] = w[c() + 2];
            return true;
        });
        HT_MARK(12);
    }
    // logical columns S-2 and S-1 are now w[0], w[1]
    cd* Hs = ws + L::HS;
    if (myrow < S) {
        Hs[((S - 2) * (S + 1)) / 2 + myrow] = w[0];
        Hs[((S - 1) * (S + 2)) / 2 + myrow] = w[1];
    }
}

// Hessenberg reduction with the subset matrix in SHARED memory (column-major,
// H[c*S + lane] = row `lane`, column c): dynamic column indices are free, so the
// column swap of the pivoting is two loads and two stores per lane, the pivot row
// is read in place (no publish), and the kernel needs few registers (higher
// occupancy hides the per-step serial latency).  Rows are relabelled (lane <->
// logical row); `lm` (logical row -> lane, double-buffered) is kept for the
// charpoly.  Same arithmetic identities as fast_hessenberg.
#ifndef HAFB_SH_REMAP
#define HAFB_SH_REMAP 1
#endif
template <int S, int W, bool LOOPS>
__device__ __forceinline__ void smem_hessenberg(cd* H, int& myrow, const TeamCtx<W>& tc, cd* ws) {
    using L = FastLayout<S, true, LOOPS>;
    const int lane = tc.lane;
    int* lm0 = reinterpret_cast<int*>(ws + L::SIG);
    if (lane < S) lm0[lane] = lane;
    tc.sync();
    cd* mus = ws + L::MU;
#pragma unroll 1
    for (int J = 0; J < S - 2; ++J) {
        const int B = J & 1;
        const int* lm = reinterpret_cast<const int*>(ws + L::SIG + B * L::SIGN);
        int* lm_next = reinterpret_cast<int*>(ws + L::SIG + (1 - B) * L::SIGN);
        HT_DECL
        const cd x = lane < S ? H[J * S + lane] : mk(0.0, 0.0);
        const double key = (myrow > J && myrow < S) ? fabs(x.re) + fabs(x.im) : 0.0;
        unsigned kbits;
        const int wl = team_argmax_lane<W>(tc, ws + L::RED + 4 * B, key, kbits);
        HT_MARK(8);
        if (kbits == 0u) {  // nothing to eliminate below the subdiagonal
            if (lane < S) lm_next[lane] = lm[lane];
            tc.sync();
            continue;
        }
        int brow;
        cd p;
        if constexpr (W <= 32) {
            const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + wl;
            brow = __shfl_sync(tc.wmask, myrow, src);
            p.re = __shfl_sync(tc.wmask, x.re, src);
            p.im = __shfl_sync(tc.wmask, x.im, src);
        } else {
            cd* r = ws + L::RED + 4 * B + 2;
            if (lane == wl) {
                r[0] = x;
                r[1] = mk((double)myrow, 0.0);
            }
            tc.sync();
            p = r[0];
            brow = (int)r[1].re;
        }
        const int lane_j1 = lm[J + 1];
        if (lane < S) lm_next[lane] = lane == J + 1 ? wl : (lane == brow ? lane_j1 : lm[lane]);
        if (myrow == brow) myrow = J + 1;
        else if (myrow == J + 1) myrow = brow;
        cd x1 = lane < S ? H[(J + 1) * S + lane] : mk(0.0, 0.0);
        if (brow != J + 1 && lane < S) {  // column swap J+1 <-> brow (own row)
            const cd xb = H[brow * S + lane];
            H[brow * S + lane] = x1;
            if constexpr (W > 32) H[(J + 1) * S + lane] = xb;  // read back as pv1 below
            x1 = xb;
        }
        HT_MARK(9);
        const cd ip = f_inv(p);
        const bool elim = myrow >= J + 2 && myrow < S;
        const cd mu = elim ? f_mul(x, ip) : mk(0.0, 0.0);
        if (elim) mus[myrow] = mu;
        cd pv1 = mk(0.0, 0.0);  // the pivot row's (swapped) column J+1 entry
        if constexpr (W <= 32) {
            const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + wl;
            pv1.re = __shfl_sync(tc.wmask, x1.re, src);
            pv1.im = __shfl_sync(tc.wmask, x1.im, src);
        }
        tc.sync();
        if constexpr (W > 32) pv1 = H[(J + 1) * S + wl];  // read before column J+1 changes
        HT_MARK(10);
        const cd hj1 = f_cms(x1, mu, pv1);
        cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
        const cd* prow = H + wl;  // the pivot row, read in place
        int c = J + 2;
        if constexpr (W == 64 && HAFB_SH_REMAP) {
            // The second warp holds only E = S - 32 rows: instead of 32 - E idle lanes walking
            // every column, its lanes split the columns -- lane l works on row 32 + l % EP for
            // the columns J + 2 + l / EP (mod G), EP = 8 or 16 row slots, G = 32 / EP column
            // groups -- and the groups' gemv partials meet in a butterfly.  A quarter (half) of
            // the second warp's shared-memory traffic and instructions; same products, the
            // partial sums associate differently (FAST).
            if (lane >= 32) {
                constexpr int E = S - 32, EP = E <= 8 ? 8 : 16, G = 32 / EP;
                const int l = lane - 32, ri = l % EP, g = l / EP;
                const int row = 32 + (ri < E ? ri : 0);
                cd mur;
                mur.re = __shfl_sync(0xffffffffu, mu.re, ri);
                mur.im = __shfl_sync(0xffffffffu, mu.im, ri);
                const bool elr = __shfl_sync(0xffffffffu, (int)elim, ri) != 0 && ri < E;
#pragma unroll 1
                for (int cc = J + 2 + g; cc < S; cc += G) {
                    const cd xa = H[cc * S + row], pa = prow[cc * S], ma = mus[cc];
                    const cd ya = f_cms(xa, mur, pa);
                    if (ri < E) acc0 = f_cma(acc0, ma, ya);
                    if (elr) H[cc * S + row] = ya;
                }
#pragma unroll
                for (int off = EP; off < 32; off <<= 1) {
                    acc0.re += __shfl_xor_sync(0xffffffffu, acc0.re, off);
                    acc0.im += __shfl_xor_sync(0xffffffffu, acc0.im, off);
                }
                c = S;  // the pair loop below is the first warp's
            }
        }
#pragma unroll 1
        for (; c + 1 < S; c += 2) {
            const cd xa = H[c * S + lane], xb = H[(c + 1) * S + lane];
            const cd pa = prow[c * S], pb = prow[(c + 1) * S];
            const cd ma = mus[c], mb = mus[c + 1];
            const cd ya = f_cms(xa, mu, pa), yb = f_cms(xb, mu, pb);
            acc0 = f_cma(acc0, ma, ya);
            acc1 = f_cma(acc1, mb, yb);
            if (elim) {
                H[c * S + lane] = ya;
                H[(c + 1) * S + lane] = yb;
            }
        }
        if (c < S) {
            const cd xa = H[c * S + lane], pa = prow[c * S], ma = mus[c];
            const cd ya = f_cms(xa, mu, pa);
            acc0 = f_cma(acc0, ma, ya);
            if (elim) H[c * S + lane] = ya;
        }
        if constexpr (W > 32) tc.sync();  // everyone has read pv1 before column J+1 changes
        if (lane < S) H[(J + 1) * S + lane] = f_add(hj1, f_add(acc0, acc1));
        HT_MARK(11);
    }
    tc.sync();
}



// ============================================================================ NS variant
// Hessenberg reduction (_numba.py:36-67) with the lane's row at STATIC column indices
// and no register window: the sweep of step J runs from column S-1 DOWN to J+2 and
// leaves at J+2, so dead columns cost nothing; columns J (the pivot column) and J+1
// travel in registers (hj, hn) from one step to the next, so the only dynamic register
// index left is the pivot column swap (one read-modify-write branch tree).  The window
// version moved every live register two places every second step (IMAD.MOV / FSEL:
// ~20 % of the issued instructions at S = 28).  The pivot row is published to shared
// memory by its lane (a broadcast LDS.128 per column instead of four 32-bit shuffles).
// Same exact-arithmetic identities as fast_hessenberg; the gemv sums the columns in
// descending order.

// t = w[b]; w[b] = v  (team-uniform runtime b in [LO, HI))
template <int S, int LO, int HI>
__device__ __forceinline__ void ns_xchg(cd (&w)[S], int b, cd& v) {
    if constexpr (HI - LO == 1) {
        const cd t = w[LO];
        vmov(w[LO].re, v.re);
        vmov(w[LO].im, v.im);
        vmov(v.re, t.re);
        vmov(v.im, t.im);
    } else if constexpr (HI > LO) {
        constexpr int MID = (LO + HI) / 2;
        if (b < MID) ns_xchg<S, LO, MID>(w, b, v);
        else ns_xchg<S, MID, HI>(w, b, v);
    }
}

// v = w[b]
template <int S, int LO, int HI>
__device__ __forceinline__ void ns_read(const cd (&w)[S], int b, cd& v) {
    if constexpr (HI - LO == 1) {
        v = w[LO];
    } else if constexpr (HI > LO) {
        constexpr int MID = (LO + HI) / 2;
        if (b < MID) ns_read<S, LO, MID>(w, b, v);
        else ns_read<S, MID, HI>(w, b, v);
    }
}


// Split rows (K > 2, one-warp teams): logical columns 2..K-1 of every lane row live in
// shared memory (slot [c][lane] at the top of the packed-Hessenberg region) instead of
// registers.  Those columns retire first -- column c leaves the sweep after step c-2 --
// so they carry a small share of the sweep's column-steps (16 % at S = 28, K = 12),
// while the 4(K-2) registers saved per lane lift the class from 12 to 16 warps per SM
// (the register file is the occupancy limit).
template <int S, int K>
struct NsSplit {
    static_assert(K == 2 || (K > 2 && K <= S), "split bound");
    // Hq[c * 32 + lane] for 2 <= c < K
    static constexpr int BASE = hs_elems(S) - (K - 2) * 32 - 2 * 32;
    // the packed column retired at step J (slots J(J+3)/2 .. +J+1) stays below the
    // split columns still live at that step (J+2 .. K-1)
    static constexpr bool disjoint() {
        for (int J = 0; J + 2 < K; ++J)
            if ((J * (J + 3)) / 2 + J + 1 >= BASE + (J + 2) * 32) return false;
        return BASE >= 0;
    }
    static_assert(K == 2 || disjoint(), "split overlaps the packed store");
};

template <int S, int W, int K = 2>
__device__ __forceinline__ void ns_hessenberg(cd (&w)[S], int& myrow, const TeamCtx<W>& tc, cd* ws) {
    static_assert(W == 16 || W == 32 || W == 64, "NS variant: half-warp, one- or two-warp teams");
    static_assert(K == 2 || W == 32, "split rows: one-warp teams");
    // W = 16: two teams per warp (team mask / lane base); their uniform branches may diverge
    const unsigned tm = W < 32 ? tc.wmask : 0xffffffffu;
    const int tb = W < 32 ? ((int)(threadIdx.x & 31) & ~(W - 1)) : 0;
    using L = FastLayout<S>;
    cd* Hs = ws + L::HS;
    cd* pr = ws + L::PR;  // pivot row, by logical column
    cd* mus = ws + L::MU;  // multiplier of each logical row
    const int lane = tc.lane;
    cd* Hq = Hs + NsSplit<S, K>::BASE;  // split columns: Hq[c * 32 + lane], 2 <= c < K
    // hn = logical column b of the lane's row (b >= 2, team-uniform)
    auto col_read = [&](int b, cd& v) {
        if constexpr (K > 2) {
            if (b < K) v = Hq[b * 32 + lane];
            else ns_read<S, K, S>(w, b, v);
        } else {
            ns_read<S, 2, S>(w, b, v);
        }
    };
    cd hj = w[0], hn = w[1];
    HT_DECL
#pragma unroll 1
    for (int J = 0; J < S - 2; ++J) {
        const double key = (myrow > J && myrow < S) ? fabs(hj.re) + fabs(hj.im) : 0.0;
#if NS_SPECINV
        // every candidate inverts its own entry while the argmax is in flight; the
        // winner's reciprocal travels with its value (the inverse leaves the serial chain)
        const cd myinv = f_inv(hj);
#endif
#if NS_HIKEY
        // argmax on the high word of the nonnegative double key (monotone in the key),
        // low 6 bits replaced by (63 - lane): larger key wins, ties -> lowest lane
        const unsigned kb = (unsigned)__double2hiint(key);
#else
        const unsigned kb = key > 0.0 ? __float_as_uint(__double2float_ru(key)) : 0u;
#endif
        unsigned mx = __reduce_max_sync(tm, (kb & ~63u) | (unsigned)(63 - lane));
        int wl = 63 - (int)(mx & 63u);
#if NS_SPECINV
        cd ip;
#endif
        int brow;
        if constexpr (W == 64) {
            // each warp's winner posts (packed key, logical row, reciprocal); one barrier
            const int src = wl & 31;
            const int wrow = __shfl_sync(0xffffffffu, myrow, src);
            cd winv;
            winv.re = __shfl_sync(0xffffffffu, myinv.re, src);
            winv.im = __shfl_sync(0xffffffffu, myinv.im, src);
            cd* R = ws + L::RED + (J & 1) * 4;
            if ((lane & 31) == 0) {
                R[2 * (lane >> 5)] = mk((double)mx, (double)wrow);
                R[2 * (lane >> 5) + 1] = winv;
            }
            tc.sync();
            const cd a0 = R[0], a1 = R[2];
            const bool second = a1.re > a0.re;
            mx = (unsigned)(second ? a1.re : a0.re);
            wl = 63 - (int)(mx & 63u);
            brow = (int)(second ? a1.im : a0.im);
            ip = second ? R[3] : R[1];
        }
        HT_MARK(8);
        const int CS = (J * (J + 3)) / 2;  // column J in the packed store
        if ((mx & ~63u) == 0u) {  // nothing to eliminate below the subdiagonal: no update
            if (myrow <= J + 1) Hs[CS + myrow] = hj;
            hj = hn;
            col_read(J + 2, hn);
            continue;
        }
#if NS_SPECINV
        if constexpr (W <= 32) {
            brow = __shfl_sync(tm, myrow, tb + wl);
            ip.re = __shfl_sync(tm, myinv.re, tb + wl);
            ip.im = __shfl_sync(tm, myinv.im, tb + wl);
        }
#else
        static_assert(W == 32, "the two-warp NS variant needs NS_SPECINV");
        brow = __shfl_sync(0xffffffffu, myrow, wl);
        cd p;
        p.re = __shfl_sync(0xffffffffu, hj.re, wl);
        p.im = __shfl_sync(0xffffffffu, hj.im, wl);
        const cd ip = f_inv(p);
#endif
        if (myrow == brow) myrow = J + 1;
        else if (myrow == J + 1) myrow = brow;
        const bool elim = myrow >= J + 2 && myrow < S;
#if NS_BRANCHLESS
        // selects and predicated stores: no divergent region (BSSY/BSYNC) on the chain
        const cd mprod = f_mul(hj, ip);
        const cd mu = mk(elim ? mprod.re : 0.0, elim ? mprod.im : 0.0);
        if constexpr (S >= W) {
            mus[myrow] = mu;
        } else {
            if (myrow < S) mus[myrow] = mu;
        }
#else
        const cd mu = elim ? f_mul(hj, ip) : mk(0.0, 0.0);
        if (myrow < S) mus[myrow] = mu;
#endif
        if (myrow <= J + 1) Hs[CS + myrow] = hj;
        // column swap J+1 <-> brow: column J+1 is hn, column brow >= J+2 sits at w[brow]
        if (brow != J + 1) {  // (a switch jump table: 6x slower)
            if constexpr (K > 2) {
                if (brow < K) {
                    cd* q = Hq + brow * 32 + lane;
                    const cd t = *q;
                    *q = hn;
                    hn = t;
                } else {
                    ns_xchg<S, K, S>(w, brow, hn);
                }
            } else {
                ns_xchg<S, 2, S>(w, brow, hn);
            }
        }
        // publish the pivot row (logical row J+1): its lane stores columns J+1 .. S-1, one
        // exit test per pair (measured alternatives: stores predicated over every column
        // +10 %; a jump into a straight run of stores +5 %; register shuffles of the pivot
        // row inside the sweep +3-5 %)
#if NS_BRANCHLESS
        {
            // warp-uniform exit test per pair of columns around stores predicated on the
            // pivot lane: no divergent region
            const bool pl = lane == wl;
            static_for<0, S - 2, 2>([&](auto ii) {
                constexpr int c = S - 1 - decltype(ii)::value;
                if constexpr (c >= K) {
                    if (pl) pr[c] = w[c];
                } else {
                    if (pl) pr[c] = Hq[c * 32 + lane];
                }
                if constexpr (c - 1 >= K) {
                    if (c - 1 >= J + 2 && pl) pr[c - 1] = w[c - 1];
                } else {
                    if (c - 1 >= J + 2 && pl) pr[c - 1] = Hq[(c - 1) * 32 + lane];
                }
                if (c - 1 <= J + 2) return false;
                return true;
            });
            if (pl) pr[J + 1] = hn;
        }
#else
        if (lane == wl) {
            static_for<0, S - 2, 2>([&](auto ii) {
                constexpr int c = S - 1 - decltype(ii)::value;
                pr[c] = w[c];
                if (c - 1 >= J + 2) pr[c - 1] = w[c - 1];
                if (c - 1 <= J + 2) return false;
                return true;
            });
            pr[J + 1] = hn;
        }
#endif
        tc.sync();
        HT_MARK(10);
        // sweep, columns S-1 down to J+2: row update fused with the column gemv; at J+2
        // stash the next step's column J+2 and finish column J+1 (the gemv target)
        cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
        cd pa = pr[S - 1], ma = mus[S - 1];
        static_for<0, S - 2>([&](auto ii) {
            constexpr int c = S - 1 - decltype(ii)::value;
            const cd pn = pr[c - 1], mn = mus[c - 1];  // next column's broadcasts (c-1 >= 1)
            cd x;
            if constexpr (c >= K) {
                w[c] = f_cms(w[c], mu, pa);
                x = w[c];
            } else {
                x = f_cms(Hq[c * 32 + lane], mu, pa);
            }
            if constexpr (c & 1) acc1 = f_cma(acc1, ma, x);
            else acc0 = f_cma(acc0, ma, x);
            pa = pn;
            ma = mn;
            if (c == J + 2) {
                hj = f_add(f_cms(hn, mu, pa), f_add(acc0, acc1));  // pa = pr[J+1]
                hn = x;  // (a split column's slot is dead from here on)
                return false;
            }
            if constexpr (c < K) Hq[c * 32 + lane] = x;
            return true;
        });
        HT_MARK(11);
    }
    // logical columns S-2 (hj) and S-1 (hn): every row
    if (myrow < S) {
        Hs[((S - 2) * (S + 1)) / 2 + myrow] = hj;
        Hs[((S - 1) * (S + 2)) / 2 + myrow] = hn;
    }
}


// ============================================================================ NSX variant
// S = 32 + E (E = 2..8): one warp per subset.  Rows 0..31 are lane rows exactly as in
// ns_hessenberg; the E extra rows are held COLUMN-wise: lane l keeps their entries of
// column l in registers, and their E x E corner (columns 32..S-1) lives in shared memory
// (lanes < E update it), so no second warp idles on E rows.  Per step the extra rows
// cost: their pivot candidates (lane J & 31), a shuffle pair (or a corner exchange) for
// the column swap, an E-row rank-1 update + gemv partial per lane, and one butterfly
// all-reduce of the E gemv partials.  Same arithmetic identities as ns_hessenberg.
#ifndef HAFB_NSX
#define HAFB_NSX 1
#endif
#ifndef HAFB_NSX_HI
#define HAFB_NSX_HI 38
#endif
constexpr bool nsx_variant(int S) { return HAFB_NSX && S >= 34 && S <= HAFB_NSX_HI; }


// sum of v[0..E) over the warp into every lane (E <= 8): reduce-scatter + butterfly + gather
template <int E>
__device__ __forceinline__ void nsx_allreduce(cd (&v)[E], int lane) {
    constexpr int P = E <= 1 ? 1 : E <= 2 ? 2 : E <= 4 ? 4 : 8;  // padded length
    constexpr int LG = P == 1 ? 0 : P == 2 ? 1 : P == 4 ? 2 : 3;
    cd x[P];
#pragma unroll
    for (int e = 0; e < P; ++e) x[e] = e < E ? v[e] : mk(0.0, 0.0);
    // level l (off = 16 >> l): keep half h = lane bit; x[0..len/2) <- x[h-half] + partner's
#pragma unroll
    for (int l = 0; l < LG; ++l) {
        const int off = 16 >> l;
        const int len = P >> l, half = len >> 1;
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const cd keep = up ? x[half + i] : x[i];
            const cd send = up ? x[i] : x[half + i];
            cd r;
            r.re = __shfl_xor_sync(0xffffffffu, send.re, off);
            r.im = __shfl_xor_sync(0xffffffffu, send.im, off);
            x[i] = f_add(keep, r);
        }
    }
    // x[0] now holds a partial of element idx = bits of lane at 16, 8, ... (LG bits)
#pragma unroll
    for (int off = 16 >> LG; off > 0; off >>= 1) {
        x[0].re += __shfl_xor_sync(0xffffffffu, x[0].re, off);
        x[0].im += __shfl_xor_sync(0xffffffffu, x[0].im, off);
    }
    // element e's total sits in the lanes whose top LG bits spell e (MSB first = level 0)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        int src = 0;
#pragma unroll
        for (int l = 0; l < LG; ++l)
            if ((e >> (LG - 1 - l)) & 1) src |= 16 >> l;
        v[e].re = __shfl_sync(0xffffffffu, x[0].re, src);
        v[e].im = __shfl_sync(0xffffffffu, x[0].im, src);
    }
}

template <int S, int K = 2>
__device__ __forceinline__ void nsx_hessenberg(cd (&w)[S], cd (&ex)[S - 32], int& myrow,
                                               int (&elab)[S - 32], const TeamCtx<32>& tc, cd* ws) {
    constexpr int E = S - 32;
    using L = FastLayout<S, false, false>;  // NSX runs without loops: the kernel's layout
    cd* Hs = ws + L::HS;
    cd* pr = ws + L::PR;
    cd* mus = ws + L::MU;
    cd* CR = ws + L::CRN;  // CR[e * E + q] = h(32 + e, 32 + q)
    const int lane = tc.lane;
    // split rows (K > 2, as in ns_hessenberg): logical columns 2..K-1 of the lane rows in
    // shared memory, so the class fits 168 registers and 12 teams per SM instead of 8
    cd* Hq = Hs + NsSplit<S, K>::BASE;
    auto col_read = [&](int b, cd& v) {
        if constexpr (K > 2) {
            if (b < K) v = Hq[b * 32 + lane];
            else ns_read<S, K, S>(w, b, v);
        } else {
            ns_read<S, 2, S>(w, b, v);
        }
    };
    cd hj = w[0], hn = w[1];
    __syncwarp();
#pragma unroll 1
    for (int J = 0; J < S - 2; ++J) {
        const int jl = J & 31;
        cd xv[E];  // extra rows' column-J entries (meaningful in lane jl)
        if (J >= 32) {
#pragma unroll
            for (int e = 0; e < E; ++e) xv[e] = CR[e * E + (J - 32)];
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) xv[e] = ex[e];
        }
        const double key = (myrow > J && myrow < S) ? fabs(hj.re) + fabs(hj.im) : 0.0;
        const cd myinv = f_inv(hj);
        unsigned pk = ((unsigned)__double2hiint(key) & ~63u) | (unsigned)(63 - lane);
        const bool pj = lane == jl;  // the lane holding the extra rows' column J
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double kx = (pj && elab[e] > J) ? fabs(xv[e].re) + fabs(xv[e].im) : 0.0;
            const unsigned c = ((unsigned)__double2hiint(kx) & ~63u) | (unsigned)(63 - (32 + e));
            pk = c > pk ? c : pk;
        }
        const unsigned mx = __reduce_max_sync(0xffffffffu, pk);
        const int pw = 63 - (int)(mx & 63u);  // physical pivot row (>= 32: an extra row)
        const int CS = (J * (J + 3)) / 2;
        if ((mx & ~63u) == 0u) {  // nothing to eliminate below the subdiagonal
            if (myrow <= J + 1) Hs[CS + myrow] = hj;
            if (lane == jl) {
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (elab[e] <= J + 1) Hs[CS + elab[e]] = xv[e];
            }
            hj = hn;
            col_read(J + 2, hn);
            continue;
        }
        int brow;
        cd ip;
        if (pw < 32) {
            brow = __shfl_sync(0xffffffffu, myrow, pw);
            ip.re = __shfl_sync(0xffffffffu, myinv.re, pw);
            ip.im = __shfl_sync(0xffffffffu, myinv.im, pw);
        } else {
            cd v = xv[0];
            int lb = elab[0];
#pragma unroll
            for (int e = 1; e < E; ++e)
                if (pw - 32 == e) {
                    v = xv[e];
                    lb = elab[e];
                }
            cd p;
            p.re = __shfl_sync(0xffffffffu, v.re, jl);
            p.im = __shfl_sync(0xffffffffu, v.im, jl);
            ip = f_inv(p);
            brow = lb;
        }
        if (myrow == brow) myrow = J + 1;
        else if (myrow == J + 1) myrow = brow;
#pragma unroll
        for (int e = 0; e < E; ++e) elab[e] = elab[e] == brow ? J + 1 : (elab[e] == J + 1 ? brow : elab[e]);
        // multipliers of every logical row (all S rewritten each step) and column J's store
        const bool elim = myrow >= J + 2 && myrow < S;
        const cd mprod = f_mul(hj, ip);
        const cd mu = mk(elim ? mprod.re : 0.0, elim ? mprod.im : 0.0);
        mus[myrow] = mu;
        if (myrow <= J + 1) Hs[CS + myrow] = hj;
#pragma unroll
        for (int e = 0; e < E; ++e) {  // stores predicated on lane jl (no divergent region)
            const cd xp = f_mul(xv[e], ip);
            const bool ee = elab[e] >= J + 2;
            if (pj) mus[elab[e]] = mk(ee ? xp.re : 0.0, ee ? xp.im : 0.0);
            if (pj && elab[e] <= J + 1) Hs[CS + elab[e]] = xv[e];
        }
        // column swap J+1 <-> brow: lane rows by the register tree; extra rows by a
        // shuffle pair (both columns < 32) or a corner exchange
        if (brow != J + 1) {
            if constexpr (K > 2) {
                if (brow < K) {
                    cd* q = Hq + brow * 32 + lane;
                    const cd t = *q;
                    *q = hn;
                    hn = t;
                } else {
                    ns_xchg<S, K, S>(w, brow, hn);
                }
            } else {
                ns_xchg<S, 2, S>(w, brow, hn);
            }
            const int a = J + 1, b = brow;  // a < b
            if (b < 32) {
                const int src = lane == a ? b : a;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    cd in;
                    in.re = __shfl_sync(0xffffffffu, ex[e].re, src);
                    in.im = __shfl_sync(0xffffffffu, ex[e].im, src);
                    if (lane == a || lane == b) ex[e] = in;
                }
            } else if (a < 32) {
                if (lane == a) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const cd t = ex[e];
                        ex[e] = CR[e * E + (b - 32)];
                        CR[e * E + (b - 32)] = t;
                    }
                }
            } else if (lane == 0) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const cd t = CR[e * E + (a - 32)];
                    CR[e * E + (a - 32)] = CR[e * E + (b - 32)];
                    CR[e * E + (b - 32)] = t;
                }
            }
            __syncwarp();
        }
        // publish the pivot row (logical row J+1) by logical column
        if (pw < 32) {
            const bool pl = lane == pw;
            static_for<0, S - 2, 2>([&](auto ii) {
                constexpr int c = S - 1 - decltype(ii)::value;
                if constexpr (c >= K) {
                    if (pl) pr[c] = w[c];
                } else {
                    if (pl) pr[c] = Hq[c * 32 + lane];
                }
                if constexpr (c - 1 >= K) {
                    if (c - 1 >= J + 2 && pl) pr[c - 1] = w[c - 1];
                } else {
                    if (c - 1 >= J + 2 && pl) pr[c - 1] = Hq[(c - 1) * 32 + lane];
                }
                if (c - 1 <= J + 2) return false;
                return true;
            });
            if (pl) pr[J + 1] = hn;
        } else {
            const int es = pw - 32;
            cd r0 = ex[0];
#pragma unroll
            for (int e = 1; e < E; ++e)
                if (es == e) r0 = ex[e];
            pr[lane] = r0;
            if (lane < E) pr[32 + lane] = CR[es * E + lane];
        }
        __syncwarp();
        cd mue[E];
#pragma unroll
        for (int e = 0; e < E; ++e) mue[e] = mus[elab[e]];
        // lane rows: sweep S-1 .. J+2 as in ns_hessenberg
        cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
        cd pa = pr[S - 1], ma = mus[S - 1];
        static_for<0, S - 2>([&](auto ii) {
            constexpr int c = S - 1 - decltype(ii)::value;
            const cd pn = pr[c - 1], mn = mus[c - 1];
            cd x;
            if constexpr (c >= K) {
                w[c] = f_cms(w[c], mu, pa);
                x = w[c];
            } else {
                x = f_cms(Hq[c * 32 + lane], mu, pa);
            }
            if constexpr (c & 1) acc1 = f_cma(acc1, ma, x);
            else acc0 = f_cma(acc0, ma, x);
            pa = pn;
            ma = mn;
            if (c == J + 2) {
                hj = f_add(f_cms(hn, mu, pa), f_add(acc0, acc1));
                hn = x;  // (a split column's slot is dead from here on)
                return false;
            }
            if constexpr (c < K) Hq[c * 32 + lane] = x;
            return true;
        });
        // extra rows: rank-1 update of my live columns (c >= J+1) and the gemv partials.
        // Finished columns are left alone: the pivot-row buffer holds stale entries there,
        // and a dead entry driven to inf would turn a zero multiplier's product into NaN.
        cd part[E];
#pragma unroll
        for (int e = 0; e < E; ++e) part[e] = mk(0.0, 0.0);
        {
            // selects instead of a divergent region: a finished column keeps its (finite)
            // value and contributes a zero coefficient
            const bool live = lane >= J + 1;
            const cd pc = pr[lane], mc0 = mus[lane];
            const cd mc = mk(live ? mc0.re : 0.0, live ? mc0.im : 0.0);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const cd nv = f_cms(ex[e], mue[e], pc);
                ex[e] = mk(live ? nv.re : ex[e].re, live ? nv.im : ex[e].im);
                part[e] = f_cma(part[e], mc, ex[e]);
            }
        }
        if (lane < E && 32 + lane >= J + 1) {
            const cd pc = pr[32 + lane], mc = mus[32 + lane];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                cd v = CR[e * E + lane];
                v = f_cms(v, mue[e], pc);
                part[e] = f_cma(part[e], mc, v);
                CR[e * E + lane] = v;
            }
        }
        // all-reduce of the E partials: reduce-scatter (each level halves the vector a lane
        // keeps: lanes with bit `off` set keep the upper half), a butterfly over the
        // remaining levels, then every lane fetches the E totals
        nsx_allreduce<E>(part, lane);
        // column J+1 of the extra rows += gemv (its owner: lane J+1, or corner lane J+1-32)
        if (J + 1 < 32) {
            if (lane == J + 1) {
#pragma unroll
                for (int e = 0; e < E; ++e) ex[e] = f_add(ex[e], part[e]);
            }
        } else if (lane == J + 1 - 32) {
#pragma unroll
            for (int e = 0; e < E; ++e) CR[e * E + lane] = f_add(CR[e * E + lane], part[e]);
        }
        __syncwarp();
    }
    // logical columns S-2 and S-1 (both >= 32): every row
    Hs[((S - 2) * (S + 1)) / 2 + myrow] = hj;
    Hs[((S - 1) * (S + 2)) / 2 + myrow] = hn;
    if (lane < E) {
        const int e = lane;
#pragma unroll
        for (int q = E - 2; q < E; ++q) {
            const int c = 32 + q;
            Hs[(c * (c + 3)) / 2 + elab[e]] = CR[e * E + q];
        }
    }
}

// team width of the FAST kernel: NSX sizes (no loops) run one-warp teams
}  // namespace hafb
#include "charpoly_mma.cuh"
#include "qr_fast.cuh"
namespace hafb {

// split-row bound K of the static-column classes (ns_hessenberg): one-warp teams in
// blocks of >= 512 threads (16 teams, <= 128 registers) keep HAFB_NS_KEEP columns
// (K..S-1) of the lane's row in registers, columns 2..K-1 in shared memory
#ifndef HAFB_NS_KEEP
#define HAFB_NS_KEEP 18
#endif
#ifndef HAFB_NS_SPLIT_LO
#define HAFB_NS_SPLIT_LO 24
#endif
#ifndef HAFB_NS_KEEP_SMALL
#define HAFB_NS_KEEP_SMALL 16
#endif
#ifndef HAFB_NS_K12T
#define HAFB_NS_K12T 2
#endif
constexpr int ns_split_k(int S, bool loops, bool sh, int nt) {
    // S = 30, 32 at their 12 teams (384 threads, 168 registers): HAFB_NS_K12T split columns
    // only relieve the register allocation (measured: K = 6 -0.07 %, K = 10 +0.06 % per n = 52
    // step; left off)
    if (ns_variant(S) && !loops && !sh && (S == 30 || S == 32) && nt == 384) return HAFB_NS_K12T;
    // S <= 22 (already 16 teams at 128 registers) would keep HAFB_NS_KEEP_SMALL columns
    // (HAFB_NS_SPLIT_LO = 20): the split there only relieves the register allocation --
    // measured -5 ms per n = 52 step but +2 % on the 4096-matrix n = 24 batch, so it is off
    const int keep = S <= 22 ? HAFB_NS_KEEP_SMALL : HAFB_NS_KEEP;
    return (ns_variant(S) && !loops && !sh && S >= HAFB_NS_SPLIT_LO && S <= 32 && nt >= 512 && S - keep > 2)
               ? S - keep
               : 2;
}

// split-row bound of the NSX classes (nsx_hessenberg) in blocks of 352..384 threads (11-12
// teams, <= 168 registers): columns 2..K-1 of the lane rows in shared memory; 2 = no split
#ifndef HAFB_NSX_K34
#define HAFB_NSX_K34 12
#endif
#ifndef HAFB_NSX_K36
#define HAFB_NSX_K36 20
#endif
#ifndef HAFB_NSX_K38
#define HAFB_NSX_K38 14
#endif
constexpr int nsx_split_k(int S, int nt) {
    // S = 38 stays at 8 teams (its workspace fits 10 at most): a split there only relieves
    // the 255-register allocation
    return S == 38 ? HAFB_NSX_K38 : nt < 320 ? 2 : S == 34 ? HAFB_NSX_K34 : S == 36 ? HAFB_NSX_K36 : 2;
}

template <int S, bool LOOPS, bool SH>
struct FastTeam {
    static constexpr bool NSX = nsx_variant(S) && !LOOPS && !SH;
    static constexpr int W = NSX ? 32 : TeamWidth<S>::W;
};

// SPEC: the spectral backend (qr_fast.cuh: shifted QR on the same packed Hessenberg
// form, power sums) instead of the charpoly; cap_mult bounds its sweeps
// minimum resident blocks per SM the register allocation must allow: the 64-lane
// shared-memory classes (one team per 64-thread block) are latency-bound at the 5 teams
// their ~240 registers leave.  Up to S = 42 shared memory holds 6 teams, so the kernel is
// capped at 168 registers (332 B of spills at S = 40): S = 40..44 at n = 56 571 -> 524 ms.
// 7 blocks (128 registers, 1.3-4 KB of spills) measured slower.
// (the launcher picks the capped instantiation only for classes that fill 6 blocks per SM:
// a class of a few waves is one serial chain per team, and the spills lengthen it)
#ifndef HAFB_SH_MINB
#define HAFB_SH_MINB 6
#endif
constexpr bool sh_capped_ok(int S, bool sh, int nt) { return sh && nt == 64 && S <= 42; }

template <int S, bool LOOPS, bool SH, int NT = kFastThreads, bool SPEC = false, int MINB = 0>
__global__ void __launch_bounds__(NT, MINB) fast_term_kernel(const cd* __restrict__ atilde,
                                                                 const cd* __restrict__ diag,
                                                                 int n_half, ClassItems ci,
                                                                 cd* __restrict__ terms,
                                                                 int8_t* __restrict__ status,
                                                                 int stage_a, int cap_mult) {
    static_assert(!SPEC || !SH, "the FAST spectral backend runs on the packed Hessenberg form");
    constexpr bool NSX = FastTeam<S, LOOPS, SH>::NSX;
    // blocks of more than 128 threads (one block per SM) keep their teams in the same phase
    // (one phase's code in the instruction cache at a time) where that measured faster:
    // the NSX classes (S = 34, 36: -15 %); the static-column classes S <= 32 run 2-3 %
    // faster without the phase barriers
    #ifndef HAFB_PSYNC_NS
#define HAFB_PSYNC_NS 0
#endif
#ifndef HAFB_PSYNC_NSX
#define HAFB_PSYNC_NSX 1
#endif
    constexpr bool PSYNC = NT > kFastThreads && ((NSX && HAFB_PSYNC_NSX) || (HAFB_PSYNC && (!ns_variant(S) || HAFB_PSYNC_NS)));
    constexpr int W = FastTeam<S, LOOPS, SH>::W;
    constexpr int TPB = NT / W;
    constexpr int NSK = NSX ? nsx_split_k(S, NT) : ns_split_k(S, LOOPS, SH, NT);
    constexpr int M = S / 2;
    constexpr int R = (kDMax + W - 1) / W;  // coefficient chunks per lane
    using L = FastLayout<S, SH, LOOPS>;
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
    const int opaque_zero = ci.nseg < 0 ? 1 : 0;  // 0, but unknown to the compiler
    // reciprocals 1/k for the exp recurrence (block-shared, written once)
    double* INV = reinterpret_cast<double*>(smem + (size_t)TPB * L::TOTAL);
    for (int k = threadIdx.x; k <= kDMax; k += blockDim.x) INV[k] = k ? 1.0 / k : 0.0;
    const int n = 2 * n_half;
    const int D = n_half;
    // each team walks a contiguous run of the class's items (successive masks by
    // Gosper's step, ItemCursor); every team runs the same trip count (block-uniform
    // loop for the phase barriers)
    const long long n_teams = (long long)gridDim.x * TPB;
    // Work distribution.  Static: team t walks items [t*chunk, (t+1)*chunk).  Dynamic
    // (one problem, ci.ctr set): blocks take chunks of TPB*ch items from an atomic
    // counter (ch items per team, walked contiguously), so the kernel's tail is one
    // chunk rather than the spread of whole-kernel team times (measured ~5 ms per big
    // class launch: 10 % of a 1/8 shard, 2-3 % of the full step).
    const bool dyn = HAFB_DYN && ci.ctr != nullptr;
    long long ch = (ci.n_items + n_teams - 1) / n_teams;  // static: the whole run
    if (dyn) {
        ch = ci.n_items / (n_teams * HAFB_DYN_PER);  // >= HAFB_DYN_PER chunks per team
        ch = ch < 1 ? 1 : (ch > HAFB_DYN_CHUNK ? HAFB_DYN_CHUNK : ch);
    }
    const long long chunk = ch;
    long long first = ((long long)blockIdx.x * TPB + tc.tib) * chunk;
    // Atilde staged in shared memory (row stride n+1: the lanes' rows fall in distinct
    // banks) for the block's first problem; the subset gathers then read shared memory
    // instead of issuing S scattered global loads per lane
    cd* As = reinterpret_cast<cd*>(INV + kInvSlots);
    const int ldA = n + 1;
    long long staged_problem = -1;
    const long long block_first = (long long)blockIdx.x * TPB * chunk;
    // stage_a == 2 (one problem, no loops): triangular staging.  Atilde = X A with A symmetric
    // satisfies Atilde[r][c] == Atilde[c^1][r^1]; then only A's lower triangle is kept
    // (A[a][b] = Atilde[a^1][b] at As[a(a+1)/2 + b], a >= b): half the bytes, so more teams fit
    // one SM.  Every block verifies the identity bit for bit while it stages; an asymmetric
    // input (never produced by the engines, but legal at the C ABI) is gathered from global
    // memory instead.
    constexpr bool TRI_OK = !LOOPS && !SH && S >= 30;
    const bool tri = TRI_OK && stage_a == 2;
    if (stage_a && (dyn || block_first < ci.n_items)) {  // (static) a block past the last item stages nothing
        staged_problem = dyn ? 0 : block_first / ci.per_problem;
        const cd* src = atilde + staged_problem * ci.at_stride;
        if (tri) {
            int bad = 0;
            for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
                const int r = i / n, c = i % n, a = r ^ 1;
                const cd v = src[i], u = src[(c ^ 1) * n + a];
                bad |= (__double_as_longlong(v.re) != __double_as_longlong(u.re)) |
                       (__double_as_longlong(v.im) != __double_as_longlong(u.im));
                if (a >= c) As[(a * (a + 1)) / 2 + c] = v;
            }
            if (__syncthreads_or(bad)) staged_problem = -1;
        } else {
            for (int i = threadIdx.x; i < n * n; i += blockDim.x) As[(i / n) * ldA + (i % n)] = src[i];
        }
    }
    __syncthreads();
    ItemCursor cur;
#ifdef HAFB_STAGGER
    // experiment: de-phase the warps of an SM so their serial sections overlap others' sweeps
    __nanosleep((unsigned)(((threadIdx.x >> 5) + 4 * (blockIdx.x % 4)) % 16) * HAFB_STAGGER);
#endif

    // the dynamic chunk base travels through the spare slot of the 1/k table
    long long* dyn_base = reinterpret_cast<long long*>(INV + (kInvSlots - 1));
    for (;;) {
    if (dyn) {
        // block-uniform: every team of the block runs the same trip count (phase barriers)
        __syncthreads();
        if (threadIdx.x == 0) *dyn_base = (long long)atomicAdd(ci.ctr, (unsigned long long)(TPB * chunk));
        __syncthreads();
        const long long b0 = *dyn_base;
        if (b0 >= ci.n_items) break;
        first = b0 + (long long)tc.tib * chunk;
        // a batch: re-stage Atilde when the block's chunk starts in another problem
        if (stage_a == 1 && b0 / ci.per_problem != staged_problem) {
            staged_problem = b0 / ci.per_problem;
            const cd* src = atilde + staged_problem * ci.at_stride;
            for (int i = threadIdx.x; i < n * n; i += blockDim.x) As[(i / n) * ldA + (i % n)] = src[i];
            __syncthreads();
        }
    }
    for (long long it = 0; it < chunk; ++it) {
        HT_DECL
        const long long item = first + it;
        const bool valid = item < ci.n_items;
        const ItemRef ir = cursor_item(ci, valid ? item : 0, cur);
        const bool from_smem = ir.problem == staged_problem;
        const cd* at = atilde + ir.problem * ci.at_stride;
        // row-major Atilde entry (r, c) gathered from the staged copy or from global
        // memory (team-uniform choice; each call site is instantiated for both spaces
        // so the loads stay LDS / LDG instead of generic)
        auto gather = [&](auto&& body) {
            if (from_smem) {
                if constexpr (TRI_OK) {
                    if (tri) {
                        body([&](int r, int c) -> cd {
                            const int a = r ^ 1;
                            const int hi = a > c ? a : c, lo = a > c ? c : a;
                            return As[(hi * (hi + 1)) / 2 + lo];
                        });
                        return;
                    }
                }
                body([&](int r, int c) -> cd { return As[r * ldA + c]; });
            } else {
                body([&](int r, int c) -> cd { return at[r * n + c]; });
            }
        };
        const cd* dg = diag + ir.problem * ci.dg_stride;
        // vertex list: vertex c = 2*bit[c/2] + (c&1); every index below is static except
        // the lane's own pair, found with __fns (no dynamically indexed local arrays)
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
        cd hr[S];
        cd* G = ws + L::G;
        // ---------------------------------------------- loop chain (_numba.py:253-273)
        if constexpr (LOOPS) {
            // lane j holds column j of B: B[i][j] = Atilde[v_{j^1}][v_{i^1}]
            const int rj = 2 * mybit + ((lane & 1) ^ 1);
            gather([&](auto&& g) {
                static_for<0, S>([&](auto i) {
                    const int ci1 = 2 * vbit[i() >> 1] + ((i() & 1) ^ 1);
                    hr[i()] = lane < S ? g(rj, ci1) : mk(0.0, 0.0);
                    return true;
                });
            });
            cd u = lane < S ? dg[2 * mybit + (lane & 1)] : mk(0.0, 0.0);
            const cd xv = lane < S ? dg[2 * mybit + ((lane & 1) ^ 1)] : mk(0.0, 0.0);
            cd* U = ws + L::U;
            for (int k = 1; k <= D; ++k) {
                cd l = f_mul(u, xv);
                constexpr int WW = W < 32 ? W : 32;
#pragma unroll
                for (int off = WW / 2; off > 0; off >>= 1) {
                    l.re += tshfl_xor<W>(l.re, off);
                    l.im += tshfl_xor<W>(l.im, off);
                }
                if constexpr (W > 32) {
                    // combine the two warps' partial sums
                    cd* X = ws + L::PX;
                    if ((lane & 31) == 0) X[(k & 1) * 2 + (lane >> 5)] = l;
                    tc.sync();
                    l = f_add(X[(k & 1) * 2], X[(k & 1) * 2 + 1]);
                }
                if (lane == 0) G[k] = l;  // ell_k; folded into g below
                if (k < D) {
                    cd* ub = U + (k & 1) * S;
                    if (lane < S) ub[lane] = u;
                    tc.sync();
                    cd acc0 = mk(0.0, 0.0), acc1 = mk(0.0, 0.0);
                    static_for<0, S>([&](auto i) {
                        if constexpr (decltype(i)::value & 1) acc1 = f_cma(acc1, ub[i()], hr[i()]);
                        else acc0 = f_cma(acc0, ub[i()], hr[i()]);
                        return true;
                    });
                    u = lane < S ? f_add(acc0, acc1) : mk(0.0, 0.0);
                }
            }
        }
        // ---------------------------------------------- gather B rows
        const int vr = 2 * mybit + (lane & 1);
        int myrow = lane;
        if constexpr (SH) {
            cd* H = ws + L::HS;
            gather([&](auto&& g) {
                static_for<0, S>([&](auto c) {
                    const int vc = 2 * vbit[c() >> 1] + (c() & 1);
                    if (lane < S) H[c() * S + lane] = g(vr, vc);
                    return true;
                });
            });
            tc.sync();
            HT_MARK(0);
            smem_hessenberg<S, W, LOOPS>(H, myrow, tc, ws);
        } else if constexpr (NSX) {
            constexpr int E = S - 32;
            cd ex[E > 0 ? E : 1];
            int elab[E > 0 ? E : 1];
            // extra rows 32+e (vertices 2 v_{16+e/2} + (e&1), pair-swapped rows of Atilde):
            // column lane in registers, columns 32+q (q < E) in the shared-memory corner
            const int cb1 = lane < E ? (int)__fns(ir.mask, 0, 16 + (lane >> 1) + 1) : 0;
            cd* CR = ws + L::CRN;
            constexpr int K = NSK;
            cd* Hq = ws + L::HS + NsSplit<S, K>::BASE;
            if constexpr (K > 2) tc.sync();  // the previous subset's readers of the region
            gather([&](auto&& g) {
                static_for<0, S>([&](auto c) {
                    const int vc = 2 * vbit[c() >> 1] + (c() & 1);
                    const cd v = g(vr, vc);
                    if constexpr (c() >= 2 && c() < K) Hq[c() * 32 + lane] = v;
                    else hr[c()] = v;
                    return true;
                });
                static_for<0, E>([&](auto ee) {
                    constexpr int e = decltype(ee)::value;
                    const int rv = 2 * vbit[16 + e / 2] + (e & 1);
                    ex[e] = g(rv, 2 * mybit + (lane & 1));
                    if (lane < E) CR[e * E + lane] = g(rv, 2 * cb1 + (lane & 1));
                    elab[e] = 32 + e;
                    return true;
                });
            });
            HT_MARK(0);
            nsx_hessenberg<S, K>(hr, ex, myrow, elab, tc, ws);
        } else {
            constexpr int K = NSK;
            cd* Hq = ws + L::HS + NsSplit<S, K>::BASE;
            if constexpr (K > 2) tc.sync();  // the previous subset's readers of the region
            gather([&](auto&& g) {
                static_for<0, S>([&](auto c) {
                    const int vc = 2 * vbit[c() >> 1] + (c() & 1);
                    const cd v = lane < S ? g(vr, vc) : mk(0.0, 0.0);
                    if constexpr (c() >= 2 && c() < K) Hq[c() * 32 + lane] = v;
                    else hr[c()] = v;
                    return true;
                });
            });
            HT_MARK(0);
            // ---------------------------------------------- Hessenberg (_numba.py:36-67)
            if constexpr (ns_variant(S)) ns_hessenberg<S, W, K>(hr, myrow, tc, ws);
            else fast_hessenberg<S, W>(hr, myrow, tc, ws);
        }
        HT_MARK(1);
        if constexpr (PSYNC) __syncthreads();
        tc.sync();
        // ---------------------------------------------- charpoly (_numba.py:203-225)
        // one-warp register classes: blocked, the old-polynomial part on the FP64 tensor
        // cores (charpoly_mma.cuh); otherwise lane d owns coefficient d of every P_k
        constexpr bool CPMMA = HAFB_CP_MMA && W == 32 && !SH && S >= 18 && S <= 40;
        bool conv = true;
        if constexpr (SPEC) {
            // ------------------------------------------ eigenvalues + power sums
            // (_numba.py:115-200): traces t_k straight into T[1..D]
            cd* eig = ws + L::A;
            int sweeps = 0;
            conv = q_eigvals<S, W>(ws + L::HS, eig, cap_mult, lane, sweeps, [&] { tc.sync(); });
            if (conv) q_power_sums<S, W>(eig, ws + L::T, D, lane);
            tc.sync();
        } else if constexpr (CPMMA) {
            charpoly_mma<S, L>(ws, lane);
        } else {
            const cd* Hs = ws + L::HS;
            // h(i, c) of the Hessenberg form: packed store, or (SH) the matrix in smem
            // with logical row i in lane lm[i]
            const int* lmf = reinterpret_cast<const int*>(ws + L::SIG + ((S - 2) & 1) * L::SIGN);
            const int my_lm = SH && lane < S ? lmf[lane] : 0;
            auto hget = [&](int i, int c) -> cd {
                if constexpr (SH) return Hs[c * S + lmf[i]];
                else return Hs[(c * (c + 3)) / 2 + i];
            };
            auto hget_mine = [&](int c) -> cd {  // h(lane, c)
                if constexpr (SH) return Hs[c * S + my_lm];
                else return Hs[(c * (c + 3)) / 2 + lane];
            };
            cd* A = ws + L::A;
            cd P[S];
            P[0] = mk(lane == 0 ? 1.0 : 0.0, 0.0);
            cd prodl = mk(1.0, 0.0);
            cd prodx = mk(1.0, 0.0);
            cd Q[NSX ? S - 32 : 1] = {};  // extra coefficients (NSX)
            static_for<1, S + 1>([&](auto kk) {
                constexpr int k = decltype(kk)::value;
                cd* cf = ws + L::CF + (k & 1) * S;
                if constexpr (k >= 2) {
                    const cd beta = hget(k - 1, k - 2);  // h[k-1][k-2]
#if NS_BRANCHLESS
                    {  // select + predicated store: no divergent region per step
                        const bool on = lane <= k - 2;
                        const cd np = f_mul(lane == k - 2 ? mk(1.0, 0.0) : prodl, beta);
                        prodl = mk(on ? np.re : prodl.re, on ? np.im : prodl.im);
                        const cd v = f_mul(hget_mine(k - 1), prodl);
                        if (on) cf[lane] = v;
                    }
#else
                    if (lane <= k - 2) {
                        prodl = f_mul(lane == k - 2 ? mk(1.0, 0.0) : prodl, beta);
                        cf[lane] = f_mul(hget_mine(k - 1), prodl);
                    }
#endif
                    if constexpr (NSX && k >= 34) {  // rows 32 + lane of the extra coefficients
                        if (lane < S - 32 && 32 + lane <= k - 2) {
                            prodx = f_mul(32 + lane == k - 2 ? mk(1.0, 0.0) : prodx, beta);
                            cf[32 + lane] = f_mul(hget(32 + lane, k - 1), prodx);
                        }
                    }
                }
                cd prev;
                if constexpr (W <= 32) {
                    prev.re = tshfl_up<W>(P[k - 1].re, 1);
                    prev.im = tshfl_up<W>(P[k - 1].im, 1);
                } else {
                    cd* X = ws + L::PX;
                    if (lane < S) X[lane] = P[k - 1];
                    tc.sync();
                    prev = lane >= 1 && lane <= S ? X[lane - 1] : mk(0.0, 0.0);
                }
                if (lane == 0) prev = mk(0.0, 0.0);
                tc.sync();
                const cd hk = hget(k - 1, k - 1);
                cd acc = f_cms(prev, hk, P[k - 1]);
                cd acc2 = mk(0.0, 0.0), acc3 = mk(0.0, 0.0), acc4 = mk(0.0, 0.0);
                // chunks of four coefficients; the opaque branch is a basic-block fence
                // that bounds how many broadcast loads the scheduler hoists at once
                static_for<1, k, 4>([&](auto ii) {
                    constexpr int i0 = decltype(ii)::value;
                    if (i0 >= k + opaque_zero) return false;
                    static_for<i0, (i0 + 4 < k ? i0 + 4 : k)>([&](auto jj) {
                        constexpr int i = decltype(jj)::value;
                        if constexpr ((i & 3) == 0) acc = f_cms(acc, cf[i - 1], P[i - 1]);
                        else if constexpr ((i & 3) == 1) acc2 = f_cms(acc2, cf[i - 1], P[i - 1]);
                        else if constexpr ((i & 3) == 2) acc3 = f_cms(acc3, cf[i - 1], P[i - 1]);
                        else acc4 = f_cms(acc4, cf[i - 1], P[i - 1]);
                        return true;
                    });
                    return true;
                });
                acc = f_add(f_add(acc, acc2), f_add(acc3, acc4));
                if constexpr (NSX && k >= 32) {
                    // coefficients 32 + lane (lanes < E) of P_k: Q[t] = P_{32+t}[32+lane]
                    constexpr int t = k - 32;
                    cd pq;
                    pq.re = __shfl_sync(0xffffffffu, P[k - 1].re, 31);
                    pq.im = __shfl_sync(0xffffffffu, P[k - 1].im, 31);
                    if constexpr (t >= 1) {
                        cd up;
                        up.re = __shfl_up_sync(0xffffffffu, Q[t - 1].re, 1);
                        up.im = __shfl_up_sync(0xffffffffu, Q[t - 1].im, 1);
                        if (lane != 0) pq = up;
                    } else {
                        if (lane != 0) pq = mk(0.0, 0.0);
                    }
                    cd q = pq;
                    if constexpr (t >= 1) q = f_cms(q, hk, Q[t - 1]);
                    static_for<32, k - 1>([&](auto ll) {
                        constexpr int l = decltype(ll)::value;
                        q = f_cms(q, cf[l], Q[l - 32]);
                        return true;
                    });
                    if constexpr (k < S) Q[t] = q;
                    else if (lane < S - 32) A[32 + lane] = q;
                }
                if constexpr (k < S) P[k] = acc;
                else if (lane < S) A[lane] = acc;
                return true;
            });
            if (lane == 0) A[S] = mk(1.0, 0.0);
            tc.sync();
        }
        HT_MARK(2);
        if constexpr (PSYNC) __syncthreads();
        // ---------------------------------------------- Newton + Cayley-Hamilton (_numba.py:228-250)
        cd* T = ws + L::T;
        cd* A = ws + L::A;
        int bad = 0;
        cd eD = mk(0.0, 0.0);
        constexpr bool QS = !LOOPS && W <= 32 && HAFB_QSERIES && !SPEC;
        if constexpr (QS) {
            // Without loop weights the series is exp(sum_k t_k x^k / (2k)) = q(x)^(-1/2) with
            // q(x) = det(I - xB) = sum_j a_j x^j, a_j = A[S-j] (the reversed charpoly), so
            // Newton's identities and the exp recurrence (_numba.py:228-250, :276-294)
            // collapse into ONE recurrence from q g' = -(1/2) q' g:
            //   g_0 = 1,  g_k = -(1/k) sum_{j=1}^{min(k,S)} a_j (k - j/2) g_{k-j},
            // evaluated in push form (lane (k-1) % W, chunk (k-1) / W accumulates g_k; each g_m
            // is broadcast once).  Exact in exact arithmetic; a non-finite coefficient or
            // result -> status 2.
            cd acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = mk(0.0, 0.0);
            const int src0 = ((int)(threadIdx.x & 31) & ~(W - 1));
#if HAFB_QS_FOLD
            // the recurrence's serial chain is broadcast -> multiply-add per step: the scale
            // -1/m of g_m and the weight (k+m)/2 are folded into the coefficient a_j off
            // the chain (acc_k += [a_j (k+m)/2 (-1/m)] P_m, with P_m = -m g_m the pushed sum)
            for (int m = 0; m < D; ++m) {
                cd pm;
                if (m == 0) {
                    pm = mk(1.0, 0.0);
                } else {
                    const int chunk = (m - 1) / W;
                    cd v = acc[0];
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        if (r == chunk) v = acc[r];
                    pm.re = __shfl_sync(tc.wmask, v.re, src0 + (m - 1) % W);
                    pm.im = __shfl_sync(tc.wmask, v.im, src0 + (m - 1) % W);
                }
                const double sc = m == 0 ? 1.0 : -INV[m];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    const int j = k - m;
                    const bool on = k <= D && j >= 1 && j <= S;
                    const double wgt = on ? 0.5 * (double)(k + m) * sc : 0.0;
                    const cd aj = A[S - (on ? j : 1)];
                    acc[r] = f_cma(acc[r], mk(wgt * aj.re, wgt * aj.im), pm);
                }
            }
#else
            for (int m = 0; m < D; ++m) {
                cd gm;
                if (m == 0) {
                    gm = mk(1.0, 0.0);
                } else {
                    const int chunk = (m - 1) / W;
                    cd v = acc[0];
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        if (r == chunk) v = acc[r];
                    const double sc = -INV[m];
                    gm.re = __shfl_sync(tc.wmask, v.re, src0 + (m - 1) % W) * sc;
                    gm.im = __shfl_sync(tc.wmask, v.im, src0 + (m - 1) % W) * sc;
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    const int j = k - m;
                    const bool on = k <= D && j >= 1 && j <= S;
                    // zero weight instead of a divergent region (the index is clamped in range)
                    const double wgt = on ? 0.5 * (double)(k + m) : 0.0;
                    acc[r] = f_cma(acc[r], A[S - (on ? j : 1)], mk(wgt * gm.re, wgt * gm.im));
                }
            }
#endif
            for (int i = lane; i <= S; i += W) {
                const cd a = A[i];
                if (!isfinite(a.re) || !isfinite(a.im)) bad = 1;
            }
            {
                const int chunk = (D - 1) / W;
                cd v = acc[0];
#pragma unroll
                for (int r = 1; r < R; ++r)
                    if (r == chunk) v = acc[r];
                eD = mk(-v.re * INV[D], -v.im * INV[D]);
            }
            if (lane == (D - 1) % W && (!isfinite(eD.re) || !isfinite(eD.im))) bad = 1;
            bad = __any_sync(tc.wmask, bad);
        } else {
        if constexpr (!SPEC) {
            cd acck[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = lane + 1 + W * r;
                acck[r] = (k <= D && k <= S) ? mk(-(double)k * A[S - k].re, -(double)k * A[S - k].im)
                                             : mk(0.0, 0.0);
            }
            for (int kk = 1; kk <= D; ++kk) {
                const int owner = (kk - 1) % W, chunk = (kk - 1) / W;
                cd tk;
                if constexpr (W <= 32) {  // register broadcast from the owner lane
                    cd v = acck[0];
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        if (r == chunk) v = acck[r];
                    const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + owner;
                    tk.re = __shfl_sync(tc.wmask, v.re, src);
                    tk.im = __shfl_sync(tc.wmask, v.im, src);
                    if (lane == owner) T[kk] = tk;
                } else {
                    if (lane == owner) {
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (r == chunk) T[kk] = acck[r];
                    }
                    tc.sync();
                    tk = T[kk];
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    const int jj = k - kk;
                    if (k <= D && jj >= 1 && jj <= S) acck[r] = f_cms(acck[r], A[S - jj], tk);
                }
            }
            tc.sync();
        }
        {
            // g_k = k s_k = t_k / 2 (+ k ell_k / 2 with loops)
            for (int k = lane + 1; k <= D; k += W) {
                cd tk = T[k];
                // non-finite traces: status 2 on the charpoly backend; the reference's
                // spectral path has no such check (_numba.py:322-331)
                if (!SPEC && (!isfinite(tk.re) || !isfinite(tk.im))) bad = 1;
                cd g = mk(0.5 * tk.re, 0.5 * tk.im);
                if constexpr (LOOPS) g = mk(fma(0.5 * k, G[k].re, g.re), fma(0.5 * k, G[k].im, g.im));
                G[k] = g;
            }
        }
        HT_MARK(3);
        // any lane saw a non-finite trace -> status 2
        if constexpr (W <= 32) {
            bad = __any_sync(tc.wmask, bad);
        } else {
            if (lane == 0) ws[L::FLAG].re = 0.0;
            tc.sync();
            if (bad) ws[L::FLAG].re = 1.0;
            tc.sync();
            bad = ws[L::FLAG].re != 0.0;
        }
        tc.sync();
        // ---------------------------------------------- exp coefficient: e_k = (1/k) sum_j g_j e_{k-j}
        eD = mk(0.0, 0.0);
        {
            cd acck[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acck[r] = mk(0.0, 0.0);
            for (int kk = 0; kk < D; ++kk) {
                const int owner = (kk - 1 + W) % W, chunk = (kk - 1) / W;
                cd ek;
                if constexpr (W <= 32) {  // register broadcast from the owner lane
                    if (kk == 0) {
                        ek = mk(1.0, 0.0);
                    } else {
                        cd v = acck[0];
#pragma unroll
                        for (int r = 1; r < R; ++r)
                            if (r == chunk) v = acck[r];
                        const int src = ((int)(threadIdx.x & 31) & ~(W - 1)) + owner;
                        const double inv = INV[kk];
                        ek.re = __shfl_sync(tc.wmask, v.re, src) * inv;
                        ek.im = __shfl_sync(tc.wmask, v.im, src) * inv;
                    }
                } else {
                    if (kk == 0) {
                        if (lane == 0) T[0] = mk(1.0, 0.0);
                    } else if (lane == owner) {
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (r == chunk) {
                                const double inv = INV[kk];
                                T[kk] = mk(acck[r].re * inv, acck[r].im * inv);
                            }
                    }
                    tc.sync();
                    ek = T[kk];
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    if (k <= D && k > kk) acck[r] = f_cma(acck[r], G[k - kk], ek);
                }
            }
            const int owner = (D - 1) % W, chunk = (D - 1) / W;
            if (lane == owner) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (r == chunk) eD = mk(acck[r].re * INV[D], acck[r].im * INV[D]);
            }
        }
        }
        if (valid && lane == ((D - 1) % W)) {
            const bool neg = ((D - M) & 1) != 0;
            terms[ir.out] = (bad || !conv) ? mk(0.0, 0.0) : (neg ? mk(-eD.re, -eD.im) : eD);
            // the buffer is zeroed by the host (no scattered byte writes)
            if (bad) status[ir.out] = 2;
            if (!conv) status[ir.out] = 1;  // eigensolver non-convergence (_numba.py:322-324)
        }
        tc.sync();
        HT_MARK(4);
    }
    if (!dyn) break;
    }
}

}  // namespace hafb
