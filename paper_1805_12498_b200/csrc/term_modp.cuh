// term_modp.cuh -- the same subset-sum formula evaluated exactly over GF(p).
//
// For integer matrices the hafnian is an integer that overflows FP64 long before
// the algorithm's reach (cfg3: 3.1e17 > 2^53; the reference's float result is
// 6.8e-7 off, SURVEY.md finding 4).  Every step of the formula is a ring
// operation except the divisions by 2k and k in the series and the exp
// coefficient, which are invertible modulo a prime p > n.  So the per-subset
// term can be computed in GF(p) (p < 2^31): Hessenberg reduction by elementary
// similarities with a first-nonzero pivot, the leading-minor characteristic
// polynomial, Newton / Cayley-Hamilton traces, the loop corrections and the
// exp recurrence e_k = k^-1 sum_j j s_j e_{k-j}.  Summing the terms mod p for a
// few primes and combining by CRT (host side) gives the exact value.
//
// Layout: one team of W lanes per subset (lane r owns row r), the subset matrix in
// shared memory as 32-bit residues; the per-team term sum is accumulated in a
// register and added to the launch total with one 64-bit atomic (residues < 2^31,
// at most 2^31 terms: no overflow).
#pragma once

#include <stdint.h>

#include "enumerate.cuh"
#include "term_fast.cuh"

namespace hafb {

// Montgomery arithmetic modulo an odd p < 2^31 with R = 2^32: residues are kept
// as x R mod p (the host uploads them in that form), a product is one 32x32->64
// multiply plus one REDC (two more multiplies), and a sum of two products
// (< 2 p^2 < p R) needs a single REDC ("lazy" accumulation).
struct ModP {
    uint32_t p;
    uint32_t nq;   // -p^-1 mod 2^32
    uint32_t one;  // R mod p (1 in Montgomery form)
    // p - 2 = (2^e_ones - 1) 2^e_r + e_low: the inversion exponent's addition chain
    int e_ones, e_r;
    uint32_t e_low;
    __device__ __forceinline__ uint32_t redc(unsigned long long t) const {  // t < p R
        const uint32_t m = (uint32_t)t * nq;
        const uint32_t u = (uint32_t)((t + (unsigned long long)m * p) >> 32);  // < 2p
        return u >= p ? u - p : u;
    }
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const {
        return redc((unsigned long long)a * b);
    }
    __device__ __forceinline__ uint32_t mul2(uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1) const {
        return redc((unsigned long long)a0 * b0 + (unsigned long long)a1 * b1);
    }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        const uint32_t s = a + b;
        return s >= p ? s - p : s;
    }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
        return a >= b ? a - b : a + p - b;
    }
    // x^-1 = x^(p-2) (Fermat): x^(2^t - 1) by the doubling chain on the bits of t,
    // then the low bits; ~31 squarings + ~10 multiplies for the primes near 2^31
    __device__ __forceinline__ uint32_t inv(uint32_t x) const {
        uint32_t a = x;
        int s = 1;
        const int top = 31 - __clz(e_ones);
        for (int bit = top - 1; bit >= 0; --bit) {
            uint32_t b = a;
            for (int i = 0; i < s; ++i) b = mul(b, b);
            a = mul(b, a);
            s *= 2;
            if ((e_ones >> bit) & 1) {
                a = mul(mul(a, a), x);
                s += 1;
            }
        }
        for (int i = e_r - 1; i >= 0; --i) {
            a = mul(a, a);
            if ((e_low >> i) & 1u) a = mul(a, x);
        }
        return a;
    }
};

inline ModP make_modp(uint32_t p) {
    ModP M;
    M.p = p;
    uint32_t x = p;  // p^-1 mod 2^32 by Newton (p p = 1 mod 8 seeds 3 bits)
    for (int i = 0; i < 5; ++i) x *= 2u - p * x;
    M.nq = 0u - x;
    M.one = (uint32_t)((1ull << 32) % p);
    const uint32_t e = p - 2;
    int L = 0;
    while (L < 32 && (e >> L)) ++L;
    int t = 0;
    while (t < L && ((e >> (L - 1 - t)) & 1u)) ++t;
    M.e_ones = t;
    M.e_r = L - t;
    M.e_low = M.e_r ? (e & ((1u << M.e_r) - 1u)) : 0u;
    return M;
}

// per-prime constant table (Montgomery form), uploaded by the host
constexpr int kModpTab = 96;   // [k] = k^-1 R, [48 + k] = k R (k = 1..47; D <= 32)
constexpr int kModpTabK = 48;

constexpr int kModpThreads = 128;

template <int S>
struct ModpLayout {  // in uint32 words
    static constexpr int LD = S + 1;
    static constexpr int H = 0;                          // S columns x LD
    static constexpr int MU = H + S * LD;                // [S+2]
    static constexpr int P = MU + S + 2;                 // [(S+1)(S+2)/2] P_k rows
    static constexpr int CF = P + (S + 1) * (S + 2) / 2; // [S]
    static constexpr int T = CF + S;                     // [kDMax+2]
    static constexpr int G = T + kDMax + 2;              // [kDMax+2]
    static constexpr int U = G + kDMax + 2;              // [2][S] loop chain
    static constexpr int LM = U + 2 * S;                 // [2][S] logical row -> lane
    static constexpr int RED = (LM + 2 * S + 1) & ~1;    // [8] cross-warp exchange (8-byte aligned)
    static constexpr int TOTAL = RED + 8;  // even: every team's RED stays 8-byte aligned
};

// team sum of per-lane residues < p (modular adds at every level)
template <int W>
__device__ __forceinline__ uint32_t team_sum_mod(const TeamCtx<W>& tc, uint32_t* red, uint32_t v,
                                                 const ModP& M) {
    constexpr int WW = W < 32 ? W : 32;
#pragma unroll
    for (int off = WW / 2; off > 0; off >>= 1) v = M.add(v, __shfl_xor_sync(0xffffffffu, v, off, WW));
    if constexpr (W > 32) {
        if ((tc.lane & 31) == 0) red[tc.lane >> 5] = v;
        tc.sync();
        v = M.add(red[0], red[1]);
        tc.sync();
    }
    return v;
}

template <int W>
__device__ __forceinline__ uint32_t team_min(const TeamCtx<W>& tc, uint32_t* red, uint32_t v) {
    uint32_t mn;
    if constexpr (W <= 32) {
        mn = __reduce_min_sync(tc.wmask, v);
    } else {
        mn = __reduce_min_sync(0xffffffffu, v);
        if ((tc.lane & 31) == 0) red[4 + (tc.lane >> 5)] = mn;
        tc.sync();
        mn = red[4] < red[5] ? red[4] : red[5];
        tc.sync();
    }
    return mn;
}

template <int W>
__device__ __forceinline__ uint32_t team_bcast_u32(const TeamCtx<W>& tc, uint32_t* red, uint32_t v,
                                                   int src_lane) {
    if constexpr (W <= 32) {
        return __shfl_sync(tc.wmask, v, ((int)(threadIdx.x & 31) & ~(W - 1)) + src_lane);
    } else {
        if (tc.lane == src_lane) red[6] = v;
        tc.sync();
        const uint32_t r = red[6];
        tc.sync();
        return r;
    }
}

// All residues in Montgomery form (x R mod p): atilde / diag from the host, `tab` the
// per-prime constants (kModpTab layout).  The launch total gets plain residues.
template <int S, bool LOOPS>
__global__ void __launch_bounds__(kModpThreads) modp_term_kernel(
    const uint32_t* __restrict__ atilde, const uint32_t* __restrict__ diag, int n_half, ClassItems ci,
    ModP M, const uint32_t* __restrict__ tab, unsigned long long* __restrict__ total) {
    constexpr int W = TeamWidth<S>::W;
    constexpr int TPB = kModpThreads / W;
    constexpr int MH = S / 2;
    constexpr int R = (kDMax + W - 1) / W;
    using L = ModpLayout<S>;
    constexpr int LD = L::LD;
    extern __shared__ uint32_t usm[];
    TeamCtx<W> tc;
    tc.tib = threadIdx.x / W;
    tc.lane = threadIdx.x % W;
    if constexpr (W < 32) {
        tc.wmask = ((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1));
    } else {
        tc.wmask = 0xffffffffu;
    }
    const int lane = tc.lane;
    uint32_t* ws = usm + (size_t)tc.tib * L::TOTAL;
    uint32_t* H = ws + L::H;
    uint32_t* MUS = ws + L::MU;
    uint32_t* PT = ws + L::P;
    uint32_t* CF = ws + L::CF;
    uint32_t* T = ws + L::T;
    uint32_t* G = ws + L::G;
    uint32_t* RED = ws + L::RED;
    const int n = 2 * n_half;
    const int D = n_half;
    const uint32_t p = M.p;
    const uint32_t inv2 = tab[2];
    unsigned long long my_sum = 0;  // lane 0: this team's terms (each < p)
    // contiguous per-team runs of the class's items (Gosper's step, ItemCursor), in
    // dynamic block chunks from the class's counter as in the FAST kernel
    const long long n_teams = (long long)gridDim.x * TPB;
    const bool dyn = HAFB_DYN && ci.ctr != nullptr;
    long long ch = (ci.n_items + n_teams - 1) / n_teams;
    if (dyn) {
        ch = ci.n_items / (n_teams * HAFB_DYN_PER);
        ch = ch < 1 ? 1 : (ch > HAFB_DYN_CHUNK ? HAFB_DYN_CHUNK : ch);
    }
    const long long chunk = ch;
    long long first = ((long long)blockIdx.x * TPB + tc.tib) * chunk;
    ItemCursor cur;
    __shared__ long long dyn_base;

    for (;;) {
    if (dyn) {
        __syncthreads();
        if (threadIdx.x == 0) dyn_base = (long long)atomicAdd(ci.ctr, (unsigned long long)(TPB * chunk));
        __syncthreads();
        const long long b0 = dyn_base;
        if (b0 >= ci.n_items) break;
        first = b0 + (long long)tc.tib * chunk;
    }
    for (long long it = 0; it < chunk; ++it) {
        const long long item = first + it;
        const bool valid = item < ci.n_items;
        const ItemRef ir = cursor_item(ci, valid ? item : 0, cur);
        int vbit[MH];
        {
            uint32_t mm = ir.mask;
#pragma unroll
            for (int q = 0; q < MH; ++q) {
                vbit[q] = __ffs(mm) - 1;
                mm &= mm - 1;
            }
        }
        const int mybit = lane < S ? (int)__fns(ir.mask, 0, (lane >> 1) + 1) : 0;
        const int vr = 2 * mybit + (lane & 1);
        if (lane < S) {
#pragma unroll
            for (int c = 0; c < S; ++c) H[c * LD + lane] = atilde[vr * n + 2 * vbit[c >> 1] + (c & 1)];
        }
        tc.sync();
        // ------------------------------------------------ loop corrections ell_k = v B^(k-1) Xv
        if constexpr (LOOPS) {
            uint32_t* U = ws + L::U;
            const uint32_t xv = lane < S ? diag[2 * mybit + ((lane & 1) ^ 1)] : 0u;
            uint32_t u = lane < S ? diag[vr] : 0u;
            for (int k = 1; k <= D; ++k) {
                const uint32_t ell = team_sum_mod<W>(tc, RED, M.mul(u, xv), M);
                if (lane == 0) G[k] = ell;  // folded into g_k below
                if (k < D) {
                    uint32_t* ub = U + (k & 1) * S;
                    if (lane < S) ub[lane] = u;
                    tc.sync();
                    uint32_t acc = 0u;
                    if (lane < S)
                        for (int i = 0; i < S; i += 2)  // S even: products in pairs, one REDC each
                            acc = M.add(acc, M.mul2(ub[i], H[lane * LD + i], ub[i + 1], H[lane * LD + i + 1]));
                    u = acc;
                }
            }
        }
        // ------------------------------------------------ Hessenberg over GF(p)
        int myrow = lane;
        uint32_t* lm0 = ws + L::LM;
        if (lane < S) lm0[lane] = lane;
        tc.sync();
#pragma unroll 1
        for (int J = 0; J < S - 2; ++J) {
            const int B = J & 1;
            const uint32_t* lm = ws + L::LM + B * S;
            uint32_t* lmn = ws + L::LM + (1 - B) * S;
            const uint32_t x = lane < S ? H[J * LD + lane] : 0u;
            // first nonzero entry of column J below the diagonal (any nonzero pivot works
            // in a field; the smallest logical row makes the choice deterministic)
            const uint32_t cand = (myrow > J && myrow < S && x != 0u) ? ((uint32_t)myrow << 6) | (uint32_t)lane
                                                                     : 0xffffffffu;
            const uint32_t best = team_min<W>(tc, RED, cand);
            if (best == 0xffffffffu) {
                if (lane < S) lmn[lane] = lm[lane];
                tc.sync();
                continue;
            }
            const int prow = (int)(best >> 6), plane = (int)(best & 63u);
            const int l_j1 = (int)lm[J + 1];
            if (lane < S) lmn[lane] = lane == J + 1 ? (uint32_t)plane : (lane == prow ? (uint32_t)l_j1 : lm[lane]);
            if (myrow == prow) myrow = J + 1;
            else if (myrow == J + 1) myrow = prow;
            uint32_t x1 = lane < S ? H[(J + 1) * LD + lane] : 0u;
            if (prow != J + 1 && lane < S) {
                const uint32_t xb = H[prow * LD + lane];
                H[prow * LD + lane] = x1;
                x1 = xb;
            }
            const uint32_t piv = team_bcast_u32<W>(tc, RED, x, plane);
            const uint32_t pv1 = team_bcast_u32<W>(tc, RED, x1, plane);
            const uint32_t ipiv = M.inv(piv);
            const bool elim = myrow >= J + 2 && myrow < S;
            const uint32_t mu = elim ? M.mul(x, ipiv) : 0u;
            if (elim) MUS[myrow] = mu;
            tc.sync();
            const uint32_t* prw = H + plane;
            uint32_t acc = 0;
            int c = J + 2;
#pragma unroll 1
            for (; c + 1 < S; c += 2) {  // row update of two columns, their column-gemv terms in one REDC
                const uint32_t x0 = lane < S ? H[c * LD + lane] : 0u;
                const uint32_t x1c = lane < S ? H[(c + 1) * LD + lane] : 0u;
                const uint32_t y0 = M.sub(x0, M.mul(mu, prw[c * LD]));
                const uint32_t y1 = M.sub(x1c, M.mul(mu, prw[(c + 1) * LD]));
                acc = M.add(acc, M.mul2(MUS[c], y0, MUS[c + 1], y1));
                if (elim) {
                    H[c * LD + lane] = y0;
                    H[(c + 1) * LD + lane] = y1;
                }
            }
            if (c < S) {
                const uint32_t xc = lane < S ? H[c * LD + lane] : 0u;
                const uint32_t y = M.sub(xc, M.mul(mu, prw[c * LD]));
                acc = M.add(acc, M.mul(MUS[c], y));
                if (elim) H[c * LD + lane] = y;
            }
            const uint32_t h1 = M.add(M.sub(x1, M.mul(mu, pv1)), acc);
            if constexpr (W > 32) tc.sync();
            if (lane < S) H[(J + 1) * LD + lane] = h1;
            tc.sync();
        }
        const uint32_t* lmf = ws + L::LM + ((S - 2) & 1) * S;
        auto h = [&](int i, int c) -> uint32_t { return H[c * LD + lmf[i]]; };
        // ------------------------------------------------ characteristic polynomial (leading minors)
        if (lane == 0) PT[0] = M.one;
        uint32_t prodl = M.one;
        tc.sync();
        for (int k = 1; k <= S; ++k) {
            if (k >= 2) {
                const uint32_t beta = h(k - 1, k - 2);
                if (lane <= k - 2) {
                    prodl = M.mul(lane == k - 2 ? M.one : prodl, beta);
                    CF[lane] = M.mul(h(lane, k - 1), prodl);  // coef of P_{lane}
                }
            }
            tc.sync();
            const uint32_t hk = h(k - 1, k - 1);
            const uint32_t* Pk1 = PT + ((k - 1) * k) / 2;
            uint32_t* Pk = PT + (k * (k + 1)) / 2;
            for (int d = lane; d <= k; d += W) {
                uint32_t v;
                if (d == k) {
                    v = Pk1[k - 1];
                } else {
                    v = M.sub(d >= 1 ? Pk1[d - 1] : 0u, M.mul(hk, Pk1[d]));
                    uint32_t s = 0u;
                    int i = d + 1;
                    for (; i + 1 < k; i += 2)
                        s = M.add(s, M.mul2(CF[i - 1], PT[((i - 1) * i) / 2 + d], CF[i], PT[(i * (i + 1)) / 2 + d]));
                    if (i < k) s = M.add(s, M.mul(CF[i - 1], PT[((i - 1) * i) / 2 + d]));
                    v = M.sub(v, s);
                }
                Pk[d] = v;
            }
            tc.sync();
        }
        const uint32_t* a = PT + (S * (S + 1)) / 2;
        // ------------------------------------------------ Newton + Cayley-Hamilton: t_k
        {
            uint32_t acck[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int k = lane + 1 + W * r;
                acck[r] = (k <= D && k <= S) ? M.sub(0u, M.mul(tab[kModpTabK + k], a[S - k])) : 0u;
            }
            for (int kk = 1; kk <= D; ++kk) {
                const int owner = (kk - 1) % W, chunk = (kk - 1) / W;
                uint32_t v = acck[0];
#pragma unroll
                for (int r = 1; r < R; ++r)
                    if (r == chunk) v = acck[r];
                const uint32_t tk = team_bcast_u32<W>(tc, RED, v, owner);
                if (lane == owner) T[kk] = tk;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    const int jj = k - kk;
                    if (k <= D && jj >= 1 && jj <= S) acck[r] = M.sub(acck[r], M.mul(a[S - jj], tk));
                }
            }
        }
        tc.sync();
        // g_k = k s_k = t_k / 2 (+ k ell_k / 2)
        for (int k = lane + 1; k <= D; k += W) {
            uint32_t t = T[k];
            if constexpr (LOOPS) t = M.add(t, M.mul(tab[kModpTabK + k], G[k]));
            G[k] = M.mul(t, inv2);
        }
        tc.sync();
        // ------------------------------------------------ exp: e_k = k^-1 sum_{j=1..k} g_j e_{k-j}
        uint32_t eD = 0;
        {
            uint32_t acck[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acck[r] = 0u;
            for (int kk = 0; kk < D; ++kk) {
                uint32_t ek;
                if (kk == 0) {
                    ek = M.one;
                } else {
                    const int owner = (kk - 1) % W, chunk = (kk - 1) / W;
                    uint32_t v = acck[0];
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        if (r == chunk) v = acck[r];
                    ek = M.mul(team_bcast_u32<W>(tc, RED, v, owner), tab[kk]);
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = lane + 1 + W * r;
                    if (k <= D && k > kk) acck[r] = M.add(acck[r], M.mul(G[k - kk], ek));
                }
            }
            const int owner = (D - 1) % W, chunk = (D - 1) / W;
            uint32_t v = acck[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
                if (r == chunk) v = acck[r];
            eD = M.redc(M.mul(team_bcast_u32<W>(tc, RED, v, owner), tab[D]));  // plain residue
        }
        if (valid && lane == 0) my_sum += ((D - MH) & 1) ? (eD ? p - eD : 0u) : eD;
        tc.sync();
    }
    if (!dyn) break;
    }
    if (lane == 0 && my_sum) atomicAdd(total, my_sum);
}

}  // namespace hafb
