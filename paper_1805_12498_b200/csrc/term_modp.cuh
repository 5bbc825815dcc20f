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

struct ModP {
    uint32_t p;
    unsigned long long m;  // floor(2^64 / p) (Barrett)
    __device__ __forceinline__ uint32_t red(unsigned long long x) const {  // x < 2^62
        const unsigned long long q = __umul64hi(x, m);
        unsigned long long r = x - q * p;
        return (uint32_t)(r >= p ? r - p : r);
    }
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const {
        return red((unsigned long long)a * b);
    }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const {
        const uint32_t s = a + b;
        return s >= p ? s - p : s;
    }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
        return a >= b ? a - b : a + p - b;
    }
    __device__ __forceinline__ uint32_t pow(uint32_t a, uint32_t e) const {
        uint32_t r = 1;
        while (e) {
            if (e & 1u) r = mul(r, a);
            a = mul(a, a);
            e >>= 1;
        }
        return r;
    }
};

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

// team sum of per-lane residues < p
template <int W>
__device__ __forceinline__ uint32_t team_sum_mod(const TeamCtx<W>& tc, uint32_t* red, uint32_t v,
                                                 const ModP& M) {
    unsigned long long s = v;
    constexpr int WW = W < 32 ? W : 32;
#pragma unroll
    for (int off = WW / 2; off > 0; off >>= 1)
        s += __shfl_xor_sync(0xffffffffu, s, off, WW);
    if constexpr (W > 32) {
        if ((tc.lane & 31) == 0) reinterpret_cast<unsigned long long*>(red)[tc.lane >> 5] = s;
        tc.sync();
        const unsigned long long* r = reinterpret_cast<unsigned long long*>(red);
        s = r[0] + r[1];
        tc.sync();
    }
    return M.red(s);
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

// inv[k] = k^-1 mod p for k = 1..kDMax (from the host)
template <int S, bool LOOPS>
__global__ void __launch_bounds__(kModpThreads) modp_term_kernel(
    const uint32_t* __restrict__ atilde, const uint32_t* __restrict__ diag, int n_half, ClassItems ci,
    ModP M, const uint32_t* __restrict__ inv, unsigned long long* __restrict__ total) {
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
    const uint32_t inv2 = inv[2];
    unsigned long long my_sum = 0;  // lane 0: this team's terms (each < p)
    const long long stride = (long long)gridDim.x * TPB;

    for (long long base = (long long)blockIdx.x * TPB; base < ci.n_items; base += stride) {
        const long long item = base + tc.tib;
        const bool valid = item < ci.n_items;
        const ItemRef ir = resolve_item(ci, valid ? item : base);
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
                    unsigned long long acc = 0;
                    if (lane < S)
                        for (int i = 0; i < S; ++i) acc += M.mul(ub[i], H[lane * LD + i]);
                    u = lane < S ? M.red(acc) : 0u;
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
            const uint32_t ipiv = M.pow(piv, p - 2);
            const bool elim = myrow >= J + 2 && myrow < S;
            const uint32_t mu = elim ? M.mul(x, ipiv) : 0u;
            if (elim) MUS[myrow] = mu;
            tc.sync();
            const uint32_t* prw = H + plane;
            uint32_t acc = 0;
            unsigned long long acc64 = 0;
#pragma unroll 1
            for (int c = J + 2; c < S; ++c) {
                const uint32_t xc = lane < S ? H[c * LD + lane] : 0u;
                const uint32_t y = M.sub(xc, M.mul(mu, prw[c * LD]));
                acc64 += M.mul(MUS[c], y);
                if (elim) H[c * LD + lane] = y;
            }
            acc = M.red(acc64);
            const uint32_t h1 = M.add(M.sub(x1, M.mul(mu, pv1)), acc);
            if constexpr (W > 32) tc.sync();
            if (lane < S) H[(J + 1) * LD + lane] = h1;
            tc.sync();
        }
        const uint32_t* lmf = ws + L::LM + ((S - 2) & 1) * S;
        auto h = [&](int i, int c) -> uint32_t { return H[c * LD + lmf[i]]; };
        // ------------------------------------------------ characteristic polynomial (leading minors)
        if (lane == 0) PT[0] = 1u;
        uint32_t prodl = 1u;
        tc.sync();
        for (int k = 1; k <= S; ++k) {
            if (k >= 2) {
                const uint32_t beta = h(k - 1, k - 2);
                if (lane <= k - 2) {
                    prodl = M.mul(lane == k - 2 ? 1u : prodl, beta);
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
                    unsigned long long s = 0;
                    for (int i = d + 1; i < k; ++i) s += M.mul(CF[i - 1], PT[((i - 1) * i) / 2 + d]);
                    v = M.sub(v, M.red(s));
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
                acck[r] = (k <= D && k <= S) ? M.sub(0u, M.mul((uint32_t)k, a[S - k])) : 0u;
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
            uint32_t g = M.mul(T[k], inv2);
            if constexpr (LOOPS) g = M.add(g, M.mul(M.mul((uint32_t)k, G[k]), inv2));
            G[k] = g;
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
                    ek = 1u;
                } else {
                    const int owner = (kk - 1) % W, chunk = (kk - 1) / W;
                    uint32_t v = acck[0];
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        if (r == chunk) v = acck[r];
                    ek = M.mul(team_bcast_u32<W>(tc, RED, v, owner), inv[kk]);
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
            eD = M.mul(team_bcast_u32<W>(tc, RED, v, owner), inv[D]);
        }
        if (valid && lane == 0) my_sum += ((D - MH) & 1) ? (eD ? p - eD : 0u) : eD;
        tc.sync();
    }
    if (lane == 0 && my_sum) atomicAdd(total, my_sum);
}

}  // namespace hafb
