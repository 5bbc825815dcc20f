/*
 * referee.c -- TEST INFRASTRUCTURE ONLY: an extended-precision referee for the
 * hafnian / loop-hafnian subset sum.
 *
 * The reference (hafnium 0.1.0) and both device arithmetics (MIRROR, FAST)
 * compute in IEEE double.  Under cancellation (cond = sum|t| / |result| up to
 * 1e7 on the BASELINE configs) they disagree with each other well above the
 * 1e-10 north-star bound, and without a more precise evaluation nobody can say
 * which one is nearer the true value.  This file evaluates the SAME formula in
 * a wider type:
 *
 *     REAL = long double   (x87 80-bit, 64-bit significand: 2^11 = 2048x
 *                           the precision of double)          -> libreferee.so
 *     REAL = __float128    (IEEE binary128, 113-bit significand,
 *                           soft-float; used to check the long
 *                           double referee on small cases)     -> libreferee_q.so
 *
 * Algorithm per subset (the charpoly route of _numba.py:297-351):
 *   gather B = atilde[idx][:, idx]                    (_numba.py:317-321)
 *   Hessenberg by pivoted elementary similarity        (_numba.py:36-67; pivot by
 *                                                       |re|^2+|im|^2, first max)
 *   monic charpoly by the leading-minor recurrence     (_numba.py:203-225)
 *   power traces by Newton's identities and, past the
 *   degree, the Cayley-Hamilton recurrence             (_numba.py:228-250)
 *   loops: ell_k = v B^(k-1) (Xv)^T on the un-reduced B (_numba.py:253-273, :337-347)
 *   s_k = t_k/(2k) (+ ell_k/2); [x^D] exp(s) by the
 *   recurrence e_k = (1/k) sum_j j s_j e_(k-j)         (tests/test_engine.py:31-42, the
 *                                                       reference's own oracle for _exp_top)
 *   sign (-1)^(D-m)                                    (_numba.py:349-351)
 * Terms are summed in REAL with Kahan compensation per fixed block of masks and
 * the block sums added in block order (the result does not depend on the thread
 * count).  Results are returned as double pairs (hi, lo) per component.
 *
 * Nothing under paper_1805_12498_b200/ loads this library; only tests/golden's
 * fixture generator (gen_referee.py) and tests/ do.
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef REF_QUAD
typedef __float128 REAL;
#define RABS(x) ((x) < 0 ? -(x) : (x))
#else
typedef long double REAL;
#define RABS(x) fabsl(x)
#endif

typedef struct { REAL re, im; } cr;

static inline cr mk(REAL a, REAL b) { cr z = {a, b}; return z; }
static inline cr add(cr a, cr b) { return mk(a.re + b.re, a.im + b.im); }
static inline cr sub(cr a, cr b) { return mk(a.re - b.re, a.im - b.im); }
static inline cr mul(cr a, cr b) { return mk(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cr scl(REAL r, cr a) { return mk(r * a.re, r * a.im); }
static inline REAL nrm(cr a) { return a.re * a.re + a.im * a.im; }
static inline cr dvd(cr a, cr b) {
    REAL d = nrm(b);
    return mk((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}
static inline int nz(cr a) { return a.re != 0 || a.im != 0; }

enum { SMAX = 128, DMAX = 64 };

typedef struct {
    cr b[SMAX * SMAX];   /* un-reduced subset matrix (loops need it) */
    cr h[SMAX * SMAX];   /* reduced in place */
    cr P[(SMAX + 1) * (SMAX + 1)];
    cr a[SMAX + 1], t[DMAX + 1], s[DMAX + 1], e[DMAX + 1], u[SMAX], un[SMAX];
} work_t;

/* _numba.py:36-67 */
static void hessenberg(cr* h, int S) {
    for (int j = 0; j < S - 2; j++) {
        int p = j + 1;
        REAL best = nrm(h[(j + 1) * S + j]);
        for (int i = j + 2; i < S; i++) {
            REAL v = nrm(h[i * S + j]);
            if (v > best) { best = v; p = i; }
        }
        if (best == 0) continue;
        if (p != j + 1) {
            for (int k = 0; k < S; k++) { cr x = h[p * S + k]; h[p * S + k] = h[(j + 1) * S + k]; h[(j + 1) * S + k] = x; }
            for (int k = 0; k < S; k++) { cr x = h[k * S + p]; h[k * S + p] = h[k * S + j + 1]; h[k * S + j + 1] = x; }
        }
        cr piv = h[(j + 1) * S + j];
        for (int i = j + 2; i < S; i++) {
            cr mu = dvd(h[i * S + j], piv);
            if (!nz(mu)) continue;
            for (int k = j; k < S; k++) h[i * S + k] = sub(h[i * S + k], mul(mu, h[(j + 1) * S + k]));
            h[i * S + j] = mk(0, 0);
            for (int k = 0; k < S; k++) h[k * S + j + 1] = add(h[k * S + j + 1], mul(mu, h[k * S + i]));
        }
    }
}

/* _numba.py:203-225: P_k = (x - h_kk) P_(k-1) - sum_i h_(i,k) prod(beta) P_(i-1); a = P_S ascending */
static void charpoly(const cr* h, int S, cr* P, cr* a) {
    int W = S + 1;
    memset(P, 0, sizeof(cr) * W * W);
    P[0] = mk(1, 0);
    for (int k = 1; k <= S; k++) {
        cr* Pk = P + k * W;
        const cr* Pp = P + (k - 1) * W;
        cr hkk = h[(k - 1) * S + (k - 1)];
        for (int d = 0; d <= k; d++) {
            cr v = d >= 1 ? Pp[d - 1] : mk(0, 0);
            if (d <= k - 1) v = sub(v, mul(hkk, Pp[d]));
            Pk[d] = v;
        }
        cr beta = mk(1, 0);
        for (int i = k - 1; i >= 1; i--) {
            beta = mul(beta, h[i * S + (i - 1)]);
            if (!nz(beta)) break;
            cr c = mul(h[(i - 1) * S + (k - 1)], beta);
            const cr* Pi = P + (i - 1) * W;
            for (int d = 0; d <= i - 1; d++) Pk[d] = sub(Pk[d], mul(c, Pi[d]));
        }
    }
    for (int d = 0; d <= S; d++) a[d] = P[S * W + d];
}

/* one signed term; returns it through *out */
static void subset_term(const cr* at, const cr* dg, int n_half, uint64_t mask, int loops,
                        work_t* w, cr* out) {
    int n = 2 * n_half, idx[SMAX], S = 0, m = 0;
    for (int i = 0; i < n_half; i++)
        if ((mask >> i) & 1) { idx[S++] = 2 * i; idx[S++] = 2 * i + 1; m++; }
    for (int r = 0; r < S; r++)
        for (int c = 0; c < S; c++) w->b[r * S + c] = w->h[r * S + c] = at[idx[r] * n + idx[c]];
    hessenberg(w->h, S);
    charpoly(w->h, S, w->P, w->a);
    int D = n_half;
    /* monic x^S + c_1 x^(S-1) + ... + c_S with c_j = a[S-j]: Newton / Cayley-Hamilton */
    for (int k = 1; k <= D; k++) {
        cr acc = mk(0, 0);
        int jm = k - 1 < S ? k - 1 : S;
        for (int j = 1; j <= jm; j++) acc = add(acc, mul(w->a[S - j], w->t[k - j]));
        if (k <= S) acc = add(acc, scl((REAL)k, w->a[S - k]));
        w->t[k] = mk(-acc.re, -acc.im);
    }
    w->s[0] = mk(0, 0);
    for (int k = 1; k <= D; k++) w->s[k] = scl((REAL)1 / (REAL)(2 * k), w->t[k]);
    if (loops) {
        cr xv[SMAX];
        for (int r = 0; r < S; r++) w->u[r] = dg[idx[r]];
        for (int p = 0; p < m; p++) { xv[2 * p] = w->u[2 * p + 1]; xv[2 * p + 1] = w->u[2 * p]; }
        for (int k = 1; k <= D; k++) {
            cr acc = mk(0, 0);
            for (int i = 0; i < S; i++) acc = add(acc, mul(w->u[i], xv[i]));
            w->s[k] = add(w->s[k], scl((REAL)0.5, acc));
            if (k < D) {
                for (int j = 0; j < S; j++) {
                    cr v = mk(0, 0);
                    for (int i = 0; i < S; i++) v = add(v, mul(w->u[i], w->b[i * S + j]));
                    w->un[j] = v;
                }
                memcpy(w->u, w->un, sizeof(cr) * S);
            }
        }
    }
    w->e[0] = mk(1, 0);
    for (int k = 1; k <= D; k++) {
        cr acc = mk(0, 0);
        for (int j = 1; j <= k; j++) acc = add(acc, scl((REAL)j, mul(w->s[j], w->e[k - j])));
        w->e[k] = scl((REAL)1 / (REAL)k, acc);
    }
    cr r = w->e[D];
    if ((n_half - m) & 1) r = mk(-r.re, -r.im);
    *out = r;
}

static void split(REAL x, double* hi, double* lo) {
    double h = (double)x;
    *hi = h;
    *lo = (double)(x - (REAL)h);
}

/* ------------------------------------------------------------------ thread pool */

typedef struct {
    const cr* at; const cr* dg; int n_half, loops;
    uint64_t lo, hi, block;
    int64_t nblocks;
    cr* bsum; REAL* babs;
    const uint64_t* masks; cr* terms;
    int64_t next;
    pthread_mutex_t mu;
} job_t;

static int64_t take(job_t* j) {
    pthread_mutex_lock(&j->mu);
    int64_t b = j->next++;
    pthread_mutex_unlock(&j->mu);
    return b;
}

static void* range_worker(void* arg) {
    job_t* j = (job_t*)arg;
    work_t* w = (work_t*)malloc(sizeof(work_t));
    for (;;) {
        int64_t b = take(j);
        if (b >= j->nblocks) break;
        uint64_t a = j->lo + (uint64_t)b * j->block, e = a + j->block;
        if (e > j->hi) e = j->hi;
        cr s = mk(0, 0), c = mk(0, 0);
        REAL sa = 0;
        for (uint64_t mask = a; mask < e; mask++) {
            if (mask == 0) continue;
            cr t;
            subset_term(j->at, j->dg, j->n_half, mask, j->loops, w, &t);
            sa += sqrtl((long double)nrm(t));
            cr y = sub(t, c), u = add(s, y);
            c = sub(sub(u, s), y);
            s = u;
        }
        j->bsum[b] = s;
        j->babs[b] = sa;
    }
    free(w);
    return NULL;
}

static void* terms_worker(void* arg) {
    job_t* j = (job_t*)arg;
    work_t* w = (work_t*)malloc(sizeof(work_t));
    for (;;) {
        int64_t b = take(j);
        if (b >= j->nblocks) break;
        uint64_t a = (uint64_t)b * 64, e = a + 64;
        if (e > j->hi) e = j->hi;
        for (uint64_t q = a; q < e; q++)
            subset_term(j->at, j->dg, j->n_half, j->masks[q], j->loops, w, &j->terms[q]);
    }
    free(w);
    return NULL;
}

static void run(job_t* j, int threads, void* (*fn)(void*)) {
    pthread_t th[256];
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_mutex_init(&j->mu, NULL);
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, fn, j);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&j->mu);
}

static cr* load(const double* x, int64_t count) {
    cr* o = (cr*)malloc(sizeof(cr) * (count ? count : 1));
    for (int64_t i = 0; i < count; i++) o[i] = mk((REAL)x[2 * i], (REAL)x[2 * i + 1]);
    return o;
}

/* Sum of the signed terms of masks [lo, hi) (mask 0 skipped).
 * out[0..3] = re_hi, re_lo, im_hi, im_lo of the sum; out[4] = sum |t|. */
int ref_sum_range(const double* atilde, const double* diag, int n_half, uint64_t lo,
                  uint64_t hi, int include_loops, int threads, double* out) {
    if (n_half < 1 || 2 * n_half > SMAX || n_half > DMAX || hi <= lo) return -1;
    int n = 2 * n_half;
    job_t j;
    memset(&j, 0, sizeof j);
    j.at = load(atilde, (int64_t)n * n);
    j.dg = load(diag, n);
    j.n_half = n_half;
    j.loops = include_loops;
    j.lo = lo;
    j.hi = hi;
    j.block = 256;
    j.nblocks = (int64_t)((hi - lo + j.block - 1) / j.block);
    j.bsum = (cr*)calloc(j.nblocks, sizeof(cr));
    j.babs = (REAL*)calloc(j.nblocks, sizeof(REAL));
    run(&j, threads, range_worker);
    cr s = mk(0, 0), c = mk(0, 0);
    REAL sa = 0;
    for (int64_t b = 0; b < j.nblocks; b++) {
        cr y = sub(j.bsum[b], c), u = add(s, y);
        c = sub(sub(u, s), y);
        s = u;
        sa += j.babs[b];
    }
    split(s.re, &out[0], &out[1]);
    split(s.im, &out[2], &out[3]);
    out[4] = (double)sa;
    free((void*)j.at); free((void*)j.dg); free(j.bsum); free(j.babs);
    return 0;
}

/* Per-term values (rounded to double) of `count` masks. */
int ref_terms(const double* atilde, const double* diag, int n_half, const uint64_t* masks,
              int64_t count, int include_loops, int threads, double* terms) {
    if (n_half < 1 || 2 * n_half > SMAX || n_half > DMAX) return -1;
    int n = 2 * n_half;
    job_t j;
    memset(&j, 0, sizeof j);
    j.at = load(atilde, (int64_t)n * n);
    j.dg = load(diag, n);
    j.n_half = n_half;
    j.loops = include_loops;
    j.masks = masks;
    j.hi = (uint64_t)count;
    j.nblocks = (count + 63) / 64;
    j.terms = (cr*)calloc(count ? count : 1, sizeof(cr));
    run(&j, threads, terms_worker);
    for (int64_t q = 0; q < count; q++) {
        terms[2 * q] = (double)j.terms[q].re;
        terms[2 * q + 1] = (double)j.terms[q].im;
    }
    free((void*)j.at); free((void*)j.dg); free(j.terms);
    return 0;
}

/* Significand bits of REAL (64 for long double, 113 for __float128). */
int ref_mant_bits(void) {
#ifdef REF_QUAD
    return 113;
#else
    return LDBL_MANT_DIG;
#endif
}
