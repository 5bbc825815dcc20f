// cplx.cuh -- complex128 arithmetic for the hafnian kernels.
//
// Two families:
//   m_*  "mirror" ops: exactly the IEEE-754 operation sequence of the reference
//        (numba complex_mul_impl / complex_div_impl (CPython _Py_c_quot) /
//        complex_abs_impl (glibc hypot), real operands promoted to (x, 0.0)).
//        Built from __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn/__dsqrt_rn, which
//        the compiler never contracts into FMA, so the device results are
//        bit-identical to the reference CPU path.
//   f_*  "fast" ops: FMA-contracted forms used by the throughput kernels.
//
// The header compiles for host too (g++ -ffp-contract=off), so the mirror ops
// can be unit-tested against glibc on the CPU (tests/test_cplx_host.py).
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

struct cd {
    double re, im;
};

HD cd mk(double r, double i) {
    cd z;
    z.re = r;
    z.im = i;
    return z;
}

#if defined(__CUDA_ARCH__)
HD double r_mul(double a, double b) { return __dmul_rn(a, b); }
HD double r_add(double a, double b) { return __dadd_rn(a, b); }
HD double r_sub(double a, double b) { return __dsub_rn(a, b); }
HD double r_div(double a, double b) { return __ddiv_rn(a, b); }
HD double r_sqrt(double a) { return __dsqrt_rn(a); }
#else
HD double r_mul(double a, double b) { return a * b; }
HD double r_add(double a, double b) { return a + b; }
HD double r_sub(double a, double b) { return a - b; }
HD double r_div(double a, double b) { return a / b; }
HD double r_sqrt(double a) { return sqrt(a); }
#endif

// ---------------------------------------------------------------- mirror ops
HD cd m_add(cd a, cd b) { return mk(r_add(a.re, b.re), r_add(a.im, b.im)); }
HD cd m_sub(cd a, cd b) { return mk(r_sub(a.re, b.re), r_sub(a.im, b.im)); }
HD cd m_neg(cd a) { return mk(-a.re, -a.im); }
HD bool m_nz(cd a) { return a.re != 0.0 || a.im != 0.0; }
HD bool m_finite(cd a) { return isfinite(a.re) && isfinite(a.im); }

// numba complex_mul_impl: (a+bi)(c+di) = (ac - bd) + (ad + bc)i
HD cd m_mul(cd x, cd y) {
    double ac = r_mul(x.re, y.re), bd = r_mul(x.im, y.im);
    double ad = r_mul(x.re, y.im), bc = r_mul(x.im, y.re);
    return mk(r_sub(ac, bd), r_add(ad, bc));
}
// real * complex, real promoted to (r, 0.0) as numba does
HD cd m_rmul(double r, cd y) { return m_mul(mk(r, 0.0), y); }

// numba complex_div_impl == CPython _Py_c_quot (Smith's algorithm)
HD cd m_div(cd a, cd b) {
    double areal = a.re, aimag = a.im, breal = b.re, bimag = b.im;
    if (fabs(breal) >= fabs(bimag)) {
        if (breal == 0.0) return mk(NAN, NAN);
        double ratio = r_div(bimag, breal);
        double denom = r_add(breal, r_mul(bimag, ratio));
        return mk(r_div(r_add(areal, r_mul(aimag, ratio)), denom),
                  r_div(r_sub(aimag, r_mul(areal, ratio)), denom));
    } else {
        if (bimag == 0.0) return mk(NAN, NAN);
        double ratio = r_div(breal, bimag);
        double denom = r_add(r_mul(breal, ratio), bimag);
        return mk(r_div(r_add(r_mul(areal, ratio), aimag), denom),
                  r_div(r_sub(r_mul(aimag, ratio), areal), denom));
    }
}
// complex / real: m_div(a, (r, 0)) with its first branch's constant parts folded --
// ratio = 0/r is a signed zero (copysign(0, r) for any non-NaN r != 0) and
// denom = r + 0*ratio = r exactly -- so two divisions instead of three, same bits
// (tests/test_cplx_host.py checks it against m_div over special values)
HD cd m_rdiv(cd a, double r) {
    if (!(fabs(r) >= 0.0) || r == 0.0) return mk(NAN, NAN);  // NaN / zero divisor, as m_div
    const double ratio = copysign(0.0, r);
    return mk(r_div(r_add(a.re, r_mul(a.im, ratio)), r), r_div(r_sub(a.im, r_mul(a.re, ratio)), r));
}

// glibc >= 2.35 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel), which is
// what numba's abs(complex) calls on this image.  Verified bit-exact against the
// host libm in tests/test_cplx_host.py.
// Attribution: the algorithm (scaling ranges and the correction terms below) is the
// one published in GNU C Library's e_hypot.c (LGPL-2.1-or-later, by Adhemerval
// Zanella / the glibc authors, after Borges' "An Improved Algorithm for hypot(a,b)");
// it is restated here operation by operation because bit-identity with the reference
// requires the same rounding sequence.
HD double hypot_kernel(double ax, double ay) {
    double h = r_sqrt(r_add(r_mul(ax, ax), r_mul(ay, ay)));
    double t1, t2;
    if (h <= r_mul(2.0, ay)) {
        double delta = r_sub(h, ay);
        t1 = r_mul(ax, r_sub(r_mul(2.0, delta), ax));
        t2 = r_mul(r_sub(delta, r_mul(2.0, r_sub(ax, ay))), delta);
    } else {
        double delta = r_sub(h, ax);
        t1 = r_mul(r_mul(2.0, delta), r_sub(ax, r_mul(2.0, ay)));
        t2 = r_add(r_mul(r_sub(r_mul(4.0, delta), ay), ay), r_mul(delta, delta));
    }
    h = r_sub(h, r_div(r_add(t1, t2), r_mul(2.0, h)));
    return h;
}

HD double m_hypot(double x, double y) {
    const double SCALE = 0x1p-600, LARGE_VAL = 0x1p+511, TINY_VAL = 0x1p-511, EPS = 0x1p-54;
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return r_add(x, y);
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x;
    double ay = x < y ? x : y;
    if (ax > LARGE_VAL) {
        if (ay <= r_mul(ax, EPS)) return r_add(ax, ay);
        return r_div(hypot_kernel(r_mul(ax, SCALE), r_mul(ay, SCALE)), SCALE);
    }
    if (ay < TINY_VAL) {
        if (ax >= r_div(ay, EPS)) return r_add(ax, ay);
        return r_mul(hypot_kernel(r_div(ax, SCALE), r_div(ay, SCALE)), SCALE);
    }
    if (ay <= r_mul(ax, EPS)) return r_add(ax, ay);
    return hypot_kernel(ax, ay);
}
HD double m_abs(cd a) { return m_hypot(a.re, a.im); }

// numba cmathimpl.sqrt_impl (NumPy npy_csqrt, CACM algorithm 312; BSD-licensed NumPy
// algorithm restated for bit-identity)
HD cd m_sqrt(cd z) {
    const double THRES = 1.7976931348623157e308 / (1. + 1.414213562373095048801688724209698079E0);
    double a = z.re, b = z.im;
    if (a == 0.0 && b == 0.0) return mk(fabs(b), b);
    if (isinf(b)) return mk(fabs(b), b);
    if (isnan(a)) return mk(a, a);
    if (isinf(a)) {
        if (a < 0.0) return mk(fabs(r_sub(b, b)), copysign(a, b));
        return mk(a, copysign(r_sub(b, b), b));
    }
    bool scale = false;
    if (fabs(a) >= THRES || fabs(b) >= THRES) {
        a = r_mul(a, 0.25);
        b = r_mul(b, 0.25);
        scale = true;
    }
    double real, imag, t;
    if (a >= 0) {
        t = r_sqrt(r_mul(r_add(a, m_hypot(a, b)), 0.5));
        real = t;
        imag = r_div(b, r_mul(2.0, t));
    } else {
        t = r_sqrt(r_mul(r_add(-a, m_hypot(a, b)), 0.5));
        real = r_div(fabs(b), r_mul(2.0, t));
        imag = copysign(t, b);
    }
    if (scale) return mk(r_mul(real, 2.0), imag);
    return mk(real, imag);
}

// ---------------------------------------------------------------- fast ops
// acc + x*y with two FMAs per component (fast kernels only)
HD cd f_cma(cd acc, cd x, cd y) {
    double re = fma(x.re, y.re, acc.re);
    re = fma(-x.im, y.im, re);
    double im = fma(x.re, y.im, acc.im);
    im = fma(x.im, y.re, im);
    return mk(re, im);
}
// acc - x*y
HD cd f_cms(cd acc, cd x, cd y) {
    double re = fma(-x.re, y.re, acc.re);
    re = fma(x.im, y.im, re);
    double im = fma(-x.re, y.im, acc.im);
    im = fma(-x.im, y.re, im);
    return mk(re, im);
}
HD cd f_mul(cd x, cd y) { return mk(fma(x.re, y.re, -x.im * y.im), fma(x.re, y.im, x.im * y.re)); }
HD double f_abs2(cd a) { return fma(a.re, a.re, a.im * a.im); }
