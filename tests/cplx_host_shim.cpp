// Host build of the device complex ops (csrc/cplx.cuh) for tests/test_cplx_host.py.
// Compiled with g++ -ffp-contract=off, so the r_* helpers are plain IEEE ops and
// the algorithms can be compared bit for bit against glibc / the oracle.
#include "../paper_1805_12498_b200/csrc/cplx.cuh"

extern "C" {
double shim_hypot(double x, double y) { return m_hypot(x, y); }
void shim_div(const double* a, const double* b, double* out) {
    cd r = m_div(mk(a[0], a[1]), mk(b[0], b[1]));
    out[0] = r.re;
    out[1] = r.im;
}
void shim_rdiv(const double* a, double r, double* out, double* ref) {
    cd x = m_rdiv(mk(a[0], a[1]), r);
    cd y = m_div(mk(a[0], a[1]), mk(r, 0.0));
    out[0] = x.re;
    out[1] = x.im;
    ref[0] = y.re;
    ref[1] = y.im;
}
void shim_sqrt(const double* a, double* out) {
    cd r = m_sqrt(mk(a[0], a[1]));
    out[0] = r.re;
    out[1] = r.im;
}
}
