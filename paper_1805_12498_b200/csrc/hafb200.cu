// hafb200.cu -- C ABI (include/hafb200.h) over the sm_100a hafnian kernels.
//
// Host side of the drop-in boundary: argument checks, per-call stream and
// stream-ordered buffers, kernel launches, status collection.  No global
// mutable state except the per-thread error string and launch counter.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hafb200.h"
#include "cplx.cuh"
#include "reduce.cuh"
#include "term_smem.cuh"

using namespace hafb;

namespace {

thread_local std::string g_err;
thread_local long long g_launches = 0;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(const char* what, cudaError_t e) {
    return fail(HAFB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_); \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int check_common(int n_half, int backend, int arith) {
    if (n_half < 1 || n_half > kMaxHalf) return fail(HAFB_ERR_ARG, "n_half must be in [1, 31]");
    if (backend != 0 && backend != 1) return fail(HAFB_ERR_ARG, "backend must be 0 or 1");
    if (arith != 0 && arith != 1) return fail(HAFB_ERR_ARG, "arith must be 0 or 1");
    return HAFB_OK;
}

// One host call: its own non-blocking stream and stream-ordered allocations,
// released (after a stream sync) when the call returns on any path.
struct Call {
    cudaStream_t st = nullptr;
    std::vector<void*> bufs;
    cudaError_t open(int device) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return e;
        return cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    }
    template <class T>
    cudaError_t alloc(T** p, size_t bytes) {
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(bytes, 16), st);
        if (e == cudaSuccess) bufs.push_back(q);
        *p = static_cast<T*>(q);
        return e;
    }
    ~Call() {
        if (!st) return;
        for (void* p : bufs) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
};

int sm_count() {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

template <int B, bool L>
cudaError_t launch_terms_t(const cd* at, const cd* dg, int n_half, MaskMap map, long long per,
                           long long total, int cap, long long at_stride, long long dg_stride,
                           cd* terms, int8_t* status, cudaStream_t st) {
    const int n = 2 * n_half;
    size_t per_warp = (size_t)smem_warp_elems(n) * sizeof(cd);
    int wpb = (int)std::min<size_t>(8, std::max<size_t>(1, (200 * 1024) / per_warp));
    size_t smem = wpb * per_warp;
    auto kern = terms_smem_kernel<B, L>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, wpb * 32, smem);
    if (e != cudaSuccess) return e;
    long long want = (total + wpb - 1) / wpb;
    long long cap_blocks = (long long)sm_count() * std::max(occ, 1);
    int grid = (int)std::max<long long>(1, std::min(want, cap_blocks));
    kern<<<grid, wpb * 32, smem, st>>>(at, dg, n_half, map, per, total, cap, at_stride, dg_stride,
                                       terms, status);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_terms(int backend, int loops, const cd* at, const cd* dg, int n_half,
                         MaskMap map, long long per, long long total, int cap, long long at_stride,
                         long long dg_stride, cd* terms, int8_t* status, cudaStream_t st) {
#define LT(B, L) \
    launch_terms_t<B, L>(at, dg, n_half, map, per, total, cap, at_stride, dg_stride, terms, status, st)
    if (backend == 1) return loops ? LT(1, true) : LT(1, false);
    return loops ? LT(0, true) : LT(0, false);
#undef LT
}

MaskMap plain_map(uint64_t lo) {
    MaskMap m;
    m.lo = lo;
    m.mask_list = nullptr;
    m.range_list = nullptr;
    m.width = 1;
    m.total = 0;
    return m;
}

size_t terms_ws_bytes(long long count) {
    return align256((size_t)count * sizeof(cd)) + align256((size_t)std::max<long long>(count, 1));
}

void carve_terms_ws(void* base, long long count, cd** terms, int8_t** status) {
    char* p = static_cast<char*>(base);
    *terms = reinterpret_cast<cd*>(p);
    *status = reinterpret_cast<int8_t*>(p + align256((size_t)count * sizeof(cd)));
}

uint64_t std_width(int n_half, int n_ranges) {
    uint64_t nterms = (1ull << n_half) - 1;
    return (nterms + n_ranges - 1) / n_ranges;
}

// enqueue: terms over masks [lo, hi), Kahan per chunk -> partials
int enqueue_mask_range(const cd* at, const cd* dg, int n_half, uint64_t lo, uint64_t hi,
                       int n_chunks, int backend, int loops, int cap, int arith, void* ws,
                       size_t ws_bytes, cd* partials, long long* fails, cudaStream_t st) {
    (void)arith;
    long long count = (long long)(hi - lo);
    if (ws_bytes < terms_ws_bytes(count)) return fail(HAFB_ERR_ARG, "workspace too small");
    cd* terms;
    int8_t* status;
    carve_terms_ws(ws, count, &terms, &status);
    if (count > 0)
        CK(launch_terms(backend, loops, at, dg, n_half, plain_map(lo), count, count, cap, 0, 0,
                        terms, status, st));
    uint64_t width = (hi - lo + n_chunks - 1) / n_chunks;
    int thr = 128;
    range_kahan_kernel<<<(n_chunks + thr - 1) / thr, thr, 0, st>>>(terms, status, lo, hi, width,
                                                                     n_chunks, 1, count, partials,
                                                                     fails);
    ++g_launches;
    CK(cudaGetLastError());
    return HAFB_OK;
}

// enqueue: terms over the listed standard ranges, Kahan per range -> partials[i]
int enqueue_range_list(const cd* at, const cd* dg, int n_half, int n_ranges, const int32_t* d_ranges,
                       int count, int backend, int loops, int cap, int arith, void* ws,
                       size_t ws_bytes, cd* partials, long long* fails, cudaStream_t st) {
    (void)arith;
    uint64_t width = std_width(n_half, n_ranges);
    long long items = (long long)count * (long long)width;
    if (ws_bytes < terms_ws_bytes(items)) return fail(HAFB_ERR_ARG, "workspace too small");
    cd* terms;
    int8_t* status;
    carve_terms_ws(ws, items, &terms, &status);
    MaskMap map;
    map.lo = 0;
    map.mask_list = nullptr;
    map.range_list = d_ranges;
    map.width = width;
    map.total = 1ull << n_half;
    if (items > 0)
        CK(launch_terms(backend, loops, at, dg, n_half, map, items, items, cap, 0, 0, terms, status,
                        st));
    int thr = 128;
    list_kahan_kernel<<<(count + thr - 1) / thr, thr, 0, st>>>(terms, status, d_ranges, count, width,
                                                               1ull << n_half, partials, fails);
    ++g_launches;
    CK(cudaGetLastError());
    return HAFB_OK;
}

// single-warp kernels for the power-trace entry points
__global__ void power_traces_kernel(const cd* b, int m, int K, int backend, int cap_mult,
                                    cd* traces, int* ok, cd* ws) {
    int lane = threadIdx.x & 31;
    WarpWs w = carve(ws, m + (m & 1));
    for (int e = lane; e < m * m; e += 32) w.H[e] = b[e];
    __syncwarp();
    if (backend == 1) {
        hess_smem(w.H, m, lane);
        charpoly_smem(w.H, m, w.P, lane);
        if (lane == 0) {
            const cd* a = w.P + m * (m + 1) / 2;
            *ok = traces_from_charpoly_seq(a, m, K, traces) ? 1 : 0;
        }
    } else {
        bool conv = hess_eigvals_smem(w.H, m, cap_mult, w.eig, lane);
        __syncwarp();
        if (lane == 0) {
            // _power_sums (_numba.py:191-200)
            for (int k = 0; k < K; ++k) traces[k] = mk(0.0, 0.0);
            for (int i = 0; i < m; ++i) {
                cd lam = w.eig[i], p = lam;
                for (int k = 0; k < K; ++k) {
                    traces[k] = m_add(traces[k], p);
                    p = m_mul(p, lam);
                }
            }
            *ok = conv ? 1 : 0;
        }
    }
}

__global__ void charpoly_coeffs_kernel(const cd* b, int m, cd* out, cd* ws) {
    int lane = threadIdx.x & 31;
    WarpWs w = carve(ws, m + (m & 1));
    for (int e = lane; e < m * m; e += 32) w.H[e] = b[e];
    __syncwarp();
    hess_smem(w.H, m, lane);
    charpoly_smem(w.H, m, w.P, lane);
    const cd* a = w.P + m * (m + 1) / 2;
    for (int d = lane; d <= m; d += 32) out[d] = a[d];
}

}  // namespace

extern "C" {

int hafb_abi_version(void) { return 1; }

const char* hafb_last_error(void) { return g_err.c_str(); }

int hafb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int64_t hafb_launch_count(int reset) {
    long long v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

size_t hafb_range_workspace_bytes(int n_half, uint64_t lo, uint64_t hi, int n_chunks) {
    (void)n_half;
    (void)n_chunks;
    if (hi < lo) return 0;
    return terms_ws_bytes((long long)(hi - lo));
}

size_t hafb_range_list_workspace_bytes(int n_half, int n_ranges, int count) {
    if (n_half < 1 || n_half > kMaxHalf || n_ranges < 1 || count < 0) return 0;
    return terms_ws_bytes((long long)count * (long long)std_width(n_half, n_ranges));
}

int hafb_sum_mask_range_async(const double* d_atilde, const double* d_diag, int n_half,
                              uint64_t lo, uint64_t hi, int n_chunks, int backend,
                              int include_loops, int cap_mult, int arith, void* d_workspace,
                              size_t workspace_bytes, double* d_partials, int64_t* d_fails,
                              void* stream) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (hi < lo || hi > (1ull << n_half) || n_chunks < 1) return fail(HAFB_ERR_ARG, "bad mask range");
    return enqueue_mask_range(reinterpret_cast<const cd*>(d_atilde),
                              reinterpret_cast<const cd*>(d_diag), n_half, lo, hi, n_chunks,
                              backend, include_loops, cap_mult, arith, d_workspace, workspace_bytes,
                              reinterpret_cast<cd*>(d_partials),
                              reinterpret_cast<long long*>(d_fails),
                              static_cast<cudaStream_t>(stream));
}

int hafb_sum_range_list_async(const double* d_atilde, const double* d_diag, int n_half,
                              int n_ranges, const int32_t* d_ranges, int count, int backend,
                              int include_loops, int cap_mult, int arith, void* d_workspace,
                              size_t workspace_bytes, double* d_partials, int64_t* d_fails,
                              void* stream) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (n_ranges < 1 || count < 0) return fail(HAFB_ERR_ARG, "bad range list");
    if (count == 0) return HAFB_OK;
    return enqueue_range_list(reinterpret_cast<const cd*>(d_atilde),
                              reinterpret_cast<const cd*>(d_diag), n_half, n_ranges, d_ranges, count,
                              backend, include_loops, cap_mult, arith, d_workspace, workspace_bytes,
                              reinterpret_cast<cd*>(d_partials),
                              reinterpret_cast<long long*>(d_fails),
                              static_cast<cudaStream_t>(stream));
}

int hafb_sum_mask_range(const double* atilde, const double* diag, int n_half, uint64_t lo,
                        uint64_t hi, int n_chunks, int backend, int include_loops, int cap_mult,
                        int arith, int device, double* partials, int64_t* fails) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (hi < lo || hi > (1ull << n_half) || n_chunks < 1) return fail(HAFB_ERR_ARG, "bad mask range");
    const int n = 2 * n_half;
    size_t ws_bytes = terms_ws_bytes((long long)(hi - lo));
    Call c;
    cd *d_at, *d_dg, *d_part;
    long long* d_fail;
    void* d_ws;
    CK(c.open(device));
    CK(c.alloc(&d_at, sizeof(cd) * n * n));
    CK(c.alloc(&d_dg, sizeof(cd) * n));
    CK(c.alloc(&d_ws, ws_bytes));
    CK(c.alloc(&d_part, sizeof(cd) * n_chunks));
    CK(c.alloc(&d_fail, sizeof(long long) * n_chunks));
    CK(cudaMemcpyAsync(d_at, atilde, sizeof(cd) * n * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_dg, diag, sizeof(cd) * n, cudaMemcpyHostToDevice, c.st));
    rc = enqueue_mask_range(d_at, d_dg, n_half, lo, hi, n_chunks, backend, include_loops, cap_mult,
                            arith, d_ws, ws_bytes, d_part, d_fail, c.st);
    if (rc) return rc;
    CK(cudaMemcpyAsync(partials, d_part, sizeof(cd) * n_chunks, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(fails, d_fail, sizeof(long long) * n_chunks, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return HAFB_OK;
}

int hafb_sum_range_list(const double* atilde, const double* diag, int n_half, int n_ranges,
                        const int32_t* ranges, int count, int backend, int include_loops,
                        int cap_mult, int arith, int device, double* partials, int64_t* fails) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (n_ranges < 1 || count < 0) return fail(HAFB_ERR_ARG, "bad range list");
    for (int i = 0; i < count; ++i)
        if (ranges[i] < 0 || ranges[i] >= n_ranges) return fail(HAFB_ERR_ARG, "range index out of bounds");
    if (count == 0) return HAFB_OK;
    const int n = 2 * n_half;
    size_t ws_bytes = hafb_range_list_workspace_bytes(n_half, n_ranges, count);
    Call c;
    cd *d_at, *d_dg, *d_part;
    long long* d_fail;
    int32_t* d_r;
    void* d_ws;
    CK(c.open(device));
    CK(c.alloc(&d_at, sizeof(cd) * n * n));
    CK(c.alloc(&d_dg, sizeof(cd) * n));
    CK(c.alloc(&d_r, sizeof(int32_t) * count));
    CK(c.alloc(&d_ws, ws_bytes));
    CK(c.alloc(&d_part, sizeof(cd) * count));
    CK(c.alloc(&d_fail, sizeof(long long) * count));
    CK(cudaMemcpyAsync(d_at, atilde, sizeof(cd) * n * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_dg, diag, sizeof(cd) * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_r, ranges, sizeof(int32_t) * count, cudaMemcpyHostToDevice, c.st));
    rc = enqueue_range_list(d_at, d_dg, n_half, n_ranges, d_r, count, backend, include_loops,
                            cap_mult, arith, d_ws, ws_bytes, d_part, d_fail, c.st);
    if (rc) return rc;
    CK(cudaMemcpyAsync(partials, d_part, sizeof(cd) * count, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(fails, d_fail, sizeof(long long) * count, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return HAFB_OK;
}

int hafb_sum_subsets_det(const double* atilde, const double* diag, int n_half, int backend,
                         int include_loops, int n_ranges, int cap_mult, int arith, int device,
                         double* partials, int64_t* fails) {
    if (n_half < 1 || n_half > kMaxHalf) return fail(HAFB_ERR_ARG, "n_half must be in [1, 31]");
    if (n_ranges < 1) return fail(HAFB_ERR_ARG, "n_ranges must be >= 1");
    // the standard ranges are the mask-range chunks of [1, 2^D) (same width, same bounds)
    uint64_t total = 1ull << n_half;
    return hafb_sum_mask_range(atilde, diag, n_half, 1, total, n_ranges, backend, include_loops,
                               cap_mult, arith, device, partials, fails);
}

int hafb_sum_subsets_fast(const double* atilde, const double* diag, int n_half, int backend,
                          int include_loops, int workers, int n_ranges, int cap_mult, int arith,
                          int device, double* wsums, int64_t* wfails) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (workers < 1 || n_ranges < 1) return fail(HAFB_ERR_ARG, "workers and n_ranges must be >= 1");
    const int n = 2 * n_half;
    const uint64_t total = 1ull << n_half;
    const long long count = (long long)(total - 1);
    const uint64_t width = std_width(n_half, n_ranges);
    size_t ws_bytes = terms_ws_bytes(count);
    Call c;
    cd *d_at, *d_dg, *d_sum, *terms;
    long long* d_fail;
    int8_t* status;
    void* d_ws;
    CK(c.open(device));
    CK(c.alloc(&d_at, sizeof(cd) * n * n));
    CK(c.alloc(&d_dg, sizeof(cd) * n));
    CK(c.alloc(&d_ws, ws_bytes));
    CK(c.alloc(&d_sum, sizeof(cd) * workers));
    CK(c.alloc(&d_fail, sizeof(long long) * workers));
    CK(cudaMemcpyAsync(d_at, atilde, sizeof(cd) * n * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_dg, diag, sizeof(cd) * n, cudaMemcpyHostToDevice, c.st));
    carve_terms_ws(d_ws, count, &terms, &status);
    CK(launch_terms(backend, include_loops, d_at, d_dg, n_half, plain_map(1), count, count,
                    cap_mult, 0, 0, terms, status, c.st));
    worker_kahan_kernel<<<(workers + 127) / 128, 128, 0, c.st>>>(terms, status, total, width,
                                                                 n_ranges, workers, d_sum, d_fail);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(wsums, d_sum, sizeof(cd) * workers, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(wfails, d_fail, sizeof(long long) * workers, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return HAFB_OK;
}

int hafb_terms(const double* atilde, const double* diag, int n_half, const uint64_t* masks,
               int64_t count, int backend, int include_loops, int cap_mult, int arith, int device,
               double* terms, int32_t* status) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (count <= 0) return HAFB_OK;
    const int n = 2 * n_half;
    std::vector<uint32_t> h_masks(count);
    std::vector<int8_t> h_st(count);
    for (int64_t q = 0; q < count; ++q) {
        if (masks[q] == 0 || masks[q] >= (1ull << n_half)) return fail(HAFB_ERR_ARG, "mask out of range");
        h_masks[q] = (uint32_t)masks[q];
    }
    Call c;
    cd *d_at, *d_dg, *d_t;
    uint32_t* d_m;
    int8_t* d_s;
    CK(c.open(device));
    CK(c.alloc(&d_at, sizeof(cd) * n * n));
    CK(c.alloc(&d_dg, sizeof(cd) * n));
    CK(c.alloc(&d_m, sizeof(uint32_t) * count));
    CK(c.alloc(&d_t, sizeof(cd) * count));
    CK(c.alloc(&d_s, count));
    CK(cudaMemcpyAsync(d_at, atilde, sizeof(cd) * n * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_dg, diag, sizeof(cd) * n, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_m, h_masks.data(), sizeof(uint32_t) * count, cudaMemcpyHostToDevice, c.st));
    MaskMap map = plain_map(0);
    map.mask_list = d_m;
    CK(launch_terms(backend, include_loops, d_at, d_dg, n_half, map, count, count, cap_mult, 0, 0,
                    d_t, d_s, c.st));
    CK(cudaMemcpyAsync(terms, d_t, sizeof(cd) * count, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(h_st.data(), d_s, count, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    for (int64_t q = 0; q < count; ++q) status[q] = h_st[q];
    return HAFB_OK;
}

int hafb_batch(const double* atilde, const double* diag, int batch, int n_half, int backend,
               int include_loops, int n_ranges, int cap_mult, int arith, int device,
               double* results, int64_t* fails) {
    g_err.clear();
    int rc = check_common(n_half, backend, arith);
    if (rc) return rc;
    if (batch <= 0) return HAFB_OK;
    if (n_ranges < 1) return fail(HAFB_ERR_ARG, "n_ranges must be >= 1");
    const int n = 2 * n_half;
    const uint64_t total = 1ull << n_half;
    const long long per = (long long)(total - 1);
    const size_t cnt = (size_t)batch * per;
    const uint64_t width = std_width(n_half, n_ranges);
    std::vector<long long> h_fail((size_t)batch * n_ranges);
    Call c;
    cd *d_at, *d_dg, *d_t, *d_part, *d_res;
    int8_t* d_s;
    long long* d_fail;
    CK(c.open(device));
    CK(c.alloc(&d_at, sizeof(cd) * n * n * (size_t)batch));
    CK(c.alloc(&d_dg, sizeof(cd) * n * (size_t)batch));
    CK(c.alloc(&d_t, sizeof(cd) * cnt));
    CK(c.alloc(&d_s, cnt));
    CK(c.alloc(&d_part, sizeof(cd) * n_ranges * (size_t)batch));
    CK(c.alloc(&d_fail, sizeof(long long) * n_ranges * (size_t)batch));
    CK(c.alloc(&d_res, sizeof(cd) * batch));
    CK(cudaMemcpyAsync(d_at, atilde, sizeof(cd) * n * n * (size_t)batch, cudaMemcpyHostToDevice, c.st));
    CK(cudaMemcpyAsync(d_dg, diag, sizeof(cd) * n * (size_t)batch, cudaMemcpyHostToDevice, c.st));
    CK(launch_terms(backend, include_loops, d_at, d_dg, n_half, plain_map(1), per, (long long)cnt,
                    cap_mult, (long long)n * n, n, d_t, d_s, c.st));
    // problem b's term for mask q+1 sits at b*per + q: the reduce runs with lo = 1
    {
        int thr = 128;
        int blocks = (int)(((long long)n_ranges * batch + thr - 1) / thr);
        range_kahan_kernel<<<blocks, thr, 0, c.st>>>(d_t, d_s, 1, total, width, n_ranges, batch,
                                                     per, d_part, d_fail);
        ++g_launches;
        CK(cudaGetLastError());
    }
    tree_reduce_kernel<<<(batch + 127) / 128, 128, 0, c.st>>>(d_part, n_ranges, batch, d_res);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(results, d_res, sizeof(cd) * batch, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(h_fail.data(), d_fail, sizeof(long long) * n_ranges * (size_t)batch,
                       cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    for (int b = 0; b < batch; ++b) {
        long long mx = 0;
        for (int r = 0; r < n_ranges; ++r) mx = std::max(mx, h_fail[(size_t)b * n_ranges + r]);
        fails[b] = mx;
    }
    return HAFB_OK;
}

int hafb_power_traces(const double* b, int m, int K, int backend, int cap_mult, int arith,
                      int device, double* traces, int64_t* sweeps, int32_t* ok) {
    g_err.clear();
    if (m < 1 || m > 2 * kMaxHalf) return fail(HAFB_ERR_ARG, "m must be in [1, 62]");
    if (K < 1) return fail(HAFB_ERR_ARG, "K must be >= 1");
    if (backend != 0 && backend != 1) return fail(HAFB_ERR_ARG, "backend must be 0 or 1");
    (void)arith;
    int mm = m + (m & 1);
    size_t ws_elems = (size_t)smem_warp_elems(mm);
    Call c;
    cd *d_b, *d_t, *d_ws;
    int* d_ok;
    int h_ok = 0;
    CK(c.open(device));
    CK(c.alloc(&d_b, sizeof(cd) * m * m));
    CK(c.alloc(&d_t, sizeof(cd) * K));
    CK(c.alloc(&d_ok, sizeof(int)));
    CK(c.alloc(&d_ws, sizeof(cd) * ws_elems));
    CK(cudaMemcpyAsync(d_b, b, sizeof(cd) * m * m, cudaMemcpyHostToDevice, c.st));
    power_traces_kernel<<<1, 32, 0, c.st>>>(d_b, m, K, backend, cap_mult, d_t, d_ok, d_ws);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(traces, d_t, sizeof(cd) * K, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(&h_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    *sweeps = -1;  // the QR sweep count is not tracked on the device
    *ok = h_ok;
    return HAFB_OK;
}

int hafb_charpoly_coefficients(const double* b, int m, int arith, int device, double* coeffs) {
    g_err.clear();
    if (m < 1 || m > 2 * kMaxHalf) return fail(HAFB_ERR_ARG, "m must be in [1, 62]");
    (void)arith;
    int mm = m + (m & 1);
    Call c;
    cd *d_b, *d_o, *d_ws;
    CK(c.open(device));
    CK(c.alloc(&d_b, sizeof(cd) * m * m));
    CK(c.alloc(&d_o, sizeof(cd) * (m + 1)));
    CK(c.alloc(&d_ws, sizeof(cd) * smem_warp_elems(mm)));
    CK(cudaMemcpyAsync(d_b, b, sizeof(cd) * m * m, cudaMemcpyHostToDevice, c.st));
    charpoly_coeffs_kernel<<<1, 32, 0, c.st>>>(d_b, m, d_o, d_ws);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(coeffs, d_o, sizeof(cd) * (m + 1), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    return HAFB_OK;
}

}  // extern "C"
