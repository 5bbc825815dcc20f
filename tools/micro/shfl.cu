// SHFL / broadcast-LDS.128 / DFMA issue-mix throughput per SM (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void shfl_k(double* out, int iters, long long* cyc) {
    unsigned x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __shfl_sync(0xffffffffu, x[i], (x[i] + it) & 31);
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345) out[0] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds_k(double* out, int iters, long long* cyc) {
    __shared__ double2 buf[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = make_double2(i, i);
    __syncthreads();
    double2 acc[4] = {};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) { double2 v = buf[(it * 4 + i) & 255]; acc[i].x += v.x; acc[i].y += v.y; }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 4; ++i) s += acc[i].x + acc[i].y;
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void mix_k(double* out, int iters, long long* cyc) {
    // 8 DFMA + 4 SHFL per unit (the sweep's column mix)
    double a[8]; unsigned x[4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int i = 0; i < 4; ++i) x[i] = threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __shfl_sync(0xffffffffu, x[i], 3);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999, (double)x[i & 3]);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    int iters = 4096; long long h;
    for (int w : {1, 4, 8, 12, 16}) {
        shfl_k<<<1, 32 * w>>>(o, iters, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("SHFL   warps=%2d: %.3f warp-SHFL/cycle/SM\n", w, 8.0 * w * iters / h);
        lds_k<<<1, 32 * w>>>(o, iters, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("LDS128 warps=%2d: %.3f warp-LDS.128(bcast)/cycle/SM\n", w, 4.0 * w * iters / h);
        mix_k<<<1, 32 * w>>>(o, iters, c); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("MIX    warps=%2d: %.3f warp-DFMA/cycle/SM (8 DFMA + 4 SHFL units)\n", w, 8.0 * w * iters / h);
    }
    return 0;
}
