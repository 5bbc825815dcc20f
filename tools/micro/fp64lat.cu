// FP64 latency / per-warp throughput microbenchmark (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chains(double* out, int iters, double a, double b, long long* cyc) {
    double x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH>
void run(int warps) {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    int iters = 4096;
    chains<CH><<<1, 32 * warps>>>(o, iters, 0.9999, 1e-9, c);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("chains=%d warps/SM=%d : %.2f cycles per dependent DFMA step, %.3f warp-DFMA/cycle/SM\n", CH, warps,
           (double)h / iters, (double)CH * warps * iters / h);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<1>(4); run<2>(4); run<4>(4); run<8>(4); run<1>(8); run<2>(8); run<4>(8); run<1>(16); run<2>(16);
    return 0;
}
