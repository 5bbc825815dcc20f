// FP64 tensor (mma.sync.m8n8k4.f64) vs DFMA throughput on one B200, alone and mixed (dev tool).
// Prints TF/s over the whole GPU for: DFMA only, DMMA only, and a warp mix of both.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// MODE 0: DFMA chains; 1: DMMA chains; 2: both in every warp (CH each)
template <int MODE, int CH>
__global__ void bench(double* out, int iters, double a, double b) {
    double x[CH];
    double c[CH][2];
    for (int i = 0; i < CH; ++i) {
        x[i] = threadIdx.x + i;
        c[i][0] = i;
        c[i][1] = threadIdx.x;
    }
    const double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (MODE != 1) x[i] = fma(x[i], a, b);
            if (MODE != 0) dmma(c[i], av, bv);
        }
    }
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i] + c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int MODE, int CH>
void run(int warps_per_block, int blocks_per_sm, int sms) {
    double* o;
    cudaMalloc(&o, 8);
    const int iters = 20000;
    const int blocks = blocks_per_sm * sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<MODE, CH><<<blocks, 32 * warps_per_block>>>(o, 100, 1.0, 1e-9);
    cudaEventRecord(e0);
    bench<MODE, CH><<<blocks, 32 * warps_per_block>>>(o, iters, 0.9999999, 1e-12);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * warps_per_block;
    const double fma_flop = (MODE != 1) ? warps * 32 * CH * (double)iters * 2 : 0;
    const double mma_flop = (MODE != 0) ? warps * CH * (double)iters * 8 * 8 * 4 * 2 : 0;
    printf("mode=%d ch=%d warps/SM=%d: %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n", MODE, CH,
           warps_per_block * blocks_per_sm, ms, fma_flop / ms / 1e9, mma_flop / ms / 1e9,
           (fma_flop + mma_flop) / ms / 1e9);
    cudaFree(o);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    run<0, 8>(4, 4, sms);
    run<0, 8>(8, 2, sms);
    run<1, 4>(4, 4, sms);
    run<1, 8>(4, 4, sms);
    run<1, 8>(8, 2, sms);
    run<1, 2>(4, 1, sms);
    run<1, 4>(4, 1, sms);
    run<2, 4>(4, 4, sms);
    run<2, 8>(4, 4, sms);
    run<2, 8>(8, 2, sms);
    return 0;
}
