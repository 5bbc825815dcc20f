// Checks the mma.sync.m8n8k4.f64 fragment layout assumed by the blocked charpoly (dev tool):
//   A (8x4, row): lane l holds A[l>>2][l&3];  B (4x8, col): lane l holds B[l&3][l>>2];
//   C (8x8): lane l holds C[l>>2][2(l&3)+i], i = 0, 1.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* C) {
    const int l = threadIdx.x;
    double a = A[(l >> 2) * 4 + (l & 3)];
    double b = B[(l & 3) * 8 + (l >> 2)];
    double c0 = 0.5, c1 = 0.25;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
    C[(l >> 2) * 8 + 2 * (l & 3)] = c0;
    C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}

int main() {
    double hA[32], hB[32], hC[64];
    for (int i = 0; i < 32; ++i) {
        hA[i] = 1.0 + i * 0.37;
        hB[i] = 2.0 - i * 0.11;
    }
    double *dA, *dB, *dC;
    cudaMalloc(&dA, 256);
    cudaMalloc(&dB, 256);
    cudaMalloc(&dC, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double ref = ((r * 8 + c) % 2 == 0) ? 0.5 : 0.25;
            for (int q = 0; q < 4; ++q) ref += hA[r * 4 + q] * hB[q * 8 + c];
            double e = ref - hC[r * 8 + c];
            if (e < 0) e = -e;
            if (e > maxerr) maxerr = e;
        }
    printf("dmma layout max err %.3e (%s)\n", maxerr, maxerr < 1e-12 ? "OK" : "MISMATCH");
    return maxerr < 1e-12 ? 0 : 1;
}
