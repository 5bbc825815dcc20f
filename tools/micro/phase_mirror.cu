// Phase timing of one FAST class kernel (dev tool): -DHAFB_TIMING -DHAFB_S=<S>.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1805_12498_b200/csrc/term_mirror.cuh"
using namespace hafb;
static unsigned long long B[33][33];
unsigned long long cb(unsigned long long x, int p, int D) {
    unsigned long long t = 0; int ones = 0;
    for (int b = D; b >= 0; --b) if ((x >> b) & 1ull) { int need = p - ones; if (need >= 0 && need <= b) t += B[b][need]; if (++ones > p) break; }
    return t;
}
int main(int argc, char** argv) {
    const int D = 26, n = 52, m = HAFB_S / 2;
    for (int b = 0; b <= 32; ++b) for (int p = 0; p <= 32; ++p) B[b][p] = p == 0 ? 1 : (b == 0 ? 0 : B[b-1][p-1] + B[b-1][p]);
    std::vector<cd> at(n * n), dg(n);
    srand(1);
    for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) { cd v = mk((rand() / (double)RAND_MAX - 0.5) / 7, (rand() / (double)RAND_MAX - 0.5) / 7); at[i * n + j] = v; at[j * n + i] = v; }
    for (int i = 0; i < n; ++i) { at[i * n + i] = mk(0, 0); dg[i] = mk(0, 0); }
    unsigned long long lo = 0, hi = 1ull << (argc > 1 ? atoi(argv[1]) : 20);
    Seg sg{lo, hi, 0};
    long long prefix[2] = {0, (long long)(cb(hi, m, D) - cb(lo, m, D))};
    unsigned long long base[1] = {cb(lo, m, D)};
    cd *d_at, *d_dg, *d_t; int8_t* d_s; Seg* d_seg; long long* d_pre; unsigned long long *d_base, *d_binom;
    cudaMalloc(&d_at, sizeof(cd) * n * n); cudaMalloc(&d_dg, sizeof(cd) * n);
    cudaMalloc(&d_t, sizeof(cd) * hi); cudaMalloc(&d_s, hi); cudaMalloc(&d_seg, sizeof(Seg));
    cudaMalloc(&d_pre, 16); cudaMalloc(&d_base, 8); cudaMalloc(&d_binom, sizeof(B));
    cudaMemcpy(d_at, at.data(), sizeof(cd) * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(d_dg, dg.data(), sizeof(cd) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(d_seg, &sg, sizeof(Seg), cudaMemcpyHostToDevice);
    cudaMemcpy(d_pre, prefix, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_base, base, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_binom, B, sizeof(B), cudaMemcpyHostToDevice);
    ClassItems ci{B[D - 1][m], d_seg, d_pre, d_base, 1, m, D, prefix[1], prefix[1], 0, 0, 0, nullptr, nullptr, sg, base[0]};
    constexpr int W = TeamWidth<HAFB_S>::W, TPB = mirror_tpb<HAFB_S>(), NT = TPB * W;
    size_t smem = (size_t)TPB * MirrorLayout<HAFB_S>::TOTAL * sizeof(cd);
    auto k = mirror_term_kernel<HAFB_S, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
    int grid = 148 * occ;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<grid, NT, smem>>>(d_at, d_dg, D, ci, d_t, d_s);
    cudaDeviceSynchronize();
#ifdef HAFB_TIMING
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z)); cudaMemcpyToSymbol(g_phase_cnt, z, sizeof(z));
#endif
    cudaEventRecord(e0);
    k<<<grid, NT, smem>>>(d_at, d_dg, D, ci, d_t, d_s);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[16] = {0}, pc[16] = {0};
#ifdef HAFB_TIMING
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph)); cudaMemcpyFromSymbol(pc, g_phase_cnt, sizeof(pc));
#endif
    printf("S=%d items=%lld grid=%d occ=%d time=%.3f ms err=%s\n", HAFB_S, prefix[1], grid, occ, ms, cudaGetErrorString(cudaGetLastError()));
    const char* names[16] = {"gather", "hessenberg", "charpoly", "newton+series", "exp+store", "h:shfl", "h:relabel+Hs", "h:inv+mu", "h:argmax", "h:shfl+lm+swap", "h:inv+mu+sync", "h:sweep", "h:shift", "EMPTY(mark cost)"};
    unsigned long long items = pc[0];
    for (int i = 0; i < 14; ++i) if (pc[i]) printf("  %-20s %10.0f cycles/item  (%llu marks)\n", names[i], (double)ph[i] / items, pc[i]);
    return 0;
}
