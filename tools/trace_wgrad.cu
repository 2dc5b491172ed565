// trace_wgrad.cu -- standalone role-timing harness for k_tc2_wgrad<LAY_MX, TANH, 256> (dev tool).
#include <cstdio>
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"
using namespace pnx;
int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 262144, K = 256, N = 256, S = 4;
    float *A, *B, *wp; double* dbp;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&B, (size_t)S * R * N * 4);
    const int tiles = (R + TC_WROWS - 1) / TC_WROWS;
    cudaMalloc(&wp, (size_t)tiles * K * N * 4); cudaMalloc(&dbp, (size_t)tiles * N * 8);
    cudaMemset(A, 0, (size_t)S * R * K * 4); cudaMemset(B, 0, (size_t)S * R * N * 4);
    TcWgradArgs w{}; w.A = A; w.Bm = B; w.wpart = wp; w.dbpart = dbp; w.Rpad = R; w.nrows = R; w.Kin = K; w.N = N;
    using Cfg = Tc2WgCfg<256>;
    const int smem = Cfg::NST * Cfg::STAGE + 1024;
    auto kern = k_tc2_wgrad<LAY_MX, ACT_TANH, 256>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<tiles * 2, TC2_THREADS, smem>>>(w, TC_WROWS);
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) printf("launch error: %s\n", cudaGetErrorString(le));
        cudaEventRecord(e1);
        cudaError_t e = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8];
        cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
        const double ctas = tiles * 2.0;
        printf("%s %.3f ms ctas %d per-CTA cycles: mma_wait_full %.0f prod0_wait_empty %.0f (kernel/CTA %.0f)\n",
               cudaGetErrorString(e), ms, (int)ctas, t[0] / ctas, t[2] / ctas, ms * 1e-3 * 1.965e9 * 148 / ctas);
    }
    return 0;
}
