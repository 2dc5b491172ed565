// trace_bwd.cu -- role-timing harness for k_tc2_bwd<LAY_MX, 128> (dev tool).
#include <cstdio>
#include <vector>
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"
using namespace pnx;
int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 262144, K = 256, N = 256, S = 4;
    float *A, *Z, *W, *img, *out;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&Z, (size_t)S * R * N * 4); cudaMalloc(&out, (size_t)S * R * N * 4);
    cudaMalloc(&W, K * N * 4); cudaMalloc(&img, 2 * K * N * 4);
    cudaMemset(A, 0, (size_t)S * R * K * 4); cudaMemset(Z, 0, (size_t)S * R * N * 4); cudaMemset(W, 0, K * N * 4);
    k_tc_prep_image<<<256, 256>>>(W, K, N, 1, 128, img);
    TcGemmArgs g{}; g.A = A; g.img = img; g.Zlow = Z; g.out = out; g.Rpad = R; g.K = K; g.N = N;
    using Cfg = Tc2BwdCfg<4, 128>;
    const int smem = Cfg::SMEM;
    auto kern = k_tc2_bwd<LAY_MX, 128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<(R / 128) * (N / 128), TC3_THREADS, smem>>>(g);
        cudaError_t le = cudaGetLastError();
        if (le != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(le));
        cudaEventRecord(e1);
        cudaError_t e = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8];
        cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
        const double ctas = (R / 128.0) * 2;
        printf("%s %.3f ms ctas %d per-CTA: mma_wait_full %.0f epi_busy %.0f (kernel/CTA %.0f)\n", cudaGetErrorString(e), ms,
               (int)ctas, t[0] / ctas, t[3] / ctas, ms * 1e-3 * 1.965e9 * 148 / ctas);
    }
    return 0;
}
