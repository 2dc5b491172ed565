// trace_fwd.cu -- standalone harness: runs k_tc2_fwd<LAY_MX, TANH, 256> on random
// data with -DPNX_TC_TRACE and prints per-role cycle totals (dev tool).
#include <cstdio>
#include <vector>
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"
using namespace pnx;
int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 262144, K = 256, N = 256, S = 4;
    float *A, *W, *img, *bias, *out;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&out, (size_t)S * R * N * 4);
    cudaMalloc(&W, K * N * 4); cudaMalloc(&img, 2 * K * N * 4); cudaMalloc(&bias, N * 4);
    std::vector<float> h((size_t)K * N);
    for (auto& x : h) x = (rand() / (float)RAND_MAX - 0.5f) * 0.1f;
    cudaMemcpy(W, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(A, 0, (size_t)S * R * K * 4); cudaMemset(bias, 0, N * 4);
    k_tc_prep_image<<<256, 256>>>(W, K, N, 0, N, img);
    TcGemmArgs g{}; g.A = A; g.img = img; g.bias = bias; g.out = out; g.Rpad = R; g.K = K; g.N = N;
    using Cfg = Tc3FwdCfg<256>;
    const int smem = Cfg::SMEM;
    auto kern = k_tc2_fwd<LAY_MX, ACT_TANH, 256>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kern<<<R / 128, TC3_THREADS, smem>>>(g);
        cudaEventRecord(e1);
        cudaError_t e = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long t[8];
        cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
        const double ctas = R / 128.0;
        printf("%s  %.3f ms  tiles %d  per-tile cycles: mma_wait_full %.0f  mma_wait_tmem %.0f  prod0_wait_empty %.0f  epi_busy %.0f  (kernel/tile at 1.965GHz*148/tiles: %.0f)\n",
               cudaGetErrorString(e), ms, (int)ctas, t[0] / ctas, t[1] / ctas, t[2] / ctas, t[3] / ctas,
               ms * 1e-3 * 1.965e9 * 148 / ctas);
    }
    return 0;
}
