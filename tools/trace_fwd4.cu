// trace_fwd4.cu -- CTA-pair forward (k_tc4_fwd) vs single-CTA forward (k_tc2_fwd):
// cross-check on random data + timing (dev tool).
#include <cstdio>
#include <vector>
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"
#include "../paper_2604_15645_b200/csrc/launch_tc.cu"
using namespace pnx;
__global__ void fill(float* p, size_t n, unsigned seed, float scale) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = ((h & 0xFFFFFF) / 16777216.0f - 0.5f) * scale;
    }
}
int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 262144, K = 256, N = 256, S = 4;
    float *A, *W, *bias, *img, *out;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&out, (size_t)S * R * N * 4);
    cudaMalloc(&W, K * N * 4); cudaMalloc(&bias, N * 4); cudaMalloc(&img, 2 * K * N * 4);
    fill<<<1024, 256>>>(A, (size_t)S * R * K, 3u, 1.6f);
    fill<<<64, 256>>>(W, K * N, 5u, 0.15f);
    fill<<<1, 256>>>(bias, N, 9u, 0.2f);
    k_tc_prep_image<<<256, 256>>>(W, K, N, 0, N, img);
    // 3xFP16 inputs: bounds (|A| <= 0.8, |W| <= 0.075) and the fp16 weight image
    unsigned* amax; uint16_t* img16;
    cudaMalloc(&amax, 8 * 4); cudaMalloc(&img16, 2 * K * N * 2);
    const float am[8] = {0.8f, 0.8f, 0.8f, 0.8f, 0.075f, 0, 0, 0};
    cudaMemcpy(amax, am, sizeof(am), cudaMemcpyHostToDevice);
    k_tc_prep_image16<<<256, 256>>>(W, K, N, 0, N, amax + 4, img16);
    TcGemmArgs g{}; g.A = A; g.img = img; g.bias = bias; g.out = out; g.Rpad = R; g.K = K; g.N = N;
    g.amax_in = amax; g.amax_w = amax + 4;
    std::vector<float> ref((size_t)S * R * N), got((size_t)S * R * N), got16((size_t)S * R * N);
    for (int mode = 0; mode < 3; ++mode) {
        g.img = mode == 2 ? reinterpret_cast<float*>(img16) : img;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(out, 0, (size_t)S * R * N * 4);
            unsigned long long z[8] = {0};
            cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int rc = mode == 2 ? launch_tc4_fwd_t<LAY_MX, ACT_TANH, true>(g, 0)
                         : mode ? launch_tc4_fwd_t<LAY_MX, ACT_TANH, false>(g, 0) : launch_tc2_fwd_t<LAY_MX, ACT_TANH, 256>(g, 0);
            cudaError_t le = cudaGetLastError();
            if (rc || le != cudaSuccess) printf("launch rc=%d %s\n", rc, cudaGetErrorString(le));
            cudaEventRecord(e1);
            cudaError_t e = cudaDeviceSynchronize();
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long t[8];
            cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
            const double ctas = R / 128.0;
            printf("%s %s %.3f ms  per-CTA: mma_wait_full %.0f mma_wait_tmem %.0f conv0_wait_empty %.0f conv0_wait_raw %.0f epi %.0f  (kernel/CTA-slot %.0f)\n",
                   mode == 2 ? "pair16" : mode ? "pair  " : "single",
                   cudaGetErrorString(e), ms, t[0] / ctas, t[1] / ctas, t[2] / ctas, t[5] / ctas, t[3] / ctas, ms * 1e-3 * 1.965e9 * 148 / ctas);
        }
        cudaMemcpy(mode == 2 ? got16.data() : mode ? got.data() : ref.data(), out, got.size() * 4, cudaMemcpyDeviceToHost);
    }
    {
        double num = 0, den = 0;
        for (size_t i = 0; i < ref.size(); ++i) { const double d = (double)got16[i] - ref[i]; num += d * d; den += (double)ref[i] * ref[i]; }
        printf("pair16 vs single: rel-L2 %.3e\n", sqrt(num / den));
    }
    double num = 0, den = 0; size_t bad = 0;
    for (size_t i = 0; i < ref.size(); ++i) {
        const double d = (double)got[i] - ref[i];
        num += d * d; den += (double)ref[i] * ref[i];
        if (!(fabs(d) <= 1e-5 + 1e-5 * fabs(ref[i]))) ++bad;
    }
    printf("pair vs single: rel-L2 %.3e, %zu elements outside 1e-5\n", sqrt(num / den), bad);
    return 0;
}
