// trace_bwd5.cu -- k_tc5_bwd (decoupled N=256 backward) vs k_tc2_bwd on random data (dev tool).
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
    float *A, *Z, *W, *img128, *img256, *out;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&Z, (size_t)S * R * N * 4); cudaMalloc(&out, (size_t)S * R * N * 4);
    cudaMalloc(&W, K * N * 4); cudaMalloc(&img128, 2 * K * N * 4); cudaMalloc(&img256, 2 * K * N * 4);
    fill<<<1024, 256>>>(A, (size_t)S * R * K, 11u, 1.0f);
    fill<<<1024, 256>>>(Z, (size_t)S * R * N, 13u, 1.8f);
    fill<<<64, 256>>>(W, K * N, 17u, 0.15f);
    k_tc_prep_image<<<256, 256>>>(W, K, N, 1, 128, img128);
    k_tc_prep_image<<<256, 256>>>(W, K, N, 1, 256, img256);
    // 3xFP16: bounds (|A| <= 0.5, |W| <= 0.075) and the fp16 transposed image
    unsigned* amax; uint16_t* img16;
    cudaMalloc(&amax, 8 * 4); cudaMalloc(&img16, 2 * K * N * 2);
    const float am[8] = {0.5f, 0.5f, 0.5f, 0.5f, 0.075f, 0, 0, 0};
    cudaMemcpy(amax, am, sizeof(am), cudaMemcpyHostToDevice);
    k_tc_prep_image16<<<256, 256>>>(W, K, N, 1, 256, amax + 4, img16);
    TcGemmArgs g{}; g.A = A; g.Zlow = Z; g.out = out; g.Rpad = R; g.K = K; g.N = N;
    g.amax_in = amax; g.amax_w = amax + 4;
    std::vector<float> ref((size_t)S * R * N), got((size_t)S * R * N);
    std::vector<float> got1((size_t)S * R * N), got16((size_t)S * R * N);
    for (int mode = 0; mode < 4; ++mode) {
        g.img = mode == 3 ? reinterpret_cast<float*>(img16) : mode ? img256 : img128;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(out, 0, (size_t)S * R * N * 4);
            unsigned long long z[8] = {0};
            cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int rc = mode == 3 ? launch_tc5_bwd_t<LAY_MX, false, true>(g, 0)
                         : mode == 2 ? launch_tc5_bwd_t<LAY_MX, true, false>(g, 0)
                         : mode == 1 ? launch_tc5_bwd_t<LAY_MX, false, false>(g, 0) : launch_tc2_bwd_t<LAY_MX, 128, false>(g, 0);
            cudaError_t le = cudaGetLastError();
            if (rc || le != cudaSuccess) printf("launch rc=%d %s\n", rc, cudaGetErrorString(le));
            cudaEventRecord(e1);
            cudaError_t e = cudaDeviceSynchronize();
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long t[8];
            cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
            const double ctas = mode ? R / 128.0 : (R / 128.0) * 2;
            printf("%s %s %.3f ms per-CTA: mma_wait_full %.0f prod0_wait_empty %.0f epi_busy %.0f (kernel/CTA %.0f)\n",
                   mode == 3 ? "tc5f16" : mode == 2 ? "tc5pair" : mode ? "tc5" : "tc2",
                   cudaGetErrorString(e), ms, t[0] / ctas, t[2] / ctas, t[3] / ctas, ms * 1e-3 * 1.965e9 * 148 / ctas);
        }
        cudaMemcpy(mode == 3 ? got16.data() : mode == 2 ? got1.data() : mode ? got.data() : ref.data(), out, got.size() * 4,
                   cudaMemcpyDeviceToHost);
    }
    double num = 0, den = 0, mx = 0;
    for (size_t i = 0; i < ref.size(); ++i) {
        const double d = (double)got[i] - ref[i];
        num += d * d; den += (double)ref[i] * ref[i]; mx = fmax(mx, fabs(d));
    }
    printf("tc5 vs tc2: rel-L2 %.3e max-abs %.3e\n", sqrt(num / den), mx);
    num = 0; mx = 0;
    for (size_t i = 0; i < ref.size(); ++i) { const double d = (double)got1[i] - ref[i]; num += d * d; mx = fmax(mx, fabs(d)); }
    printf("tc5pair vs tc2: rel-L2 %.3e max-abs %.3e\n", sqrt(num / den), mx);
    num = 0; mx = 0;
    for (size_t i = 0; i < ref.size(); ++i) { const double d = (double)got16[i] - ref[i]; num += d * d; mx = fmax(mx, fabs(d)); }
    printf("tc5f16 vs tc2: rel-L2 %.3e max-abs %.3e\n", sqrt(num / den), mx);
    return 0;
}
