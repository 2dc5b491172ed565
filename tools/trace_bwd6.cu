// trace_bwd6.cu -- the k_tc6_bwd experiment (tools/tc6_bwd_experiment.cuh: one stream per pass, TMEM double-buffered, staging-free
// epilogue) vs k_tc5_bwd<F16> on random data (dev tool): bit-identity of the
// outputs and the recorded |Zb_in| bounds, and the time per launch.
//   trace_bwd6 [rows] [layout: 3 = LAY_MX (S = 4), 1 = LAY_XT (S = 3)]
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"
#include "../paper_2604_15645_b200/csrc/launch_tc.cu"
#include "tc6_bwd_experiment.cuh"
using namespace pnx;
__global__ void fill(float* p, size_t n, unsigned seed, float scale) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)i * 2654435761u ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = ((h & 0xFFFFFF) / 16777216.0f - 0.5f) * scale;
    }
}
template <int L>
int run(int R) {
    constexpr int S = Streams<L>::S;
    const int K = 256, N = 256;
    float *A, *Z, *W, *out5, *out6;
    cudaMalloc(&A, (size_t)S * R * K * 4);
    cudaMalloc(&Z, (size_t)S * R * N * 4);
    cudaMalloc(&out5, (size_t)S * R * N * 4);
    cudaMalloc(&out6, (size_t)S * R * N * 4);
    cudaMalloc(&W, K * N * 4);
    fill<<<1024, 256>>>(A, (size_t)S * R * K, 11u, 1.0f);
    fill<<<1024, 256>>>(Z, (size_t)S * R * N, 13u, 1.8f);
    fill<<<64, 256>>>(W, K * N, 17u, 0.15f);
    unsigned *amax, *am5, *am6;
    uint16_t *img, *imgp;
    cudaMalloc(&amax, 8 * 4);
    cudaMalloc(&am5, 8 * 4);
    cudaMalloc(&am6, 8 * 4);
    cudaMalloc(&img, 2 * K * N * 2);
    cudaMalloc(&imgp, 2 * K * N * 2);
    const float am[8] = {0.5f, 0.5f, 0.5f, 0.5f, 0.075f, 0, 0, 0};
    cudaMemcpy(amax, am, sizeof(am), cudaMemcpyHostToDevice);
    k_tc_prep_image16<<<256, 256>>>(W, K, N, 1, 256, amax + 4, img);
    k_tc6_prep_image16<<<256, 256>>>(W, K, N, amax + 4, imgp);
    TcGemmArgs g{};
    g.A = A; g.Zlow = Z; g.Rpad = R; g.K = K; g.N = N; g.amax_in = amax; g.amax_w = amax + 4; g.f16 = 1;
    double t5 = 0, t6 = 0;
    for (int rep = 0; rep < 4; ++rep) {
        for (int v = 0; v < 2; ++v) {
            TcGemmArgs a = g;
            a.out = v ? out6 : out5;
            a.img = reinterpret_cast<const float*>(v ? imgp : img);
            a.amax_out = v ? am6 : am5;
            cudaMemset(a.out, 0, (size_t)S * R * N * 4);
            cudaMemset(a.amax_out, 0, 32);
#ifdef PNX_TC_TRACE
            unsigned long long z[8] = {0};
            cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
#endif
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int rc = v ? (getenv("TC6_PAIR") ? launch_tc6_bwd_t<L, true>(a, 0) : launch_tc6_bwd_t<L, false>(a, 0))
                             : launch_tc5_bwd_t<L, false, true>(a, 0);
            cudaEventRecord(e1);
            cudaError_t e = cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rc || e != cudaSuccess) {
                printf("%s launch rc=%d %s\n", v ? "tc6" : "tc5", rc, cudaGetErrorString(e));
                return 1;
            }
            if (rep > 0) (v ? t6 : t5) += ms / 3;
#ifdef PNX_TC_TRACE
            if (v && rep == 3) {
                unsigned long long t[8];
                cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
                const double nt = R / 128.0;
                printf("  tc6 per tile: mma_wait_full %.0f mma_wait_drain %.0f prod0_wait_empty %.0f epi_busy %.0f "
                       "epi_wait_full %.0f (kernel %.0f cycles/tile at 1.965 GHz)\n",
                       t[0] / nt, t[1] / nt, t[2] / nt, t[3] / nt, t[4] / nt, ms * 1e-3 * 1.965e9 * 148 / nt);
            }
#endif
        }
    }
    std::vector<float> h5((size_t)S * R * N), h6((size_t)S * R * N);
    cudaMemcpy(h5.data(), out5, h5.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h6.data(), out6, h6.size() * 4, cudaMemcpyDeviceToHost);
    unsigned a5[8], a6[8];
    cudaMemcpy(a5, am5, 32, cudaMemcpyDeviceToHost);
    cudaMemcpy(a6, am6, 32, cudaMemcpyDeviceToHost);
    size_t ndiff = 0, first = (size_t)-1;
    double mx = 0, ref = 0;
    for (size_t i = 0; i < h5.size(); ++i) {
        if (memcmp(&h5[i], &h6[i], 4) != 0) {
            ++ndiff;
            if (first == (size_t)-1) first = i;
            mx = fmax(mx, fabs((double)h5[i] - h6[i]));
        }
        ref = fmax(ref, fabs((double)h5[i]));
    }
    printf("L=%d S=%d R=%d: tc5f16 %.3f ms  tc6 %.3f ms  (%.1f%%)  differing words %zu (first %zd, max-abs %.3e of %.3e)"
           "  amax %s\n",
           L, S, R, t5, t6, 100.0 * (t6 / t5 - 1.0), ndiff, first == (size_t)-1 ? (ssize_t)-1 : (ssize_t)first, mx, ref,
           memcmp(a5, a6, 4 * S) == 0 ? "equal" : "DIFFER");
    if (ndiff) {
        const size_t i = first;
        const size_t s = i / ((size_t)R * N), r = (i / N) % R, f = i % N;
        printf("  first diff at stream %zu row %zu feature %zu: tc5 %.9g tc6 %.9g\n", s, r, f, h5[i], h6[i]);
    }
    cudaFree(A); cudaFree(Z); cudaFree(out5); cudaFree(out6); cudaFree(W);
    return ndiff ? 2 : 0;
}
int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 262144;
    const int lay = argc > 2 ? atoi(argv[2]) : 3;
    return lay == 1 ? run<LAY_XT>(R) : run<LAY_MX>(R);
}
