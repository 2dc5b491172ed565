// trace_wgrad.cu -- role timing + pair/single cross-check for k_tc2_wgrad<LAY_MX, TANH, 256, PAIR> (dev tool).
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
    const int WR = argc > 2 ? atoi(argv[2]) : TC_WROWS;
    float *A, *B, *wp; double* dbp;
    cudaMalloc(&A, (size_t)S * R * K * 4); cudaMalloc(&B, (size_t)S * R * N * 4);
    const int tiles = (R + WR - 1) / WR;
    cudaMalloc(&wp, (size_t)tiles * K * N * 4); cudaMalloc(&dbp, (size_t)tiles * N * 8);
    fill<<<1024, 256>>>(A, (size_t)S * R * K, 1u, 1.6f);
    fill<<<1024, 256>>>(B, (size_t)S * R * N, 7u, 1.0f);
    TcWgradArgs w{}; w.A = A; w.Bm = B; w.wpart = wp; w.dbpart = dbp; w.Rpad = R; w.nrows = R; w.Kin = K; w.N = N;
    std::vector<float> ref, out, out16;
    std::vector<double> dref, dout, dout16;
    unsigned* amax;
    cudaMalloc(&amax, 2 * S * 4);
    const float am[2 * S] = {0.8f, 0.8f, 0.8f, 0.8f, 0.5f, 0.5f, 0.5f, 0.5f};  // |A| <= 0.8 (fill 1.6), |B| <= 0.5
    cudaMemcpy(amax, am, sizeof(am), cudaMemcpyHostToDevice);
    w.amaxA = amax;
    w.amaxB = amax + S;
    w.f16 = 1;
    for (int mode = 0; mode < 3; ++mode) {
        const bool pair = mode >= 1;
        for (int rep = 0; rep < 2; ++rep) {
            unsigned long long z[8] = {0};
            cudaMemcpyToSymbol(g_tc_trace, z, sizeof(z));
            cudaMemset(wp, 0, (size_t)tiles * K * N * 4);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            int rc = mode == 2 ? launch_tc2_wgrad_t<LAY_MX, ACT_TANH, 256, true, true>(w, tiles, WR, 0)
                     : pair    ? launch_tc2_wgrad_t<LAY_MX, ACT_TANH, 256, true>(w, tiles, WR, 0)
                               : launch_tc2_wgrad_t<LAY_MX, ACT_TANH, 256, false>(w, tiles, WR, 0);
            cudaError_t le = cudaGetLastError();
            if (rc || le != cudaSuccess) printf("launch error rc=%d %s\n", rc, cudaGetErrorString(le));
            cudaEventRecord(e1);
            cudaError_t e = cudaDeviceSynchronize();
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long t[8];
            cudaMemcpyFromSymbol(t, g_tc_trace, sizeof(t));
            const double ctas = tiles * 2.0;
            printf("%s %s %.3f ms per-CTA cycles: mma_wait_full %.0f conv0_wait_empty %.0f conv0_wait_raw %.0f compute %.0f store %.0f (kernel/CTA %.0f)\n",
                   mode == 2 ? "pair16" : pair ? "pair  " : "single", cudaGetErrorString(e), ms, t[0] / ctas, t[2] / ctas, t[1] / ctas, t[5] / ctas, t[6] / ctas,
                   ms * 1e-3 * 1.965e9 * 148 / ctas);
        }
        std::vector<float>& o = mode == 2 ? out16 : pair ? out : ref;
        std::vector<double>& d = mode == 2 ? dout16 : pair ? dout : dref;
        o.resize((size_t)tiles * K * N); d.resize((size_t)tiles * N);
        cudaMemcpy(o.data(), wp, o.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(d.data(), dbp, d.size() * 8, cudaMemcpyDeviceToHost);
    }
    double num = 0, den = 0, dmax = 0;
    for (size_t i = 0; i < ref.size(); ++i) { num += (double)(out[i] - ref[i]) * (out[i] - ref[i]); den += (double)ref[i] * ref[i]; }
    for (size_t i = 0; i < dref.size(); ++i) dmax = fmax(dmax, fabs(dout[i] - dref[i]));
    printf("pair vs single: wpart rel-L2 %.3e  db max-abs diff %.3e\n", sqrt(num / den), dmax);
    num = 0; double mx = 0;
    for (size_t i = 0; i < ref.size(); ++i) { const double dd = (double)(out16[i] - ref[i]); num += dd * dd; mx = fmax(mx, fabs(dd)); }
    printf("pair16 vs single: wpart rel-L2 %.3e max-abs %.3e\n", sqrt(num / den), mx);
    return 0;
}
