// acc_probe.cu -- accuracy of tcgen05 kind::tf32 accumulation schedules (dev tool).
// D[128x128] = A[128xK] B^T with A,B ~ U(-1,1); reports rel-L2 error vs FP64 for
// several 3xTF32 schedules, and FP32 sequential FMA for comparison.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2604_15645_b200/csrc/tc_common.cuh"
using namespace pnx::tc;
constexpr int M = 128, N = 128;

// schedule: 0 = per k-step (hh, hl, lh); 1 = per k-step (lh, hl, hh); 2 = per k-step +ll;
// 3 = all small terms over K first, then hh over K; 4 = hh only;
// 5 = two accumulators: hh in D0, (hl+lh) in D1, summed in the epilogue
// 6 = hh chain split in 4 accumulators over K quarters (+ small into D4), summed in epilogue
template <int K>
__global__ void acc_kernel(const float* A, const float* B, float* D, int sched) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int ab = M * K * 4;
    uint8_t *sAh = smem, *sAl = smem + ab, *sBh = smem + 2 * ab, *sBl = smem + 3 * ab;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < M * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        uint32_t off = (k / 8) * M * 32 + sw32_off(r, k % 8);
        float h, l;
        split3(A[i], h, l); *(float*)(sAh + off) = h; *(float*)(sAl + off) = l;
        split3(B[i], h, l); *(float*)(sBh + off) = h; *(float*)(sBl + off) = l;
    }
    fence_proxy_async_smem();
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t id = make_idesc_tf32(M, N, 0, 0);
    if (tid == 0) {
        auto d = [&](uint8_t* p, int ks) { return make_sdesc(smem_u32(p) + ks * M * 32, 16, 256, 6); };
        const int nk = K / 8;
        if (sched <= 2) {
            for (int ks = 0; ks < nk; ++ks) {
                uint32_t a0 = ks > 0;
                if (sched == 0) { mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, a0); mma_tf32(tm, d(sAh, ks), d(sBl, ks), id, 1); mma_tf32(tm, d(sAl, ks), d(sBh, ks), id, 1); }
                if (sched == 1) { mma_tf32(tm, d(sAl, ks), d(sBh, ks), id, a0); mma_tf32(tm, d(sAh, ks), d(sBl, ks), id, 1); mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, 1); }
                if (sched == 2) { mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, a0); mma_tf32(tm, d(sAh, ks), d(sBl, ks), id, 1); mma_tf32(tm, d(sAl, ks), d(sBh, ks), id, 1); mma_tf32(tm, d(sAl, ks), d(sBl, ks), id, 1); }
            }
        } else if (sched == 3) {
            for (int ks = 0; ks < nk; ++ks) { mma_tf32(tm, d(sAh, ks), d(sBl, ks), id, ks > 0); mma_tf32(tm, d(sAl, ks), d(sBh, ks), id, 1); }
            for (int ks = 0; ks < nk; ++ks) mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, 1);
        } else if (sched == 4) {
            for (int ks = 0; ks < nk; ++ks) mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, ks > 0);
        } else if (sched == 5) {
            for (int ks = 0; ks < nk; ++ks) {
                mma_tf32(tm, d(sAh, ks), d(sBh, ks), id, ks > 0);
                mma_tf32(tm + N, d(sAh, ks), d(sBl, ks), id, ks > 0); mma_tf32(tm + N, d(sAl, ks), d(sBh, ks), id, 1);
            }
        } else {
            for (int ks = 0; ks < nk; ++ks) {
                int q = ks * 3 / nk;  // 3 hh accumulators
                mma_tf32(tm + q * N, d(sAh, ks), d(sBh, ks), id, ks * 3 % nk >= 3 ? 1u : (ks == q * nk / 3 ? 0u : 1u));
                mma_tf32(tm + 3 * N, d(sAh, ks), d(sBl, ks), id, ks > 0); mma_tf32(tm + 3 * N, d(sAl, ks), d(sBh, ks), id, 1);
            }
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int q = warp % 4, ncg = blockDim.x / 128, cg = warp / 4;
    const int nacc = sched == 5 ? 2 : (sched == 6 ? 4 : 1);
    for (int c0 = cg * 16; c0 < N; c0 += 16 * ncg) {
        float acc[16] = {0};
        for (int a = nacc - 1; a >= 0; --a) {
            float v[16];
            tmem_ld16(tm + ((uint32_t)(q * 32) << 16) + a * N + c0, v);
            tmem_ld_wait();
            for (int j = 0; j < 16; ++j) acc[j] += v[j];
        }
        const int row = q * 32 + tid % 32;
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = acc[j];
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int K>
void run() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(7);
    for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
    for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
    std::vector<double> ref(M * N);
    double e32 = 0, nr = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double r = 0; float f = 0;
        for (int k = 0; k < K; ++k) { r += (double)A[m * K + k] * B[n * K + k]; f = fmaf(A[m * K + k], B[n * K + k], f); }
        ref[m * N + n] = r; e32 += (f - r) * (f - r); nr += r * r;
    }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int smem = 4 * M * K * 4 + 1024;
    cudaFuncSetAttribute(acc_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    printf("K=%d  fp32 sequential FMA: rel-L2 %.3e\n", K, sqrt(e32 / nr));
    const char* names[] = {"hh,hl,lh", "lh,hl,hh", "+ll", "small-first", "hh only", "2 acc (hh | small)", "3 hh acc + small acc"};
    for (int s = 0; s < 7; ++s) {
        acc_kernel<K><<<1, 256, smem>>>(dA, dB, dD, s);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double e = 0;
        for (int i = 0; i < M * N; ++i) e += (D[i] - ref[i]) * (D[i] - ref[i]);
        printf("  sched %d %-22s rel-L2 %.3e\n", s, names[s], sqrt(e / nr));
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
}
int main() { run<64>(); run<256>(); run<96>(); return 0; }
