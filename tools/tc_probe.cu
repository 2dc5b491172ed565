// tc_probe.cu -- standalone check of the tcgen05 kind::tf32 conventions used by
// paper_2604_15645_b200/csrc (descriptor bit layouts, 128 B swizzle, K-major and
// MN-major operands, TMEM lane/column mapping, 3xTF32 accuracy, MMA rate).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tc_probe.cu -o tc_probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2604_15645_b200/csrc/tc_common.cuh"

using namespace pnx::tc;

constexpr int M = 128;

// A: [M][K] (a_mn=0) or [K][M] (a_mn=1); B: [N][K] (b_mn=0) or [K][N] (b_mn=1).
__device__ int g_swap;
template <int N, int K>
__global__ void probe(const float* A, const float* B, float* D, int a_mn, int b_mn, int passes, int reps,
                      long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int a_bytes = M * K * 4, b_bytes = N * K * 4;
    uint8_t* sAh = smem;
    uint8_t* sAl = sAh + a_bytes;
    uint8_t* sBh = sAl + a_bytes;
    uint8_t* sBl = sBh + b_bytes;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;

    // layout helpers (byte offsets)
    auto kmaj = [](int row, int k, int rows) -> uint32_t {  // [K/32 atoms][rows][128B]
        return (uint32_t)((k / 32) * rows * 128) + sw128_off(row, (k % 32) / 4) + (k % 4) * 4;
    };
    auto mnmaj = [](int k, int mn, int mnext) -> uint32_t {  // SW128_32B atoms: [K/4][mn/32][4 rows][128B]
        return (uint32_t)((k / 4) * (mnext / 32) * 512 + (mn / 32) * 512) + (k % 4) * 128 +
               ((((mn % 32) / 8) ^ (k % 4)) * 32) + (mn % 8) * 4;
    };
    for (int i = tid; i < M * K; i += blockDim.x) {
        int m, k;
        if (a_mn) { k = i / M; m = i % M; } else { m = i / K; k = i % K; }
        float hi, lo;
        split3(A[i], hi, lo);
        uint32_t off = a_mn ? mnmaj(k, m, M) : kmaj(m, k, M);
        *(float*)(sAh + off) = hi;
        *(float*)(sAl + off) = lo;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int n, k;
        if (b_mn) { k = i / N; n = i % N; } else { n = i / K; k = i % K; }
        float hi, lo;
        split3(B[i], hi, lo);
        uint32_t off = b_mn ? mnmaj(k, n, N) : kmaj(n, k, N);
        *(float*)(sBh + off) = hi;
        *(float*)(sBl + off) = lo;
    }
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<256>(&tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = make_idesc_tf32(M, N, a_mn, b_mn);
    long long t0 = clock64();
    if (tid == 0) {
        for (int rep = 0; rep < reps; ++rep) {
            for (int ks = 0; ks < K / 8; ++ks) {
                uint64_t ad[2], bd[2];
                for (int h = 0; h < 2; ++h) {
                    uint32_t abase = smem_u32(h ? sAl : sAh), bbase = smem_u32(h ? sBl : sBh);
                    if (a_mn) ad[h] = g_swap ? make_sdesc(abase + ks * 2 * (M / 32) * 512, (M / 32) * 512, 512, 1) : make_sdesc(abase + ks * 2 * (M / 32) * 512, 512, (M / 32) * 512, 1);
                    else ad[h] = make_sdesc_sw128(abase + (ks / 4) * M * 128 + (ks % 4) * 32, 16, 1024);
                    if (b_mn) bd[h] = g_swap ? make_sdesc(bbase + ks * 2 * (N / 32) * 512, (N / 32) * 512, 512, 1) : make_sdesc(bbase + ks * 2 * (N / 32) * 512, 512, (N / 32) * 512, 1);
                    else bd[h] = make_sdesc_sw128(bbase + (ks / 4) * N * 128 + (ks % 4) * 32, 16, 1024);
                }
                uint32_t acc = (rep > 0 || ks > 0) ? 1u : 0u;
                mma_tf32(tmem, ad[0], bd[0], idesc, acc);          // hi*hi
                if (passes >= 2) mma_tf32(tmem, ad[0], bd[1], idesc, 1u);  // hi*lo
                if (passes >= 3) mma_tf32(tmem, ad[1], bd[0], idesc, 1u);  // lo*hi
            }
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    tc_fence_after();
    if (tid == 0) *cycles = t1 - t0;
    // epilogue: warp w reads lanes 32*(w%4).. and columns [16*(w/4) ...] stride 16*(nwarps/4)
    const int q = warp % 4, cgrp = warp / 4, ncg = blockDim.x / 128;
    for (int c0 = cgrp * 16; c0 < N; c0 += 16 * ncg) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
        const int row = q * 32 + (tid % 32);
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tmem);
}


// K-major probe for SW32 (KB=8) / SW64 (KB=16) / SW128 (KB=32) tiles: [K/KB][rows][KB*4 B]
template <int N, int K, int KB>
__global__ void probe_k(const float* A, const float* B, float* D, int passes) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int a_bytes = M * K * 4, b_bytes = N * K * 4;
    uint8_t* sAh = smem; uint8_t* sAl = sAh + a_bytes; uint8_t* sBh = sAl + a_bytes; uint8_t* sBl = sBh + b_bytes;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;
    auto off = [](int row, int k, int rows) -> uint32_t {
        uint32_t blk = (uint32_t)(k / KB) * rows * KB * 4;
        int kk = k % KB;
        if (KB == 8) return blk + sw32_off(row, kk);
        if (KB == 16) return blk + sw64_off(row, kk);
        return blk + sw128_off(row, kk / 4) + (kk % 4) * 4;
    };
    for (int i = tid; i < M * K; i += blockDim.x) {
        int m = i / K, k = i % K; float hi, lo; split3(A[i], hi, lo);
        *(float*)(sAh + off(m, k, M)) = hi; *(float*)(sAl + off(m, k, M)) = lo;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int n = i / K, k = i % K; float hi, lo; split3(B[i], hi, lo);
        *(float*)(sBh + off(n, k, N)) = hi; *(float*)(sBl + off(n, k, N)) = lo;
    }
    fence_proxy_async_smem();
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<256>(&tmem_base);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = make_idesc_tf32(M, N, 0, 0);
    const uint32_t lay = KB == 8 ? 6u : (KB == 16 ? 4u : 2u);
    const uint32_t sbo = 8 * KB * 4;
    if (tid == 0) {
        for (int ks = 0; ks < K / 8; ++ks) {
            uint64_t ad[2], bd[2];
            for (int h = 0; h < 2; ++h) {
                uint32_t abase = smem_u32(h ? sAl : sAh), bbase = smem_u32(h ? sBl : sBh);
                uint32_t kin = (ks * 8) % KB, blk = (ks * 8) / KB;
                ad[h] = make_sdesc(abase + blk * M * KB * 4 + kin * 4, 16, sbo, lay);
                bd[h] = make_sdesc(bbase + blk * N * KB * 4 + kin * 4, 16, sbo, lay);
            }
            mma_tf32(tmem, ad[0], bd[0], idesc, ks > 0 ? 1u : 0u);
            if (passes >= 2) mma_tf32(tmem, ad[0], bd[1], idesc, 1u);
            if (passes >= 3) mma_tf32(tmem, ad[1], bd[0], idesc, 1u);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int q = warp % 4, cgrp = warp / 4, ncg = blockDim.x / 128;
    for (int c0 = cgrp * 16; c0 < N; c0 += 16 * ncg) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
        const int row = q * 32 + (tid % 32);
        for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tmem);
}

template <int N, int K, int KB>
int run_k(int passes, bool exact) {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(99);
    for (auto& x : A) x = exact ? (float)(rand() % 7 - 3) : (float)rand() / RAND_MAX * 2 - 1;
    for (auto& x : B) x = exact ? (float)(rand() % 5 - 2) : (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    size_t smem = 2 * (M * K * 4) + 2 * (N * K * 4) + 1024;
    cudaFuncSetAttribute(probe_k<N, K, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_k<N, K, KB><<<1, 256, smem>>>(dA, dB, dD, passes);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n])); maxref = fmax(maxref, fabs(ref));
    }
    printf("K-major KB=%d N=%d K=%d passes=%d exact=%d: max|err|=%.3e rel %.3e\n", KB, N, K, passes, (int)exact, maxerr, maxerr / maxref);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return 0;
}

template <int N, int K>
int run(int a_mn, int b_mn, int passes, int reps, bool exact) {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(1234);
    for (auto& x : A) x = exact ? (float)(rand() % 7 - 3) : (float)rand() / RAND_MAX * 2 - 1;
    for (auto& x : B) x = exact ? (float)(rand() % 5 - 2) : (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    size_t smem = 2 * (M * K * 4) + 2 * (N * K * 4) + 1024;
    cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<N, K><<<1, 256, smem>>>(dA, dB, dD, a_mn, b_mn, passes, reps, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    long long cyc;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) {
                double a = a_mn ? A[k * M + m] : A[m * K + k];
                double b = b_mn ? B[k * N + n] : B[n * K + k];
                ref += a * b;
            }
            ref *= reps;
            maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
            maxref = fmax(maxref, fabs(ref));
        }
    if (getenv("PROBE_DUMP") && exact && (a_mn || b_mn)) {
        for (int m = 0; m < 2; ++m)
            for (int n = 0; n < 6; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (a_mn ? A[k * M + m] : A[m * K + k]) * (b_mn ? B[k * N + n] : B[n * K + k]);
                printf("  D[%d][%d]=%g ref=%g\n", m, n, D[m * N + n], ref);
            }
        // find which (m', n') of the reference each D entry matches
        int found = 0;
        for (int m = 0; m < 2 && found < 6; ++m) for (int n = 0; n < 4; ++n) {
            for (int mm = 0; mm < M; ++mm) for (int nn = 0; nn < N; ++nn) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (a_mn ? A[k * M + mm] : A[mm * K + k]) * (b_mn ? B[k * N + nn] : B[nn * K + k]);
                if (ref == D[m * N + n] && D[m*N+n] != 0) { printf("  D[%d][%d] == ref[%d][%d]\n", m, n, mm, nn); found++; goto nxt; }
            }
            nxt:;
        }
    }
    double mmas = (double)reps * (K / 8) * passes;
    printf("N=%d K=%d a_mn=%d b_mn=%d passes=%d reps=%d exact=%d: max|err|=%.3e (rel %.3e)  %.1f cyc/MMA\n", N, K,
           a_mn, b_mn, passes, reps, (int)exact, maxerr, maxerr / maxref, cyc / mmas);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dc);
    return 0;
}

int main(int argc, char** argv) {
    int sw = argc > 1 ? atoi(argv[1]) : 0;
    cudaMemcpyToSymbol(g_swap, &sw, 4);
    printf("swap=%d\n", sw);
    int bad = 0;
    bad |= run_k<128, 64, 8>(1, true);
    bad |= run_k<256, 32, 8>(1, true);
    bad |= run_k<128, 64, 16>(1, true);
    bad |= run_k<256, 64, 16>(1, true);
    bad |= run_k<128, 64, 32>(1, true);
    bad |= run_k<128, 64, 8>(3, false);
    bad |= run_k<128, 64, 16>(3, false);
    if (argc > 2) return bad;
    for (int am = 0; am < 2; ++am)
        for (int bm = 0; bm < 2; ++bm) bad |= run<128, 64>(am, bm, 1, 1, true);
    bad |= run<256, 32>(0, 0, 1, 1, true);
    bad |= run<256, 32>(1, 1, 1, 1, true);
    for (int p = 1; p <= 3; ++p) bad |= run<128, 64>(0, 0, p, 1, false);
    for (int p = 1; p <= 3; ++p) bad |= run<128, 64>(1, 1, p, 1, false);
    // throughput
    bad |= run<128, 64>(0, 0, 3, 2000, false);
    bad |= run<256, 32>(0, 0, 3, 2000, false);
    bad |= run<256, 32>(1, 1, 3, 2000, false);
    bad |= run<64, 64>(0, 0, 3, 2000, false);
    return bad;
}
