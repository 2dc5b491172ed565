// rate_probe.cu -- tcgen05 kind::tf32 MMA rate vs issue pattern (dev tool)
#include <cstdio>
#include <cstdlib>
#include "../paper_2604_15645_b200/csrc/tc_common.cuh"
using namespace pnx::tc;
// mode 0: 1 MMA per k-step per acc (A_k, B_k)
// mode 1: 3 MMAs per k-step per acc: (Ah,Bh) (Ah,Bl) (Al,Bh)
// mode 2: like 1 but accumulators interleaved innermost
__global__ void rate(int N, int nacc, int iters, int mode, int rnd, int f16, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned s = 12345u + threadIdx.x;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
        s = s * 1664525u + 1013904223u;
        const float v = rnd ? ((s >> 9) * (1.0f / 8388608.0f) - 0.5f) : 0.5f;
        if (f16) ((uint32_t*)smem)[i] = pack_half2(v, -v); else ((float*)smem)[i] = v;
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t id = f16 ? make_idesc_f16(128, N, 0, 0) : make_idesc_tf32(128, N, 0, 0);
#define mma_tf32(d, a, b, i, acc) (f16 ? mma_f16(d, a, b, i, acc) : mma_tf32(d, a, b, i, acc))
    const uint32_t sb = smem_u32(smem);
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const uint32_t k = it & 3;
            const uint64_t ah = make_sdesc(sb + k * 4096, 16, 256, 6), al = make_sdesc(sb + 16384 + k * 4096, 16, 256, 6);
            const uint64_t bh = make_sdesc(sb + 32768 + k * 8192, 16, 256, 6), bl = make_sdesc(sb + 65536 + k * 8192, 16, 256, 6);
            if (mode == 0) {
                for (int a = 0; a < nacc; ++a) mma_tf32(tbase + a * N, ah, bh, id, it > 0);
            } else if (mode == 1) {
                for (int a = 0; a < nacc; ++a) {
                    mma_tf32(tbase + a * N, ah, bh, id, it > 0);
                    mma_tf32(tbase + a * N, ah, bl, id, 1);
                    mma_tf32(tbase + a * N, al, bh, id, 1);
                }
            } else if (mode == 2) {
                for (int a = 0; a < nacc; ++a) mma_tf32(tbase + a * N, ah, bh, id, it > 0);
                for (int a = 0; a < nacc; ++a) mma_tf32(tbase + a * N, ah, bl, id, 1);
                for (int a = 0; a < nacc; ++a) mma_tf32(tbase + a * N, al, bh, id, 1);
            } else {  // mode 3: nacc big/small PAIRS: hh -> big, hl, lh -> small
                for (int a = 0; a < nacc; ++a) {
                    mma_tf32(tbase + (2 * a) * N, ah, bh, id, it > 0);
                    mma_tf32(tbase + (2 * a + 1) * N, ah, bl, id, it > 0);
                    mma_tf32(tbase + (2 * a + 1) * N, al, bh, id, 1);
                }
            }
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) *out = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tbase);
}
int main() {
    long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int cfg[][4] = {{256, 1, 3, 1}, {128, 1, 3, 1}, {128, 2, 3, 1}, {64, 4, 3, 1}, {128, 1, 0, 0}, {128, 1, 0, 1}, {128, 1, 1, 0}, {128, 1, 1, 1}, {128, 4, 1, 1}, {128, 4, 2, 1},
                    {64, 8, 1, 1}, {64, 8, 2, 1}, {256, 2, 1, 1}, {256, 2, 2, 1}, {128, 4, 0, 1}, {64, 8, 0, 1}};
    for (int f16 = 0; f16 < 2; ++f16)
    for (auto& c : cfg) {
        rate<<<1, 128, 100 * 1024>>>(c[0], c[1], 2000, c[2], c[3], f16, d);
        cudaDeviceSynchronize();
        long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        double nm = 2000.0 * c[1] * (c[2] == 0 ? 1 : 3);
        double per = (double)cyc / nm;
        printf("%s N=%3d nacc=%d mode=%d rnd=%d: %6.1f cyc/MMA -> %4.0f flop/cyc (%.0f%% of 4096 tf32)\n", f16 ? "f16 K=16" : "tf32 K=8", c[0], c[1], c[2], c[3], per,
               2.0 * 128 * c[0] * (f16 ? 16 : 8) / per, 100.0 * 2.0 * 128 * c[0] * (f16 ? 16 : 8) / per / 4096);
    }
    return 0;
}
