// tmem_layout_probe.cu -- which (lane, column) of TMEM each thread receives from
// tcgen05.ld.16x256b (dev tool). Warp 0 stores value = 1000 * lane + column with
// the known 32x32b shape (thread t <-> lane t), then reads it back with
// 16x256b.x1 / .x2 at lane offsets 0 and 16 and prints the mapping.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(int* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tbase;
    if (warp == 0) {
        uint32_t v[16];
        for (int c = 0; c < 16; ++c) v[c] = 1000u * lane + c;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        uint32_t a[4], b[4], c2[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                     : "r"(t));
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "r"(t + (16u << 16)));
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(c2[0]), "=r"(c2[1]), "=r"(c2[2]), "=r"(c2[3]), "=r"(c2[4]), "=r"(c2[5]), "=r"(c2[6]),
                       "=r"(c2[7])
                     : "r"(t));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int i = 0; i < 4; ++i) out[lane * 16 + i] = (int)a[i];
        for (int i = 0; i < 4; ++i) out[lane * 16 + 4 + i] = (int)b[i];
        for (int i = 0; i < 8; ++i) out[lane * 16 + 8 + i] = (int)c2[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
    int* d;
    cudaMalloc(&d, 32 * 16 * 4);
    probe<<<1, 128>>>(d);
    int h[32 * 16];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("status %s  (entries: lane*1000 + column)\n", cudaGetErrorString(e));
    for (int l = 0; l < 32; ++l) {
        printf("thread %2d | x1@0:", l);
        for (int i = 0; i < 4; ++i) printf(" %5d", h[l * 16 + i]);
        printf(" | x1@16:");
        for (int i = 0; i < 4; ++i) printf(" %5d", h[l * 16 + 4 + i]);
        printf(" | x2@0:");
        for (int i = 0; i < 8; ++i) printf(" %5d", h[l * 16 + 8 + i]);
        printf("\n");
    }
    return 0;
}
