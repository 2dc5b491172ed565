// mma_sync_probe.cu -- throughput of the warp-level mma.sync shapes on sm_100a
// (dev tool): chains of independent m16n8k8 tf32 / m16n8k16 f16 MMAs per warp,
// 16 warps per CTA, one CTA per SM. Prints chip-wide TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(512, 1) probe(float* out, int iters) {
    float c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = 0.0f;
    unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3u, a2 = threadIdx.x * 5u, a3 = threadIdx.x * 7u;
    unsigned b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (KIND == 0) {
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else {
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, (size_t)nsm * 512 * 4);
    const int iters = 20000;
    for (int kind = 0; kind < 2; ++kind) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (kind == 0) probe<0><<<nsm, 512>>>(out, iters);
            else probe<1><<<nsm, 512>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double k = kind == 0 ? 8 : 16;
            const double flops = 2.0 * 16 * 8 * k * 8.0 * iters * 16 * nsm;  // per MMA x MMAs/warp x warps
            printf("%s: %.3f ms  %.1f TFLOP/s (%s)\n", kind == 0 ? "m16n8k8 tf32" : "m16n8k16 f16", ms,
                   flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
