// launch.h -- host-side launchers of the jet kernels (template dispatch on
// stream layout / activation / PDE), split over translation units so the
// sm_100a build compiles in parallel.
#pragma once
#include <cuda_runtime.h>
#include "kernels_simt.cuh"
#include "tc_gemm.cuh"

#include <atomic>
#include <cstdint>
#include <string>

struct pnx_ctx;

namespace pnx {
// device pointer of the context's last Poynting penalty (NULL when disabled)
const double* ctx_penalty_ptr(pnx_ctx* c);
// message returned by pnx_create_error() (pnx_dp_create failures)
void set_create_error(const std::string& m);
// Dynamic shared-memory opt-in of kernel `Kern` for the CURRENT device (function
// attributes are per device), remembered per device ordinal; thread-safe (racing
// threads may both set the attribute, which is idempotent).
template <auto Kern>
inline int ensure_smem(int smem) {
    static std::atomic<int> done_bytes[64];  // largest opt-in per device ordinal
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::atomic<int>& d = done_bytes[dev & 63];
    int prev = d.load(std::memory_order_acquire);
    if (smem <= prev) return 0;
    if (cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
    while (smem > prev && !d.compare_exchange_weak(prev, smem)) {
    }
    return 0;
}
// SM count of the current device (cached per device ordinal)
inline int device_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int n = cache[dev & 63].load(std::memory_order_relaxed);
    if (n == 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n < 2) n = 2;
        cache[dev & 63].store(n, std::memory_order_relaxed);
    }
    return n;
}

void launch_input(int L, const InputArgs& a, cudaStream_t st);
void launch_input_bwd(int L, const InputArgs& a, const float* Hb, double* partP, int grid, cudaStream_t st);
void launch_gemm(int L, int pro, int epi, int eact, const GemmArgs& g, cudaStream_t st);
void launch_wgrad(int L, int pro, const WgradArgs& w, int nsplit, cudaStream_t st);
void launch_head(int pde, int act, const HeadArgs& h, int grid, cudaStream_t st);
void launch_layer0_fwd(int L, int act, const InputArgs& a, const float* W0, const float* b0, float* Z0, int H,
                       unsigned* amax, cudaStream_t st);
void launch_layer0_wgrad(int L, const InputArgs& a, const float* Zb0, int H, double* part, int grid, cudaStream_t st);
int launch_tc_layer(int L, int mode, int pro, const TcGemmArgs& g, cudaStream_t st);
int launch_tc2_fwd(int L, int pro, const TcGemmArgs& g, cudaStream_t st);
int launch_tc2_wgrad(int L, int pro, const TcWgradArgs& w, int ntiles, int wrows, cudaStream_t st);
struct SmallArgs;
int launch_small(int pde, int HP, const SmallArgs& a, int grid, cudaStream_t st);
void launch_small_finalize(const double* slot, int nblk, int64_t P, const double* loss_part, const double* inv_n,
                           float* grad, double* losses, cudaStream_t st);
}  // namespace pnx
