// launch.h -- host-side launchers of the jet kernels (template dispatch on
// stream layout / activation / PDE), split over translation units so the
// sm_100a build compiles in parallel.
#pragma once
#include <cuda_runtime.h>
#include "kernels_simt.cuh"
#include "tc_gemm.cuh"

namespace pnx {
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
}  // namespace pnx
