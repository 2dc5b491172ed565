// tc_gemm.cuh -- tcgen05 (5th-gen tensor core) 3xTF32 path (placeholder until
// the sm_100a kernels land; the FFMA engine is used meanwhile).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "kernels_simt.cuh"

namespace pnx {
struct TcWorkspace {
    int dummy = 0;
};
inline int tc_workspace_alloc(TcWorkspace&, int, int64_t, int, int) { return 0; }
inline void tc_workspace_free(TcWorkspace&) {}
inline bool tc_enabled(int, int, int) { return false; }
inline int tc_forward(TcWorkspace&, int, int, const GemmArgs&, cudaStream_t, int64_t*) { return -1; }
inline int tc_backward(TcWorkspace&, int, int, const GemmArgs&, cudaStream_t, int64_t*) { return -1; }
inline int tc_wgrad(TcWorkspace&, int, int, const WgradArgs&, int, cudaStream_t, int64_t*) { return -1; }
}  // namespace pnx
