// launch_small.cu -- dispatch of the single-kernel narrow-network step (small_net.cuh).
#include <algorithm>
#include <cstdlib>

#include "launch.h"
#include "small_net.cuh"

namespace pnx {

template <int P, int HP, int NT>
int launch_small_t(const SmallArgs& a, int grid, cudaStream_t st) {
    constexpr int S = Streams<PdeTraits<P>::L>::S;
    const size_t smem = (size_t)sn_smem_floats(HP, S, a.D) * sizeof(float);
    constexpr auto kern = k_small_step<P, HP, NT>;
    if (ensure_smem<kern>((int)smem)) return -1;
    kern<<<grid, NT, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int P>
int launch_small_p(int HP, const SmallArgs& a, int grid, cudaStream_t st) {
    // 16 warps per CTA (32 warps measured slower: smaller register tiles make the
    // GEMM phases shared-memory bound, C1 0.159 -> 0.225 ms)
    return HP == 32 ? launch_small_t<P, 32, SN_THREADS>(a, grid, st) : launch_small_t<P, 64, SN_THREADS>(a, grid, st);
}

int launch_small(int pde, int HP, const SmallArgs& a, int grid, cudaStream_t st) {
    switch (pde) {
        case PDE_ADVECTION: return launch_small_p<PDE_ADVECTION>(HP, a, grid, st);
        case PDE_ALLEN_CAHN: return launch_small_p<PDE_ALLEN_CAHN>(HP, a, grid, st);
        case PDE_BURGERS: return launch_small_p<PDE_BURGERS>(HP, a, grid, st);
        case PDE_MAXWELL: return launch_small_p<PDE_MAXWELL>(HP, a, grid, st);
        case PDE_MAXWELL_EH: return launch_small_p<PDE_MAXWELL_EH>(HP, a, grid, st);
    }
    return -1;
}

void launch_small_finalize(const double* slot, int nblk, int64_t P, const double* loss_part, const double* inv_n,
                           float* grad, double* losses, cudaStream_t st) {
    k_small_finalize<<<(unsigned)std::min<int64_t>((P + 127) / 128, 1184), 128, 0, st>>>(slot, nblk, P, loss_part,
                                                                                       inv_n, grad, losses);
}

}  // namespace pnx
