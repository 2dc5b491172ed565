#include <cstdlib>
// launch_simt.cu -- dispatch of the FP32 CUDA-core (FFMA) kernels.
#include <algorithm>

#include "launch.h"

namespace pnx {

// ---- template dispatch -----------------------------------------------------

template <int L>
void launch_input_t(const InputArgs& a, cudaStream_t st) {
    const int per_row = a.rff_w > 0 ? a.rff_w : 1;
    const int64_t total = (int64_t)a.Rpad * per_row;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_input<L><<<grid, 256, 0, st>>>(a);
}
void launch_input(int L, const InputArgs& a, cudaStream_t st) {
    switch (L) {
        case LAY_XT: launch_input_t<LAY_XT>(a, st); break;
        case LAY_AC: launch_input_t<LAY_AC>(a, st); break;
        case LAY_MX: launch_input_t<LAY_MX>(a, st); break;
        case LAY_NS: launch_input_t<LAY_NS>(a, st); break;
    }
}
void launch_input_bwd(int L, const InputArgs& a, const float* Hb, double* partP, int grid, cudaStream_t st) {
    switch (L) {
        case LAY_XT: k_input_bwd<LAY_XT><<<grid, 256, 0, st>>>(a, Hb, partP); break;
        case LAY_AC: k_input_bwd<LAY_AC><<<grid, 256, 0, st>>>(a, Hb, partP); break;
        case LAY_MX: k_input_bwd<LAY_MX><<<grid, 256, 0, st>>>(a, Hb, partP); break;
        case LAY_NS: k_input_bwd<LAY_NS><<<grid, 256, 0, st>>>(a, Hb, partP); break;
    }
}

// Only the (prologue, epilogue) pairs the step uses are instantiated:
//   forward : PRO in {NONE (layer 0), act}, EPI_BIAS with EACT = act
//   reverse : PRO NONE, EPI_ACTT with EACT = act
//   input   : PRO NONE, EPI_RAW
template <int L, int ACT>
void launch_gemm_a(int pro, int epi, const GemmArgs& g, dim3 grid, cudaStream_t st) {
    if (epi == EPI_BIAS) {
        if (pro == ACT_NONE) k_gemm<L, ACT_NONE, EPI_BIAS, ACT><<<grid, 256, 0, st>>>(g);
        else k_gemm<L, ACT, EPI_BIAS, ACT><<<grid, 256, 0, st>>>(g);
    } else {
        k_gemm<L, ACT_NONE, EPI_ACTT, ACT><<<grid, 256, 0, st>>>(g);
    }
}
template <int L>
void launch_gemm_l(int pro, int epi, int eact, const GemmArgs& g, dim3 grid, cudaStream_t st) {
    if (epi == EPI_RAW) {
        k_gemm<L, ACT_NONE, EPI_RAW, ACT_NONE><<<grid, 256, 0, st>>>(g);
        return;
    }
    switch (eact) {
        case ACT_TANH: launch_gemm_a<L, ACT_TANH>(pro, epi, g, grid, st); break;
        case ACT_SINE: launch_gemm_a<L, ACT_SINE>(pro, epi, g, grid, st); break;
        default: launch_gemm_a<L, ACT_SWISH>(pro, epi, g, grid, st); break;
    }
}
void launch_gemm(int L, int pro, int epi, int eact, const GemmArgs& g, cudaStream_t st) {
    dim3 grid((unsigned)(g.Rpad / GT_M), (unsigned)((g.N + GT_N - 1) / GT_N));
    switch (L) {
        case LAY_XT: launch_gemm_l<LAY_XT>(pro, epi, eact, g, grid, st); break;
        case LAY_AC: launch_gemm_l<LAY_AC>(pro, epi, eact, g, grid, st); break;
        case LAY_MX: launch_gemm_l<LAY_MX>(pro, epi, eact, g, grid, st); break;
        case LAY_NS: launch_gemm_l<LAY_NS>(pro, epi, eact, g, grid, st); break;
    }
}

template <int L>
void launch_wgrad_l(int pro, const WgradArgs& w, dim3 grid, cudaStream_t st) {
    switch (pro) {
        case ACT_TANH: k_wgrad<L, ACT_TANH><<<grid, 256, 0, st>>>(w); break;
        case ACT_SINE: k_wgrad<L, ACT_SINE><<<grid, 256, 0, st>>>(w); break;
        case ACT_SWISH: k_wgrad<L, ACT_SWISH><<<grid, 256, 0, st>>>(w); break;
        default: k_wgrad<L, ACT_NONE><<<grid, 256, 0, st>>>(w); break;
    }
}
void launch_wgrad(int L, int pro, const WgradArgs& w, int nsplit, cudaStream_t st) {
    dim3 grid((unsigned)((w.N + 63) / 64), (unsigned)((w.K + 63) / 64), (unsigned)nsplit);
    switch (L) {
        case LAY_XT: launch_wgrad_l<LAY_XT>(pro, w, grid, st); break;
        case LAY_AC: launch_wgrad_l<LAY_AC>(pro, w, grid, st); break;
        case LAY_MX: launch_wgrad_l<LAY_MX>(pro, w, grid, st); break;
        case LAY_NS: launch_wgrad_l<LAY_NS>(pro, w, grid, st); break;
    }
}

template <int P, int ACT, int J>
void launch_head_a(const HeadArgs& h, int grid, cudaStream_t st) {
    const int smem = kHeadWarps * (h.H * PdeTraits<P>::F + PdeTraits<P>::F) * (int)sizeof(double);
    constexpr auto kern = k_head<P, ACT, J>;
    ensure_smem<kern>(smem);  // smem grows with H: the per-device opt-in keeps the largest
    kern<<<grid, 32 * kHeadWarps, smem, st>>>(h);
}
template <int P, int J>
void launch_head_j(int act, const HeadArgs& h, int grid, cudaStream_t st) {
    switch (act) {
        case ACT_TANH: launch_head_a<P, ACT_TANH, J>(h, grid, st); break;
        case ACT_SINE: launch_head_a<P, ACT_SINE, J>(h, grid, st); break;
        default: launch_head_a<P, ACT_SWISH, J>(h, grid, st); break;
    }
}
template <int P>
void launch_head_p(int act, const HeadArgs& h, int grid, cudaStream_t st) {
    if (h.H <= 32) launch_head_j<P, 1>(act, h, grid, st);
    else if (h.H <= 64) launch_head_j<P, 2>(act, h, grid, st);
    else if (h.H <= 128) launch_head_j<P, 4>(act, h, grid, st);
    else if (h.H <= 256) launch_head_j<P, 8>(act, h, grid, st);
    else launch_head_j<P, 16>(act, h, grid, st);
}
void launch_head(int pde, int act, const HeadArgs& h, int grid, cudaStream_t st) {
    switch (pde) {
        case PDE_ADVECTION: launch_head_p<PDE_ADVECTION>(act, h, grid, st); break;
        case PDE_ALLEN_CAHN: launch_head_p<PDE_ALLEN_CAHN>(act, h, grid, st); break;
        case PDE_BURGERS: launch_head_p<PDE_BURGERS>(act, h, grid, st); break;
        case PDE_MAXWELL: launch_head_p<PDE_MAXWELL>(act, h, grid, st); break;
        case PDE_MAXWELL_EH: launch_head_p<PDE_MAXWELL_EH>(act, h, grid, st); break;
        case PDE_NS: launch_head_p<PDE_NS>(act, h, grid, st); break;
    }
}

template <int L>
void launch_layer0_fwd_l(int act, const InputArgs& a, const float* W0, const float* b0, float* Z0, int H,
                         unsigned* amax, cudaStream_t st) {
    const int grid = std::min(148 * 8, (a.Rpad + L0_ROWS - 1) / L0_ROWS);
    switch (act) {
        case ACT_TANH: k_layer0_fwd<L, ACT_TANH><<<grid, 256, 0, st>>>(a, W0, b0, Z0, H, amax); break;
        case ACT_SINE: k_layer0_fwd<L, ACT_SINE><<<grid, 256, 0, st>>>(a, W0, b0, Z0, H, amax); break;
        default: k_layer0_fwd<L, ACT_SWISH><<<grid, 256, 0, st>>>(a, W0, b0, Z0, H, amax); break;
    }
}
void launch_layer0_fwd(int L, int act, const InputArgs& a, const float* W0, const float* b0, float* Z0, int H,
                       unsigned* amax, cudaStream_t st) {
    switch (L) {
        case LAY_XT: launch_layer0_fwd_l<LAY_XT>(act, a, W0, b0, Z0, H, amax, st); break;
        case LAY_AC: launch_layer0_fwd_l<LAY_AC>(act, a, W0, b0, Z0, H, amax, st); break;
        case LAY_MX: launch_layer0_fwd_l<LAY_MX>(act, a, W0, b0, Z0, H, amax, st); break;
        case LAY_NS: launch_layer0_fwd_l<LAY_NS>(act, a, W0, b0, Z0, H, amax, st); break;
    }
}
template <int L, int NC>
static bool launch_l0w_stream_nc(const InputArgs& a, const float* Zb0, int H, double* part, int grid, cudaStream_t st) {
    const int warps = grid * 8;
    const int rpw = (int)((((int64_t)a.nrows + warps - 1) / warps + 31) / 32 * 32);
    if (a.E <= 3) k_layer0_wgrad_stream<L, 3, NC><<<grid, 256, 0, st>>>(a, Zb0, H, rpw, part);
    else if (a.E <= 4) k_layer0_wgrad_stream<L, 4, NC><<<grid, 256, 0, st>>>(a, Zb0, H, rpw, part);
    else if (a.E <= 6) k_layer0_wgrad_stream<L, 6, NC><<<grid, 256, 0, st>>>(a, Zb0, H, rpw, part);
    else if (a.E <= 8) k_layer0_wgrad_stream<L, 8, NC><<<grid, 256, 0, st>>>(a, Zb0, H, rpw, part);
    else return false;
    return true;
}
template <int L>
static bool launch_l0w_stream(const InputArgs& a, const float* Zb0, int H, double* part, int grid, cudaStream_t st) {
    if (getenv("PNX_L0W_OLD")) return false;
    if (H == 256) return launch_l0w_stream_nc<L, 8>(a, Zb0, H, part, grid, st);
    if (H == 128) return launch_l0w_stream_nc<L, 4>(a, Zb0, H, part, grid, st);
    return false;
}
void launch_layer0_wgrad(int L, const InputArgs& a, const float* Zb0, int H, double* part, int grid, cudaStream_t st) {
    bool done = false;
    switch (L) {
        case LAY_XT: done = launch_l0w_stream<LAY_XT>(a, Zb0, H, part, grid, st); break;
        case LAY_AC: done = launch_l0w_stream<LAY_AC>(a, Zb0, H, part, grid, st); break;
        case LAY_MX: done = launch_l0w_stream<LAY_MX>(a, Zb0, H, part, grid, st); break;
        case LAY_NS: done = launch_l0w_stream<LAY_NS>(a, Zb0, H, part, grid, st); break;
    }
    if (done) return;
    switch (L) {
        case LAY_XT: k_layer0_wgrad<LAY_XT><<<grid, 256, 0, st>>>(a, Zb0, H, part); break;
        case LAY_AC: k_layer0_wgrad<LAY_AC><<<grid, 256, 0, st>>>(a, Zb0, H, part); break;
        case LAY_MX: k_layer0_wgrad<LAY_MX><<<grid, 256, 0, st>>>(a, Zb0, H, part); break;
        case LAY_NS: k_layer0_wgrad<LAY_NS><<<grid, 256, 0, st>>>(a, Zb0, H, part); break;
    }
}

}  // namespace pnx
