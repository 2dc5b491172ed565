// launch_tc.cu -- dispatch of the tcgen05 (3xTF32) kernels.
#include "launch.h"

namespace pnx {

// ---- tcgen05 dispatch --------------------------------------------------------

template <int L, int MODE, int PRO, int NT>
int launch_tc_layer_t(const TcGemmArgs& g, cudaStream_t st) {
    constexpr int S = Streams<L>::S;
    using Cfg = TcFwdCfg<S, NT>;
    const int smem = Cfg::NST * Cfg::STAGE + 1024;
    auto kern = k_tc_layer<L, MODE, PRO, ACT_TANH, NT>;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
        attr = true;
    }
    const int grid = (g.Rpad / TC_M) * (g.N / NT);
    kern<<<grid, 256, smem, st>>>(g);
    return 0;
}
template <int L, int NT>
int launch_tc2_bwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc2BwdCfg<Streams<L>::S, NT>;
    const int smem = Cfg::SMEM;
    auto kern = k_tc2_bwd<L, NT>;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
        attr = true;
    }
    kern<<<(g.Rpad / TC_M) * (g.N / NT), TC3_THREADS, smem, st>>>(g);
    return 0;
}
template <int L>
int launch_tc_layer_l(int mode, int pro, const TcGemmArgs& g, cudaStream_t st) {
    constexpr int NT = tc_nt(Streams<L>::S);
    (void)mode;
    (void)pro;
    return launch_tc2_bwd_t<L, NT>(g, st);
}
int launch_tc_layer(int L, int mode, int pro, const TcGemmArgs& g, cudaStream_t st) {
    switch (L) {
        case LAY_XT: return launch_tc_layer_l<LAY_XT>(mode, pro, g, st);
        case LAY_AC: return launch_tc_layer_l<LAY_AC>(mode, pro, g, st);
        case LAY_MX: return launch_tc_layer_l<LAY_MX>(mode, pro, g, st);
        case LAY_NS: return launch_tc_layer_l<LAY_NS>(mode, pro, g, st);
    }
    return -1;
}

template <int L, int PRO, int NF>
int launch_tc2_fwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc3FwdCfg<NF>;
    const int smem = Cfg::SMEM;
    auto kern = k_tc2_fwd<L, PRO, NF>;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
        attr = true;
    }
    kern<<<g.Rpad / TC_M, TC3_THREADS, smem, st>>>(g);
    return 0;
}
template <int L>
int launch_tc2_fwd_l(int pro, const TcGemmArgs& g, cudaStream_t st) {
    if (g.N == 256) return pro == ACT_NONE ? launch_tc2_fwd_t<L, ACT_NONE, 256>(g, st) : launch_tc2_fwd_t<L, ACT_TANH, 256>(g, st);
    if (g.N == 128) return pro == ACT_NONE ? launch_tc2_fwd_t<L, ACT_NONE, 128>(g, st) : launch_tc2_fwd_t<L, ACT_TANH, 128>(g, st);
    return -1;
}
int launch_tc2_fwd(int L, int pro, const TcGemmArgs& g, cudaStream_t st) {
    switch (L) {
        case LAY_XT: return launch_tc2_fwd_l<LAY_XT>(pro, g, st);
        case LAY_AC: return launch_tc2_fwd_l<LAY_AC>(pro, g, st);
        case LAY_MX: return launch_tc2_fwd_l<LAY_MX>(pro, g, st);
        case LAY_NS: return launch_tc2_fwd_l<LAY_NS>(pro, g, st);
    }
    return -1;
}
template <int L, int PRO, int NF>
int launch_tc2_wgrad_t(const TcWgradArgs& w, int ntiles, cudaStream_t st) {
    using Cfg = Tc2WgCfg<NF>;
    const int smem = Cfg::NST * Cfg::STAGE + 1024;
    auto kern = k_tc2_wgrad<L, PRO, NF>;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1;
        attr = true;
    }
    kern<<<ntiles * (w.Kin / 128), TC2_THREADS, smem, st>>>(w, TC_WROWS);
    return 0;
}
template <int L>
int launch_tc2_wgrad_l(int pro, const TcWgradArgs& w, int ntiles, cudaStream_t st) {
    if (w.N == 256) return pro == ACT_NONE ? launch_tc2_wgrad_t<L, ACT_NONE, 256>(w, ntiles, st) : launch_tc2_wgrad_t<L, ACT_TANH, 256>(w, ntiles, st);
    if (w.N == 128) return pro == ACT_NONE ? launch_tc2_wgrad_t<L, ACT_NONE, 128>(w, ntiles, st) : launch_tc2_wgrad_t<L, ACT_TANH, 128>(w, ntiles, st);
    return -1;
}
int launch_tc2_wgrad(int L, int pro, const TcWgradArgs& w, int ntiles, cudaStream_t st) {
    switch (L) {
        case LAY_XT: return launch_tc2_wgrad_l<LAY_XT>(pro, w, ntiles, st);
        case LAY_AC: return launch_tc2_wgrad_l<LAY_AC>(pro, w, ntiles, st);
        case LAY_MX: return launch_tc2_wgrad_l<LAY_MX>(pro, w, ntiles, st);
        case LAY_NS: return launch_tc2_wgrad_l<LAY_NS>(pro, w, ntiles, st);
    }
    return -1;
}

}  // namespace pnx
