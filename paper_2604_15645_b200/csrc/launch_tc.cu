// launch_tc.cu -- dispatch of the tcgen05 (3xTF32) kernels.
#include "launch.h"

#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdlib>

namespace pnx {

int tc_make_tmap(CUtensorMap* map, const float* base, int rank, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                 uint32_t b1, uint32_t b2, bool sw128) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return -1;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<float*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

// ---- tcgen05 dispatch --------------------------------------------------------

template <int L, int NT, bool PAIR, bool F16 = false>
int launch_tc2_bwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc2BwdCfg<Streams<L>::S, NT, PAIR>;
    const int smem = Cfg::SMEM;
    constexpr auto kern = k_tc2_bwd<L, NT, PAIR, F16>;
    if (ensure_smem<kern>(smem)) return -1;
    TcGemmArgs a = g;
    if (PAIR && tc_make_tmap(&a.tmB, g.img, 2, 8, (uint64_t)(g.N / NT) * (g.K / 8) * 2 * NT, 1, 8, Cfg::NTL, 1, false))
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((g.Rpad / TC_M) * (g.N / NT));
    cfg.blockDim = dim3(TC3_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = PAIR ? 2 : 1;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? 0 : -1;
}
template <int L, bool PAIR, bool F16>
int launch_tc5_bwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc5BwdCfg<L, PAIR>;
    constexpr auto kern = k_tc5_bwd<L, PAIR, F16>;
    if (ensure_smem<kern>(Cfg::SMEM)) return -1;
    TcGemmArgs a = g;
    if (PAIR && tc_make_tmap(&a.tmB, g.img, 2, 8, (uint64_t)(g.K / (F16 ? 16 : 8)) * 2 * Cfg::NF, 1, 8, Cfg::NFL, 1,
                             false))
        return -1;
    cudaLaunchConfig_t cfg = {};
    // persistent: one CTA (pair) per SM (pair of SMs) walking the row tiles;
    // PNX_TC5_ONESHOT=1: one tile per CTA (the round-1 launch, A/B)
    static const bool oneshot = getenv("PNX_TC5_ONESHOT") != nullptr;
    const int nsm = device_sm_count();
    const int ntiles = g.Rpad / (PAIR ? 256 : TC_M);
    const int groups = oneshot ? ntiles : (PAIR ? std::min(nsm / 2, ntiles) : std::min(nsm, ntiles));
    cfg.gridDim = dim3(PAIR ? 2 * groups : groups);
    cfg.blockDim = dim3(TC3_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = PAIR ? 2 : 1;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? 0 : -1;
}
template <int L>
int launch_tc_layer_l(int mode, int pro, const TcGemmArgs& g, cudaStream_t st) {
    if constexpr (L == LAY_XT || L == LAY_MX) {
        // the pair variant is bit-identical but not faster (the MMA phase is shared-
        // memory bound, tools/trace_bwd5.cu), so it is opt-in
        static const bool pair5 = getenv("PNX_TC5_PAIR") != nullptr;
        if (tc5_bwd_ok(L, g.N, g.K)) {
            if (g.f16)
                return pair5 && g.Rpad % 256 == 0 ? launch_tc5_bwd_t<L, true, true>(g, st)
                                                  : launch_tc5_bwd_t<L, false, true>(g, st);
            return pair5 && g.Rpad % 256 == 0 ? launch_tc5_bwd_t<L, true, false>(g, st)
                                              : launch_tc5_bwd_t<L, false, false>(g, st);
        }
    }
    if (g.f16) return launch_tc2_bwd_t<L, tc_nt(Streams<L>::S), false, true>(g, st);  // 3xFP16, single CTA
    constexpr int NT = tc_nt(Streams<L>::S);
    (void)mode;
    (void)pro;
    // the pair variant is bit-identical but not faster (N=128 MMAs are tensor-pipe
    // bound, not smem bound: tools/trace_bwd.cu), so it is opt-in
    static const bool pair = getenv("PNX_BWD_PAIR") != nullptr;
    if (pair && NT == 128 && g.Rpad % 256 == 0) return launch_tc2_bwd_t<L, NT, true>(g, st);
    return launch_tc2_bwd_t<L, NT, false>(g, st);
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

template <int L, int PRO, int NF, bool F16 = false>
int launch_tc2_fwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc3FwdCfg<NF>;
    const int smem = Cfg::SMEM;
    constexpr auto kern = k_tc2_fwd<L, PRO, NF, F16>;
    if (ensure_smem<kern>(smem)) return -1;
    kern<<<g.Rpad / TC_M, TC3_THREADS, smem, st>>>(g);
    return 0;
}
template <int L, int PRO, bool F16>
int launch_tc4_fwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc4FwdCfg<L>;
    const int smem = Cfg::SMEM;
    constexpr auto kern = k_tc4_fwd<L, PRO, F16>;
    if (ensure_smem<kern>(smem)) return -1;
    TcGemmArgs a = g;
    constexpr int S = Streams<L>::S;
    const int nkb = g.K / (F16 ? 16 : 8);
    if (tc_make_tmap(&a.tmA, g.A, 3, g.K, g.Rpad, S, 32, 128, 1, true) ||
        tc_make_tmap(&a.tmB, g.img, 2, 8, (uint64_t)nkb * 2 * Cfg::NF, 1, 8, 128, 1, false) ||
        tc_make_tmap(&a.tmO, g.out, 3, Cfg::NF, g.Rpad, S, 32, 32, 1, true))
        return -1;
    cudaLaunchConfig_t cfg = {};
    // persistent pairs: one per two SMs (each walks tiles pair, pair + npairs, ...)
    const int nsm = device_sm_count();
    const int ntiles = g.Rpad / 256;
    cfg.gridDim = dim3(2 * (ntiles < nsm / 2 ? ntiles : nsm / 2));
    cfg.blockDim = dim3(TC4_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? 0 : -1;
}
template <int L>
int launch_tc2_fwd_l(int pro, const TcGemmArgs& g, cudaStream_t st) {
    static const bool pair = getenv("PNX_FWD_NOPAIR") == nullptr;
    if (g.N == 256 && pair && g.Rpad % 256 == 0 && g.K % 32 == 0) {
        if (g.f16)
            return pro == ACT_NONE ? launch_tc4_fwd_t<L, ACT_NONE, true>(g, st)
                                   : launch_tc4_fwd_t<L, ACT_TANH, true>(g, st);
        return pro == ACT_NONE ? launch_tc4_fwd_t<L, ACT_NONE, false>(g, st)
                               : launch_tc4_fwd_t<L, ACT_TANH, false>(g, st);
    }
    if (g.f16) {  // 3xFP16 single-CTA forward (the producer -- a layer or k_input -- recorded the bounds)
        if (g.N == 256)
            return pro == ACT_NONE ? launch_tc2_fwd_t<L, ACT_NONE, 256, true>(g, st)
                                   : launch_tc2_fwd_t<L, ACT_TANH, 256, true>(g, st);
        if (g.N == 128)
            return pro == ACT_NONE ? launch_tc2_fwd_t<L, ACT_NONE, 128, true>(g, st)
                                   : launch_tc2_fwd_t<L, ACT_TANH, 128, true>(g, st);
        return -1;
    }
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
template <int L, int PRO, int NF, bool PAIR, bool F16 = false>
int launch_tc2_wgrad_t(const TcWgradArgs& w, int ntiles, int segrows, cudaStream_t st) {
    using Cfg = Tc2WgCfg<Streams<L>::S, NF, PAIR>;
    const int smem = Cfg::SMEM;
    constexpr auto kern = k_tc2_wgrad<L, PRO, NF, PAIR, F16>;
    if (ensure_smem<kern>(smem)) return -1;
    TcWgradArgs a = w;
    constexpr int S = Streams<L>::S;
    if (tc_make_tmap_3d(&a.tmA, w.A, w.Kin, w.Rpad, S, 128, 8, S) ||
        tc_make_tmap_3d(&a.tmB, w.Bm, NF, w.Rpad, S, Cfg::NFL, 8, S))
        return -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles * (w.Kin / 128));
    cfg.blockDim = dim3(TCW_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = PAIR ? 2 : 1;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, segrows, ntiles) == cudaSuccess ? 0 : -1;
}
template <int L, int NF, bool PAIR>
int launch_tc2_wgrad_p(int pro, const TcWgradArgs& w, int ntiles, int wrows, cudaStream_t st) {
    // 3xFP16 operands (the producers recorded the per-stream bounds)
    if (w.f16 && w.amaxA && w.amaxB)
        return pro == ACT_NONE ? launch_tc2_wgrad_t<L, ACT_NONE, NF, PAIR, true>(w, ntiles, wrows, st)
                               : launch_tc2_wgrad_t<L, ACT_TANH, NF, PAIR, true>(w, ntiles, wrows, st);
    return pro == ACT_NONE ? launch_tc2_wgrad_t<L, ACT_NONE, NF, PAIR>(w, ntiles, wrows, st)
                           : launch_tc2_wgrad_t<L, ACT_TANH, NF, PAIR>(w, ntiles, wrows, st);
}
template <int L>
int launch_tc2_wgrad_l(int pro, const TcWgradArgs& w, int ntiles, int wrows, cudaStream_t st) {
    static const bool pair = getenv("PNX_WG_NOPAIR") == nullptr;
    if (w.N == 256 && w.Kin == 256 && pair) return launch_tc2_wgrad_p<L, 256, true>(pro, w, ntiles, wrows, st);
    if (w.N == 256) return launch_tc2_wgrad_p<L, 256, false>(pro, w, ntiles, wrows, st);
    if (w.N == 128) return launch_tc2_wgrad_p<L, 128, false>(pro, w, ntiles, wrows, st);
    return -1;
}
int launch_tc2_wgrad(int L, int pro, const TcWgradArgs& w, int ntiles, int wrows, cudaStream_t st) {
    switch (L) {
        case LAY_XT: return launch_tc2_wgrad_l<LAY_XT>(pro, w, ntiles, wrows, st);
        case LAY_AC: return launch_tc2_wgrad_l<LAY_AC>(pro, w, ntiles, wrows, st);
        case LAY_MX: return launch_tc2_wgrad_l<LAY_MX>(pro, w, ntiles, wrows, st);
        case LAY_NS: return launch_tc2_wgrad_l<LAY_NS>(pro, w, ntiles, wrows, st);
    }
    return -1;
}

}  // namespace pnx
