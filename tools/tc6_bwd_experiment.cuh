// tc6_bwd_experiment.cuh -- EXPERIMENT, not built into libpnx (measured slower than
// k_tc5_bwd at S = 4). Used by tools/trace_bwd6.cu.
//
// First-order tanh backward (LAY_XT S = 3, LAY_MX S = 4, N = 256,
// 3xFP16) with the epilogue of one stream overlapping the MMAs of the next.
//
// k_tc5_bwd runs two streams per pass into both halves of TMEM, so every pass's
// MMAs wait for the previous pass's drain. Here each pass is ONE stream
// (N = 256, one accumulator: 96% of the two-accumulator issue rate,
// profiles/round1/tcgen05_mma_rate_probe_f16.txt) and TMEM holds two pass
// buffers: the epilogue of pass p reads buffer p & 1 while the MMAs of pass p+1
// fill the other. Streams run 1, 2, (3,) 0: zb_s = d hb_s for s >= 1 while
// P = sum_s z_s hb_s accumulates in shared memory (same order as k_tc5_bwd), then
// zb_0 = d (hb_0 - 2 t P).
//
// The epilogue needs no staging: tcgen05.ld.16x256b gives a thread rows
// (l, l + 8) x columns (2q, 2q + 1) of every 8-column group
// (tools/tmem_layout_probe.cu); the weight image's rows are permuted within each
// 16-feature block (k_tc_prep_image16, perm16) so that those TMEM columns are 4
// consecutive features -- one float4 of t, z and the output per row, 32 B runs
// per 4 lanes, straight from / to global memory. The freed ring space buys a
// 4-stage operand ring next to the 128 KB of P.
// Results are bit-identical to k_tc5_bwd<L, false, true> (same MMA order per
// stream, same epilogue arithmetic).
#pragma once
#include "../paper_2604_15645_b200/csrc/tc_gemm.cuh"

#ifndef PNX_TC6_LOOK
#define PNX_TC6_LOOK 3
#endif

namespace pnx {

// TMEM column of feature f: within each 16-feature block, f % 16 = 4q + 2j + e
// goes to column 8j + 2q + e (so a 16x256b.x2 load gives 4 consecutive features)
__host__ __device__ constexpr int tc6_col_of_feature(int f) {
    return (f & ~15) | (((f >> 1) & 1) << 3) | (((f >> 2) & 3) << 1) | (f & 1);
}

// k_tc_prep_image16 (transpose_b = 1, NT = 256) with the rows in tc6 column order
static __global__ void k_tc6_prep_image16(const float* __restrict__ W, int K, int N,
                                          const unsigned* __restrict__ wamax, uint16_t* __restrict__ img) {
    const int rowsB = K, KB = N;
    const float sc = ldexpf(1.0f, tc::f16_exp_bits(*wamax));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)rowsB * KB;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i / KB), k = (int)(i % KB);
        const float w = W[(int64_t)n * N + k] * sc;
        const __half hi = __float2half_rn(w);
        const __half lo = __float2half_rn(w - __half2float(hi));
        const int64_t blk = (int64_t)(k / 16) * (2 * 256 * 16);
        const uint32_t off = tc::sw32h_off((uint32_t)tc6_col_of_feature(n % 256), (uint32_t)(k % 16)) / 2;
        img[blk + off] = __half_as_ushort(hi);
        img[blk + 256 * 16 + off] = __half_as_ushort(lo);
    }
}

// PAIR: a 2-CTA cluster covers 256 rows with cta_group::2 MMAs (M = 256); each
// CTA stages half of the weight rows, halving the per-SM weight traffic.
template <int L, bool PAIR = false>
struct Tc6BwdCfg {
    static constexpr int S = Streams<L>::S;
    static constexpr int NF = 256;
    static constexpr int NFL = PAIR ? NF / 2 : NF;    // weight rows staged by this CTA
    static constexpr int NP = S;                      // passes per tile, one stream each
    static constexpr int A_T = TC_TILE_BYTES;         // 128 rows x 16 fp16
    static constexpr int B_T = NFL * 32;              // weight rows x 16 fp16
    static constexpr int STAGE = 2 * A_T + 2 * B_T;   // A hi, lo ; B hi, lo
    static constexpr int P_BYTES = TC_M * NF * 4;
    static constexpr int NST = (227 * 1024 - P_BYTES - 1024) / STAGE;
    static constexpr int SMEM = NST * STAGE + P_BYTES + 1024;
    static_assert(NST >= 3, "tc6 operand ring");
    static_assert(SMEM <= 227 * 1024, "tc6 shared memory");
    __host__ __device__ static constexpr int stream(int pass) { return pass + 1 < S ? pass + 1 : 0; }
};

namespace tc6 {
__device__ __forceinline__ void tmem_ld_x2(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
// the wait carries the registers, so no use of them can be scheduled above it
template <int G>
__device__ __forceinline__ void tmem_wait(uint32_t (&r)[G][8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int g = 0; g < G; ++g)
        asm volatile("" : "+r"(r[g][0]), "+r"(r[g][1]), "+r"(r[g][2]), "+r"(r[g][3]), "+r"(r[g][4]), "+r"(r[g][5]),
                     "+r"(r[g][6]), "+r"(r[g][7]));
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
}  // namespace tc6

template <int L, bool PAIR = false>
__global__ void __launch_bounds__(TC3_THREADS, 1) k_tc6_bwd(const __grid_constant__ TcGemmArgs g) {
    using Cfg = Tc6BwdCfg<L, PAIR>;
    constexpr int NST = Cfg::NST, NF = Cfg::NF, NP = Cfg::NP;
    constexpr int G = 2;  // 16-column blocks per epilogue step (registers bound it)
    static_assert(L == LAY_XT || L == LAY_MX, "first-order layouts only");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[NST], empty[NST], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // persistent: CTA blockIdx.x walks tiles blockIdx.x, + gridDim.x, ...; the pass
    // index gp = NP * local tile + pass keeps every barrier counting across tiles
    const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
    const int ngrp = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x, grp = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ntiles = g.Rpad / (PAIR ? 2 * TC_M : TC_M);
    const int nloc = grp < ntiles ? (ntiles - 1 - grp) / ngrp + 1 : 0;
    const int npass = NP * nloc;
    auto row0 = [&](int lt) { return PAIR ? (grp + lt * ngrp) * 2 * TC_M + (int)rank * TC_M : (grp + lt * ngrp) * TC_M; };
    const int nkb = g.K / 16;
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * NF;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], PAIR ? 17 : 9);  // producer warps (both CTAs) + the weight copy's expect_tx
            tc::mbar_init(&empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], PAIR ? 16 : 8);  // the epilogue warps (of both CTAs)
        }
        tc::fence_barrier_init();
    }
    if (warp == 8) {
        if constexpr (PAIR) tc::tmem_alloc_pair<512>(&tmem_base);
        else tc::tmem_alloc<512>(&tmem_base);
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t sbase = tc::smem_u32(smem);
    const uint32_t sP = sbase + NST * Cfg::STAGE;
    // the leader's barriers as cluster addresses (PAIR)
    const uint32_t full0 = PAIR ? tc::mapa(tc::smem_u32(&full[0]), 0) : tc::smem_u32(&full[0]);
    const uint32_t tempty0 = PAIR ? tc::mapa(tc::smem_u32(&tempty[0]), 0) : tc::smem_u32(&tempty[0]);

    if (warp < 8) {
        // ---------------- producers: A = Zb_out[s] rows, fp16 hi/lo, one k-step per stage ----------------
        const int prow = tid >> 1, pc = tid & 1;
        const uint32_t aoff = tc::sw32_chunk((uint32_t)prow, (uint32_t)pc);
#pragma unroll 1
        for (int gp = 0; gp < npass; ++gp) {
            const int s = Cfg::stream(gp % NP);
            const float* asrc = g.A + s * RK + (int64_t)(row0(gp / NP) + prow) * g.K + pc * 8;
            const float sc = ldexpf(1.0f, tc::f16_exp_bits(g.amax_in[s]));
            constexpr int D = 2;
            float4 ra[D][2];
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int u = 0; u < 2; ++u)
                    ra[d][u] = d < nkb ? ldg4(asrc + d * 16 + 4 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int kb0 = 0; kb0 < nkb; kb0 += D)
#pragma unroll
                for (int cur = 0; cur < D; ++cur) {
                    const int kb = kb0 + cur;
                    if (kb >= nkb) break;
                    uint4 ahi, alo;
                    {
                        const float h[8] = {ra[cur][0].x, ra[cur][0].y, ra[cur][0].z, ra[cur][0].w,
                                            ra[cur][1].x, ra[cur][1].y, ra[cur][1].z, ra[cur][1].w};
                        tc::split_h8(h, sc, ahi, alo);
                    }
                    if (kb + D < nkb) {
#pragma unroll
                        for (int u = 0; u < 2; ++u) ra[cur][u] = ldg4(asrc + (kb + D) * 16 + 4 * u);
                    }
                    const int it = gp * nkb + kb, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        if (tid == 0) TC_ACC(2);
                    }
                    if (tid == 0) {
                        if constexpr (PAIR) {
                            // image rows (32 B) of k-step kb: [hi: 256][lo: 256]; this CTA's half
                            const int rowb = kb * 2 * NF + (int)rank * Cfg::NFL;
                            if (rank == 0) tc::mbar_arrive_expect_tx(&full[st], 2 * 2 * Cfg::B_T);
                            tc::tma_load_2d_pair(stage + 2 * Cfg::A_T, &g.tmB, 0, rowb, full0 + st * 8);
                            tc::tma_load_2d_pair(stage + 2 * Cfg::A_T + Cfg::B_T, &g.tmB, 0, rowb + NF, full0 + st * 8);
                        } else {
                            tc::mbar_arrive_expect_tx(&full[st], 2 * Cfg::B_T);
                            tc::bulk_g2s(stage + 2 * Cfg::A_T, g.img + (int64_t)kb * (2 * Cfg::B_T / 4), 2 * Cfg::B_T,
                                         &full[st]);
                        }
                    }
                    sts128u(stage + aoff, ahi);
                    sts128u(stage + Cfg::A_T + aoff, alo);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                        else tc::mbar_arrive(&full[st]);
                    }
                }
        }
    } else if (warp == 8) {
        // ---------------- MMA issuer: pass gp into TMEM buffer gp & 1 ----------------
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = tc::make_idesc_f16(PAIR ? 2 * TC_M : TC_M, NF, 0, 0);
            for (int gp = 0; gp < npass; ++gp) {
                const int b = gp & 1, u = gp >> 1;
                if (u > 0) {  // buffer drained
                    TC_T0();
                    tc::mbar_wait(&tempty[b], (uint32_t)(u - 1) & 1u);
                    TC_ACC(1);
                }
                tc::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(b * NF);
                for (int kb = 0; kb < nkb; ++kb) {
                    const int it = gp * nkb + kb, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                        TC_ACC(0);
                    }
                    tc::tc_fence_after();
                    const uint64_t adh = tc::make_sdesc(stage, 16, 256, 6);
                    const uint64_t adl = tc::make_sdesc(stage + Cfg::A_T, 16, 256, 6);
                    const uint64_t bh = tc::make_sdesc(stage + 2 * Cfg::A_T, 16, 256, 6);
                    const uint64_t bl = tc::make_sdesc(stage + 2 * Cfg::A_T + Cfg::B_T, 16, 256, 6);
                    if constexpr (PAIR) {
                        tc::mma_f16_pair(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_f16_pair(d, adh, bl, idesc, 1u);
                        tc::mma_f16_pair(d, adl, bh, idesc, 1u);
                        tc::mma_commit_pair(&empty[st], 3);
                    } else {
                        tc::mma_f16(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_f16(d, adh, bl, idesc, 1u);
                        tc::mma_f16(d, adl, bh, idesc, 1u);
                        tc::mma_commit(&empty[st]);
                    }
                }
                if constexpr (PAIR) tc::mma_commit_pair(&tfull[b], 3);
                else tc::mma_commit(&tfull[b]);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: warps 9-16, TMEM lane quarter warp % 4, column half ----------------
        const int ew = warp - 9, q4 = warp & 3, cq = ew >> 2;
        const uint32_t pw = sP + (uint32_t)ew * (32u * 32u * 16u);  // 32 float4 per lane, [slot][lane]
        uint64_t keep, stream_pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream_pol));
        const float usw = ldexpf(1.0f, -tc::f16_exp_bits(*g.amax_w));
        // The epilogue is latency-bound (one step of loads in flight per warp fits the
        // registers), so each step prefetches into L2 the rows LOOK steps ahead,
        // running into the next pass: lane l -> tensor l >> 4 (t, z_s), row l & 15 of
        // the 16-row half, one 128 B line (G = 2 blocks of 16 features).
        constexpr int NQ = 2 * (8 / G), LOOK = PNX_TC6_LOOK;
        auto prefetch = [&](int gp2, int q) {
            if (gp2 >= npass) return;
            const int s2 = Cfg::stream(gp2 % NP), h2 = q / (8 / G), blk2 = (q % (8 / G)) * G, tz = lane >> 4;
            if (tz == 1 && s2 == 0) return;
            const int row = row0(gp2 / NP) + 32 * q4 + 16 * h2 + (lane & 15);
            const float* p = g.Zlow + (tz ? s2 * RN : 0) + (int64_t)row * NF + 128 * cq + 16 * blk2;
            if (tz) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            else asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
        };
        for (int q = 0; q < LOOK; ++q) prefetch(0, q);
#pragma unroll 1
        for (int gp = 0; gp < npass; ++gp) {
            const int b = gp & 1, u = gp >> 1, pass = gp % NP, s = Cfg::stream(pass);
            const int r0 = row0(gp / NP);
            const float us = usw * ldexpf(1.0f, -tc::f16_exp_bits(g.amax_in[s]));
            // t = tanh z_0 is read by every pass of the tile: keep it in L2 until the last
            const uint64_t tpol = s == 0 ? stream_pol : keep;
            float mx = 0.0f;
            {
                TC_T0();
                tc::mbar_wait(&tfull[b], (uint32_t)u & 1u);
                if (ew == 0 && lane == 0) TC_ACC(4);
            }
            tc::tc_fence_after();
            TC_T0();
#pragma unroll 1
            for (int qi = 0; qi < NQ; ++qi) {
                {
                    const int qa = qi + LOOK;
                    if (qa < NQ) prefetch(gp, qa);
                    else prefetch(gp + 1, qa - NQ);
                }
                const int h = qi / (8 / G), blk0 = (qi % (8 / G)) * G;
                const int ra = 32 * q4 + 16 * h + (lane >> 2);  // rows ra, ra + 8 of the tile
                const int64_t rowA = (int64_t)(r0 + ra) * NF, rowB = rowA + 8 * NF;
                const uint32_t tl = tmem + ((uint32_t)(32 * q4 + 16 * h) << 16) + (uint32_t)(b * NF + 128 * cq);
                {
                    uint32_t hv[G][8];
                    float4 tA[G], tB[G], zA[G], zB[G], pA[G], pB[G];
#pragma unroll
                    for (int gi = 0; gi < G; ++gi) tc6::tmem_ld_x2(tl + (uint32_t)(16 * (blk0 + gi)), hv[gi]);
#pragma unroll
                    for (int gi = 0; gi < G; ++gi) {
                        const int f = 128 * cq + 16 * (blk0 + gi) + 4 * (lane & 3);
                        tA[gi] = tc6::ldg4_hint(g.Zlow + rowA + f, tpol);
                        tB[gi] = tc6::ldg4_hint(g.Zlow + rowB + f, tpol);
                        if (s > 0) {
                            zA[gi] = tc6::ldg4_hint(g.Zlow + s * RN + rowA + f, stream_pol);
                            zB[gi] = tc6::ldg4_hint(g.Zlow + s * RN + rowB + f, stream_pol);
                        }
                        const uint32_t slot = (uint32_t)(((h * 8 + blk0 + gi) * 2) * 32 + lane) * 16u;
                        if (pass > 0) {
                            pA[gi] = lds128(pw + slot);
                            pB[gi] = lds128(pw + slot + 32u * 16u);
                        }
                    }
                    tc6::tmem_wait<G>(hv);
#pragma unroll
                    for (int gi = 0; gi < G; ++gi) {
                        // row ra: registers {0,1,4,5} = features 4q..4q+3; row ra + 8: {2,3,6,7}
                        const int f = 128 * cq + 16 * (blk0 + gi) + 4 * (lane & 3);
                        const uint32_t slot = (uint32_t)(((h * 8 + blk0 + gi) * 2) * 32 + lane) * 16u;
#pragma unroll
                        for (int rs = 0; rs < 2; ++rs) {
                            const float hh[4] = {__uint_as_float(hv[gi][rs * 2 + 0]) * us,
                                                 __uint_as_float(hv[gi][rs * 2 + 1]) * us,
                                                 __uint_as_float(hv[gi][rs * 2 + 4]) * us,
                                                 __uint_as_float(hv[gi][rs * 2 + 5]) * us};
                            const float4 t4 = rs ? tB[gi] : tA[gi];
                            const float tt[4] = {t4.x, t4.y, t4.z, t4.w};
                            float zz[4] = {0.f, 0.f, 0.f, 0.f}, pp[4] = {0.f, 0.f, 0.f, 0.f};
                            if (s > 0) {
                                const float4 z4 = rs ? zB[gi] : zA[gi];
                                zz[0] = z4.x; zz[1] = z4.y; zz[2] = z4.z; zz[3] = z4.w;
                            }
                            if (pass > 0) {
                                const float4 p4 = rs ? pB[gi] : pA[gi];
                                pp[0] = p4.x; pp[1] = p4.y; pp[2] = p4.z; pp[3] = p4.w;
                            }
                            float o[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float t = tt[e];
                                const float d = 1.0f - t * t;
                                if (s > 0) {
                                    // zb_s = d hb_s ; P (+)= z_s hb_s (k_tc5_bwd's order)
                                    o[e] = d * hh[e];
                                    float P = pass > 0 ? pp[e] : 0.0f;
                                    P += zz[e] * hh[e];
                                    pp[e] = P;
                                } else {
                                    // zb_0 = d (hb_0 - 2 t P)
                                    float tbar = hh[e];
                                    tbar += -2.0f * t * pp[e];
                                    o[e] = d * tbar;
                                }
                                mx = fmaxf(mx, fabsf(o[e]));
                            }
                            if (s > 0) sts128(pw + slot + (uint32_t)rs * (32u * 16u), make_float4(pp[0], pp[1], pp[2], pp[3]));
                            float* dst = g.out + s * RN + (rs ? rowB : rowA) + f;
                            *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
                        }
                    }
                }
            }
            if (g.amax_out) tc::warp_amax(g.amax_out + s, __float_as_uint(mx));
            if (ew == 0 && lane == 0) TC_ACC(3);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) tc::mbar_arrive_cluster(tempty0 + b * 8);
                else tc::mbar_arrive(&tempty[b]);
            }
        }
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    if (warp == 8) {
        if constexpr (PAIR) tc::tmem_dealloc_pair<512>(tmem);
        else tc::tmem_dealloc<512>(tmem);
    }
}

template <int L, bool PAIR = false>
int launch_tc6_bwd_t(const TcGemmArgs& g, cudaStream_t st) {
    using Cfg = Tc6BwdCfg<L, PAIR>;
    constexpr auto kern = k_tc6_bwd<L, PAIR>;
    if (ensure_smem<kern>(Cfg::SMEM)) return -1;
    TcGemmArgs a = g;
    if (PAIR && tc_make_tmap(&a.tmB, g.img, 2, 8, (uint64_t)(g.K / 16) * 2 * Cfg::NF, 1, 8, Cfg::NFL, 1, false))
        return -1;
    // persistent: one CTA (pair) per SM (pair of SMs)
    const int nsm = device_sm_count();
    const int ntiles = g.Rpad / (PAIR ? 256 : TC_M);
    const int groups = PAIR ? std::min(nsm / 2, ntiles) : std::min(nsm, ntiles);
    cudaLaunchConfig_t cfg = {};
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

}  // namespace pnx
