// small_net.cuh -- the whole worker step of a narrow network in ONE kernel
// (C1: Burgers, tanh 4x64, 10k points; also the small golden models).
//
// At width <= 64 the multi-kernel path (input, L forward GEMMs, head, L reverse
// GEMMs, L weight gradients, reductions: ~24 launches) is launch- and
// latency-bound: C1 moves 2.25 GFLOP in 0.6 ms. Here one CTA per SM walks tiles
// of TR = 32 rows; for a tile everything stays in shared memory:
//
//   e    = input jets of the rows (FP64 embedding, model.cpp:134-154)
//   Z_l  = e W_0 (+b), then act(Z_{l-1}) W_l (+b)  -- all hidden layers kept
//   O    = act(Z_{D-1}) W_D + b_D, residual / IC / BC losses and seeds
//          (losses.cpp:26-144; the same device rules as k_head)
//   reverse: Zb_{l-1} = act^T(Zb_l W_l^T ; Z_{l-1}), dW_l += act(Z_{l-1})^T Zb_l,
//            db_l += colsum Zb_l[0]   (graph.cpp:468-502)
//
// Weights (zero-padded to HP = 32 or 64 features: padded features stay exactly
// zero through every activation rule and contribute nothing) live in shared
// memory for the whole launch. Activation tiles are [j = s*TR + r][feature]
// with a row stride of HP + 4 floats (16 B aligned, conflict-free LDS.128).
// GEMMs: lane = row r, warp = a group of HP/16 output features, all S streams
// per thread (the jet epilogues need every stream of an element together).
// Each thread owns a fixed block of every dW_l, sums it per tile in FP32 and
// adds that into its CTA's FP64 slot of the flat gradient (L2-resident,
// read-modify-write by that thread only: deterministic); bias sums are taken in
// FP64 per row, so contributions that cancel exactly in exact arithmetic (e.g.
// the IC term of an odd network on a symmetric IC grid) cancel to FP64 noise as
// in the reference, not to FP32 noise (which Adam's eps = 1e-8 would turn into
// a full step). k_small_finalize sums the CTA slots in fixed order in FP64.
// FP32 FMA elsewhere (the FFMA engine's accuracy).
#pragma once
#include "kernels_simt.cuh"

namespace pnx {

constexpr int SN_TR = 32;       // rows per tile (= lanes)
constexpr int SN_THREADS = 512;  // 16 warps
constexpr int SN_MAXK0 = 8;

struct SmallArgs {
    InputArgs ia;          // coordinates, embedding (no RFF)
    const float* params;   // flat trainable() vector
    LayerTab tab;
    int D, H, K0;          // hidden layers, width, embedded width
    int64_t T;             // rows [bc_a | ic | interior]
    int64_t bca0, bca1, ic0, ic1, int0, int1;
    int bc_mode;
    const float* ic_t;     // [F][n_ic]
    const float* bc_t;     // [F][n_bc]
    float w_pde, w_ic, w_bc;
    PdeConst pc;
    int* bad;
    float* resid_out;
    double* slot;          // [grid][P] FP64 gradient accumulators (one per CTA)
    double* loss_part;     // [grid][3]
    int64_t P;
};

// width 64: the hidden-layer contractions run as 3xTF32 warp MMAs
// (mma.sync m16n8k8: the FFMA loops were shared-memory-bandwidth bound --
// l1tex 73% busy -- and a fragment moves the same operands in 2.3x fewer
// shared-memory wavefronts); the weights then sit at a row stride of HP + 8
// (conflict-free B fragments of the forward)
__host__ __device__ constexpr bool sn_mma(int HP) { return HP == 64; }
__host__ __device__ constexpr int sn_ws(int HP) { return sn_mma(HP) ? HP + 8 : HP; }

// shared-memory footprint (floats) of a configuration
__host__ __device__ inline int64_t sn_smem_floats(int HP, int S, int D) {
    const int J = S * SN_TR, LD = HP + 4, WS = sn_ws(HP);
    const int64_t w = (int64_t)SN_MAXK0 * WS + (int64_t)(D - 1) * HP * WS + (int64_t)HP * 4 + (int64_t)D * HP + 4;
    return w + (int64_t)J * SN_MAXK0 + (int64_t)(D + 2) * J * LD + (int64_t)SN_TR * S * 4;
}

namespace sn {
// hi = x with the 13 low mantissa bits cleared (exact in TF32), lo = x - hi
// (exact in FP32); the tensor core reads lo's TF32 part, so |x - hi - lo'| is
// within 2^-21 |x| -- two integer/FP ops instead of two conversions
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    const uint32_t h = __float_as_uint(x) & 0xffffe000u;
    hi = h;
    lo = __float_as_uint(x - __uint_as_float(h));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// 3xTF32: c += al bh + ah bl + ah bh
__device__ __forceinline__ void mma3(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     const uint32_t (&bh)[2], const uint32_t (&bl)[2]) {
    mma_tf32(c, al, bh);
    mma_tf32(c, ah, bl);
    mma_tf32(c, ah, bh);
}
// A fragment (m16 x k8, row-major at stride ld) from FP32 shared memory, split
__device__ __forceinline__ void frag_a(const float* base, int ld, uint32_t (&ah)[4], uint32_t (&al)[4]) {
    split_tf32(base[0], ah[0], al[0]);
    split_tf32(base[8 * ld], ah[1], al[1]);
    split_tf32(base[4], ah[2], al[2]);
    split_tf32(base[8 * ld + 4], ah[3], al[3]);
}
}  // namespace sn

template <int P, int HP, int NT = SN_THREADS>
__global__ void __launch_bounds__(NT, 1) k_small_step(SmallArgs a) {
    using Tr = PdeTraits<P>;
    constexpr int L = Tr::L, F = Tr::F, K = Tr::K;
    constexpr int S = Streams<L>::S;
    constexpr int TR = SN_TR, J = S * TR, LD = HP + 4;
    constexpr int NWARP = NT / 32;
    constexpr bool MMA = sn_mma(HP) && NWARP == 16;
    constexpr int WS = MMA ? sn_ws(HP) : HP;                       // weight row stride
    constexpr int NC = HP / NWARP;                                 // output features per warp in the row GEMMs
    constexpr int EPT = HP * HP / NT;                              // dW entries per thread: BK x BN
    constexpr int BN = EPT >= 4 ? 4 : EPT;
    constexpr int BK = EPT / BN;
    static_assert(HP * HP == NT * BK * BN && NC >= 1, "dW blocks tile the weight");
    extern __shared__ float4 sn_smem4[];
    float* sm = reinterpret_cast<float*>(sn_smem4);
    const int D = a.D, H = a.H, K0 = a.K0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // ---- shared-memory carve-up ----
    float* W0 = sm;                                    // [8][WS]
    float* Wh = W0 + SN_MAXK0 * WS;                    // hidden l = 1..D-1: [HP][WS] each
    float* Wo = Wh + (int64_t)(D - 1) * HP * WS;       // head [HP][4]
    float* Bs = Wo + HP * 4;                           // biases [D][HP] + head [4]
    float* E = Bs + D * HP + 4;                        // [J][8] input jets
    float* Zs = E + J * SN_MAXK0;                      // [D][J][LD] stored pre-activations (t for s = 0)
    float* Hb = Zs + (int64_t)D * J * LD;              // [J][LD] act(Z) / reverse scratch
    float* ZB = Hb + J * LD;                           // [J][LD] adjoints of the current layer
    float* OB = ZB + J * LD;                           // [TR][S][4] output seeds
    __shared__ double lacc[NWARP][3];

    // ---- weights -> shared memory, zero-padded ----
    const LayerTab& t = a.tab;
    auto wlayer = [&](int l) { return l == 0 ? W0 : (l < D ? Wh + (int64_t)(l - 1) * HP * WS : Wo); };
    for (int l = 0; l <= D; ++l) {
        const int Kl = t.K[l], Nl = t.N[l];
        const int rows = l == 0 ? SN_MAXK0 : HP, cols = l == D ? 4 : HP, ld = l == D ? 4 : WS;
        float* dst = wlayer(l);
        // four independent global loads in flight per thread before the stores
        for (int i0 = tid; i0 < rows * cols; i0 += 4 * NT) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * NT, k = i / cols, n = i % cols;
                v[u] = (i < rows * cols && k < Kl && n < Nl) ? __ldg(a.params + t.offW[l] + (int64_t)k * Nl + n) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * NT;
                if (i < rows * cols) dst[(i / cols) * ld + i % cols] = v[u];
            }
        }
        const int bn = l == D ? 4 : HP;
        for (int n = tid; n < bn; n += NT) Bs[l * HP + n] = n < Nl ? a.params[t.offB[l] + n] : 0.0f;
    }
    if (tid < 3 * NWARP) lacc[tid / 3][tid % 3] = 0.0;
    double* slot = a.slot + (int64_t)blockIdx.x * a.P;
    const int ntiles = (int)((a.T + TR - 1) / TR);
    bool first = true;
    // slot[idx] (+)= v: a plain store on the CTA's first tile, then fire-and-forget
    // FP64 reductions (no load latency in the tile loop). Only this thread ever
    // updates slot[idx], so the updates apply in program (= tile) order.
    auto acc_slot = [&](int64_t idx, double v) {
        if (first) slot[idx] = v;
        else asm volatile("red.global.add.f64 [%0], %1;" ::"l"(slot + idx), "d"(v) : "memory");
    };
    __syncthreads();

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t g0 = (int64_t)tile * TR;
        // ---- input jets (FP64 embedding, stored as FP32) ----
        if (tid < TR) {
            const int64_t g = g0 + tid;
            double e[S][2 * kMaxAxes];
            if (g < a.T) embed_row<L>(a.ia, g, e);
#pragma unroll
            for (int s = 0; s < S; ++s)
                for (int k = 0; k < SN_MAXK0; ++k)
                    E[(s * TR + tid) * SN_MAXK0 + k] = (g < a.T && k < K0) ? (float)e[s][k] : 0.0f;
        }
        __syncthreads();

        // ---- forward: Z_l = A W_l (+b on the value stream), H = act(Z_l) ----
        for (int l = 0; l < D; ++l) {
            const float* A = l == 0 ? E : Hb;
            const int lda = l == 0 ? SN_MAXK0 : LD, Kd = l == 0 ? SN_MAXK0 : HP;
            const float* Wl = wlayer(l);
            if constexpr (MMA) {
                // warp = (row half h of every stream's 32 rows, 8-column tile nt): the S
                // m-tiles s*32 + 16h of one n-tile, so a thread holds every stream of its
                // four (row, column) outputs for the jet epilogue
                const int h = warp & 1, nt = warp >> 1, g = lane >> 2, tq = lane & 3;
                float acc[S][4];
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[s][i] = 0.0f;
#pragma unroll 2
                for (int k0 = 0; k0 < Kd; k0 += 8) {
                    uint32_t bh[2], bl[2];
                    sn::split_tf32(Wl[(k0 + tq) * WS + nt * 8 + g], bh[0], bl[0]);
                    sn::split_tf32(Wl[(k0 + tq + 4) * WS + nt * 8 + g], bh[1], bl[1]);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        uint32_t ah[4], al[4];
                        sn::frag_a(A + (s * TR + 16 * h + g) * lda + k0 + tq, lda, ah, al);
                        sn::mma3(acc[s], ah, al, bh, bl);
                    }
                }
                __syncthreads();  // every read of A (= Hb) done before it is overwritten
                float* Zl = Zs + (int64_t)l * J * LD;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = 16 * h + g + 8 * (i >> 1), n = nt * 8 + 2 * tq + (i & 1);
                    float zz[S], hh[S];
                    zz[0] = store_value<ACT_TANH>(acc[0][i] + Bs[l * HP + n]);
#pragma unroll
                    for (int s = 1; s < S; ++s) zz[s] = acc[s][i];
                    act_fwd<L, ACT_TANH>(zz, hh, 1.0f);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        Zl[(s * TR + r) * LD + n] = zz[s];
                        Hb[(s * TR + r) * LD + n] = hh[s];
                    }
                }
                __syncthreads();
                continue;
            }
            const int n0 = warp * NC;
            float z[S][NC];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < NC; ++c) z[s][c] = 0.0f;
#pragma unroll 2
            for (int k = 0; k < Kd; k += 4) {
                float4 av[S];
#pragma unroll
                for (int s = 0; s < S; ++s) av[s] = *reinterpret_cast<const float4*>(A + (s * TR + lane) * lda + k);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    float w[NC];
                    if constexpr (NC == 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(Wl + (k + kk) * WS + n0);
                        w[0] = w4.x;
                        w[1] = w4.y;
                        w[2] = w4.z;
                        w[3] = w4.w;
                    } else {
#pragma unroll
                        for (int c = 0; c < NC; ++c) w[c] = Wl[(k + kk) * WS + n0 + c];
                    }
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const float x = kk == 0 ? av[s].x : (kk == 1 ? av[s].y : (kk == 2 ? av[s].z : av[s].w));
#pragma unroll
                        for (int c = 0; c < NC; ++c) z[s][c] = fmaf(x, w[c], z[s][c]);
                    }
                }
            }
            __syncthreads();  // every read of A (= Hb) done before it is overwritten
            float* Zl = Zs + (int64_t)l * J * LD;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int n = n0 + c;
                float zz[S], hh[S];
                zz[0] = store_value<ACT_TANH>(z[0][c] + Bs[l * HP + n]);
#pragma unroll
                for (int s = 1; s < S; ++s) zz[s] = z[s][c];
                act_fwd<L, ACT_TANH>(zz, hh, 1.0f);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    Zl[(s * TR + lane) * LD + n] = zz[s];
                    Hb[(s * TR + lane) * LD + n] = hh[s];
                }
            }
            __syncthreads();
        }

        // ---- head: outputs, residual / IC / BC losses and seeds (two rows per warp) ----
        for (int rr = warp; rr < TR; rr += NWARP) {
            float o[S * F];
#pragma unroll
            for (int i = 0; i < S * F; ++i) o[i] = 0.0f;
            for (int k = lane; k < HP; k += 32)
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const float h = Hb[(s * TR + rr) * LD + k];
#pragma unroll
                    for (int f = 0; f < F; ++f) o[s * F + f] = fmaf(h, Wo[k * 4 + f], o[s * F + f]);
                }
#pragma unroll
            for (int i = 0; i < S * F; ++i) {
                float v = o[i];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                o[i] = v;
            }
#pragma unroll
            for (int f = 0; f < F; ++f) o[f] += Bs[D * HP + f];
            float ob[S * F];
#pragma unroll
            for (int i = 0; i < S * F; ++i) ob[i] = 0.0f;
            const int64_t g = g0 + rr;
            if (g < a.T) {
                if (g >= a.int0 && g < a.int1) {
                    float res[K], rb[K];
                    residual<P>(o, res, a.pc);
                    float sq = 0.0f;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        sq += res[k] * res[k];
                        rb[k] = a.w_pde * res[k];
                        if (lane == 0 && !isfinite(res[k])) atomicMin(&a.bad[k], (int)(g - a.int0));
                    }
                    if (a.resid_out && lane == 0) {
                        const int64_t n_int = a.int1 - a.int0;
#pragma unroll
                        for (int k = 0; k < K; ++k) a.resid_out[k * n_int + (g - a.int0)] = res[k];
                    }
                    if (lane == 0) lacc[warp][0] += (double)sq;
                    residual_seed<P>(o, rb, ob, a.pc);
                } else if (g >= a.ic0 && g < a.ic1) {
                    const int64_t i = g - a.ic0, n = a.ic1 - a.ic0;
                    float sq = 0.0f;
#pragma unroll
                    for (int f = 0; f < F; ++f) {
                        const float d = o[f] - a.ic_t[f * n + i];
                        sq += d * d;
                        ob[f] = a.w_ic * d;
                    }
                    if (lane == 0) lacc[warp][1] += (double)sq;
                } else if (a.bc_mode == 2 && g >= a.bca0 && g < a.bca1) {
                    const int64_t i = g - a.bca0, n = a.bca1 - a.bca0;
                    float sq = 0.0f;
#pragma unroll
                    for (int f = 0; f < F; ++f) {
                        const float d = o[f] - a.bc_t[f * n + i];
                        sq += d * d;
                        ob[f] = a.w_bc * d;
                    }
                    if (lane == 0) lacc[warp][2] += (double)sq;
                }
            }
            if (lane < S * 4) {
                const int s = lane / 4, f = lane % 4;
                OB[(rr * S + s) * 4 + f] = f < F ? ob[s * F + f] : 0.0f;
            }
        }
        __syncthreads();

        // head reverse: dW_D += H^T Obar, db_D += Obar[0]; ZB = act^T(Obar W_D^T ; Z_{D-1})
        if (tid < HP * F) {
            const int k = tid / F, f = tid % F;
            float v = 0.0f;
            for (int s = 0; s < S; ++s)
                for (int r = 0; r < TR; ++r) v = fmaf(Hb[(s * TR + r) * LD + k], OB[(r * S + s) * 4 + f], v);
            if (k < H) acc_slot(t.offW[D] + (int64_t)k * F + f, v);
        } else if (tid >= NT - F) {
            const int f = tid - (NT - F);
            double v = 0.0;
            for (int r = 0; r < TR; ++r) v += (double)OB[(r * S) * 4 + f];
            acc_slot(t.offB[D] + f, v);
        }
        {
            const float* Zl = Zs + (int64_t)(D - 1) * J * LD;
            for (int e = tid; e < TR * HP; e += NT) {
                const int r = e / HP, k = e % HP;
                float zz[S], hb[S], zb[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    zz[s] = Zl[(s * TR + r) * LD + k];
                    float v = 0.0f;
#pragma unroll
                    for (int f = 0; f < F; ++f) v = fmaf(OB[(r * S + s) * 4 + f], Wo[k * 4 + f], v);
                    hb[s] = v;
                }
                act_bwd<L, ACT_TANH>(zz, hb, zb, 1.0f);
#pragma unroll
                for (int s = 0; s < S; ++s) ZB[(s * TR + r) * LD + k] = zb[s];
            }
        }
        __syncthreads();

        // ---- reverse through the hidden layers ----
        for (int l = D - 1; l >= 0; --l) {
            const float* A = l == 0 ? E : Hb;
            const int lda = l == 0 ? SN_MAXK0 : LD;
            if (l > 0) {  // Hb = act(Z_{l-1}) (the layer's input activations)
                const float* Zp = Zs + (int64_t)(l - 1) * J * LD;
                for (int e = tid; e < TR * HP; e += NT) {
                    const int r = e / HP, k = e % HP;
                    float zz[S], hh[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) zz[s] = Zp[(s * TR + r) * LD + k];
                    act_fwd<L, ACT_TANH>(zz, hh, 1.0f);
#pragma unroll
                    for (int s = 0; s < S; ++s) Hb[(s * TR + r) * LD + k] = hh[s];
                }
                __syncthreads();
            }
            // dW_l += A^T ZB (this thread's BK x BN block), db_l += colsum ZB[value stream]
            const int Kl = l == 0 ? K0 : H;
            if (MMA && l > 0) {
                // dW[k][n] = sum_j Hb[j][k] ZB[j][n]: warp = (16-feature m-tile, two
                // 8-column n-tiles), the reduction runs over every row of every stream
                const int mt = warp & 3, ntp = (warp >> 2) * 2, g = lane >> 2, tq = lane & 3;
                float acc[2][4];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[u][i] = 0.0f;
#pragma unroll 2
                for (int j0 = 0; j0 < J; j0 += 8) {
                    uint32_t ah[4], al[4];
                    const float* Ar = A + (j0 + tq) * lda + mt * 16 + g;
                    sn::split_tf32(Ar[0], ah[0], al[0]);          // (m = g,     k = tq)
                    sn::split_tf32(Ar[8], ah[1], al[1]);          // (m = g + 8, k = tq)
                    sn::split_tf32(Ar[4 * lda], ah[2], al[2]);    // (m = g,     k = tq + 4)
                    sn::split_tf32(Ar[4 * lda + 8], ah[3], al[3]);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        uint32_t bh[2], bl[2];
                        const float* Br = ZB + (j0 + tq) * LD + (ntp + u) * 8 + g;
                        sn::split_tf32(Br[0], bh[0], bl[0]);
                        sn::split_tf32(Br[4 * LD], bh[1], bl[1]);
                        sn::mma3(acc[u], ah, al, bh, bl);
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int k = mt * 16 + g + 8 * (i >> 1), n = (ntp + u) * 8 + 2 * tq + (i & 1);
                        if (k < Kl && n < H) acc_slot(t.offW[l] + (int64_t)k * H + n, acc[u][i]);
                    }
            } else if (l > 0) {
                const int kb = (tid / (HP / BN)) * BK, nb = (tid % (HP / BN)) * BN;
                float acc[BK][BN];
#pragma unroll
                for (int i = 0; i < BK; ++i)
#pragma unroll
                    for (int j = 0; j < BN; ++j) acc[i][j] = 0.0f;
#pragma unroll 4
                for (int jj = 0; jj < J; ++jj) {
                    float av[BK], bv[BN];
                    if constexpr (BK == 1 && BN == 4) {  // LDS.32 + LDS.128
                        const float4 b4 = *reinterpret_cast<const float4*>(ZB + jj * LD + nb);
                        av[0] = A[jj * lda + kb];
                        bv[0] = b4.x;
                        bv[1] = b4.y;
                        bv[2] = b4.z;
                        bv[3] = b4.w;
                    } else if constexpr (BK == 2 && BN == 4) {  // LDS.64 + LDS.128 (16 B-aligned rows)
                        const float2 a2 = *reinterpret_cast<const float2*>(A + jj * lda + kb);
                        const float4 b4 = *reinterpret_cast<const float4*>(ZB + jj * LD + nb);
                        av[0] = a2.x;
                        av[1] = a2.y;
                        bv[0] = b4.x;
                        bv[1] = b4.y;
                        bv[2] = b4.z;
                        bv[3] = b4.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < BK; ++i) av[i] = A[jj * lda + kb + i];
#pragma unroll
                        for (int j = 0; j < BN; ++j) bv[j] = ZB[jj * LD + nb + j];
                    }
#pragma unroll
                    for (int i = 0; i < BK; ++i)
#pragma unroll
                        for (int j = 0; j < BN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                }
#pragma unroll
                for (int i = 0; i < BK; ++i)
#pragma unroll
                    for (int j = 0; j < BN; ++j)
                        if (kb + i < Kl && nb + j < H) acc_slot(t.offW[l] + (int64_t)(kb + i) * H + nb + j, acc[i][j]);
            } else {
                for (int e = tid; e < K0 * HP; e += NT) {
                    const int k = e / HP, n = e % HP;
                    float v = 0.0f;
                    for (int jj = 0; jj < J; ++jj) v = fmaf(A[jj * lda + k], ZB[jj * LD + n], v);
                    if (n < H) acc_slot(t.offW[0] + (int64_t)k * H + n, v);
                }
            }
            if (tid < 4 * HP) {  // db: four lanes per column (rows q, q + 4, ...), fixed shuffle tree
                const int col = tid >> 2, q = tid & 3;
                double v = 0.0;
#pragma unroll
                for (int r = q; r < TR; r += 4) v += (double)ZB[r * LD + col];
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (q == 0 && col < H) acc_slot(t.offB[l] + col, v);
            }
            if (l == 0) break;
            // Hbar = ZB W_l^T (registers), then ZB = act^T(Hbar ; Z_{l-1}) in place
            const float* Wl = wlayer(l);
            if constexpr (MMA) {
                // warp = (row half h, 8-feature tile kt) over every stream, as the forward
                const int h = warp & 1, kt = warp >> 1, g = lane >> 2, tq = lane & 3;
                float hbm[S][4];
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int i = 0; i < 4; ++i) hbm[s][i] = 0.0f;
#pragma unroll 2
                for (int n0 = 0; n0 < HP; n0 += 8) {
                    uint32_t bh[2], bl[2];  // B[n][k] = W[k][n]: (k-row n0 + tq (+4), column kt*8 + g)
                    sn::split_tf32(Wl[(kt * 8 + g) * WS + n0 + tq], bh[0], bl[0]);
                    sn::split_tf32(Wl[(kt * 8 + g) * WS + n0 + tq + 4], bh[1], bl[1]);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        uint32_t ah[4], al[4];
                        sn::frag_a(ZB + (s * TR + 16 * h + g) * LD + n0 + tq, LD, ah, al);
                        sn::mma3(hbm[s], ah, al, bh, bl);
                    }
                }
                __syncthreads();  // all reads of ZB (and of Hb by the dW loop) done
                const float* Zp = Zs + (int64_t)(l - 1) * J * LD;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = 16 * h + g + 8 * (i >> 1), k = kt * 8 + 2 * tq + (i & 1);
                    float zz[S], hh[S], zb[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        zz[s] = Zp[(s * TR + r) * LD + k];
                        hh[s] = hbm[s][i];
                    }
                    act_bwd<L, ACT_TANH>(zz, hh, zb, 1.0f);
#pragma unroll
                    for (int s = 0; s < S; ++s) ZB[(s * TR + r) * LD + k] = zb[s];
                }
                __syncthreads();
                continue;
            }
            const int k0 = warp * NC;
            float hb[S][NC];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < NC; ++c) hb[s][c] = 0.0f;
#pragma unroll 2
            for (int n = 0; n < HP; n += 4) {
                float4 zv[S];
#pragma unroll
                for (int s = 0; s < S; ++s) zv[s] = *reinterpret_cast<const float4*>(ZB + (s * TR + lane) * LD + n);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const float4 w = *reinterpret_cast<const float4*>(Wl + (k0 + c) * WS + n);
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        hb[s][c] = fmaf(zv[s].x, w.x, fmaf(zv[s].y, w.y, fmaf(zv[s].z, w.z, fmaf(zv[s].w, w.w, hb[s][c]))));
                }
            }
            __syncthreads();  // all reads of ZB (and of Hb by the dW loop) done
            const float* Zp = Zs + (int64_t)(l - 1) * J * LD;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int k = k0 + c;
                float zz[S], hh[S], zb[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    zz[s] = Zp[(s * TR + lane) * LD + k];
                    hh[s] = hb[s][c];
                }
                act_bwd<L, ACT_TANH>(zz, hh, zb, 1.0f);
#pragma unroll
                for (int s = 0; s < S; ++s) ZB[(s * TR + lane) * LD + k] = zb[s];
            }
            __syncthreads();
        }
        first = false;
        __syncthreads();
    }
    __syncthreads();
    if (tid < 3) {  // fixed-order fold of the warps' loss sums
        double v = 0.0;
        for (int w = 0; w < NWARP; ++w) v += lacc[w][tid];
        a.loss_part[blockIdx.x * 3 + tid] = v;
    }
}

// flat gradient = sum of the CTA slots (fixed order, FP64); losses * 1/n per term
static __global__ void k_small_finalize(const double* __restrict__ slot, int nblk, int64_t P,
                                        const double* __restrict__ loss_part, const double* __restrict__ inv_n,
                                        float* __restrict__ grad, double* __restrict__ losses) {
    // one thread per entry (coalesced across the warp), four interleaved partial
    // sums over the slots (loads in flight), combined in fixed order
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int b = 0;
        for (; b + 4 <= nblk; b += 4) {
            s0 += slot[(int64_t)b * P + i];
            s1 += slot[(int64_t)(b + 1) * P + i];
            s2 += slot[(int64_t)(b + 2) * P + i];
            s3 += slot[(int64_t)(b + 3) * P + i];
        }
        for (; b < nblk; ++b) s0 += slot[(int64_t)b * P + i];
        grad[i] = (float)((s0 + s1) + (s2 + s3));
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += loss_part[b * 3 + threadIdx.x];
        losses[threadIdx.x] = s * inv_n[threadIdx.x];
    }
}

}  // namespace pnx
