// kernels_simt.cuh -- FP32 CUDA-core (FFMA) kernels of the jet train step.
//
// Data layout in HBM (per chunk of Rpad rows, Rpad a multiple of 64):
//   Hin  [S][Rpad][K0]   input-feature jets after embedding / RFF
//   Z_l  [S][Rpad][H]    pre-activation jets of hidden layer l
//   Zb   [S][Rpad][H]    adjoints of a hidden layer's pre-activation jets
// Stream-major, feature-contiguous: every GEMM operand is a plain row-major
// [rows x features] matrix per stream, and all S streams of one
// (point, feature) element meet in one thread for the jet epilogues.
//
// Reverse mode of the jet program (see oracle/pinn_oracle.py):
//   forward   Z_l[s] = act(Z_{l-1})[s] W_l + [s==0] b_l         (model.cpp:163-175)
//   head      O = act(Z_{L-2}) W_L + b_L, residual, seeds Obar     (losses.cpp:26-95)
//   reverse   Zb_{l-1} = act^T(Zb_l W_l^T ; Z_{l-1})              (graph.cpp:468-502)
//             dW_l = sum_s act(Z_{l-1})[s]^T Zb_l[s],  db_l = colsum Zb_l[0]
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "jets.cuh"
#include "residuals.cuh"

namespace pnx {

constexpr int kMaxLayers = 16;
constexpr int kMaxAxes = 4;

// ---------------------------------------------------------------------------
// parameter preparation: W = V*exp(s) (model.cpp:117-126), W^T, bias
// ---------------------------------------------------------------------------
struct LayerTab {
    int n;                       // number of linear layers (depth + 1)
    int K[kMaxLayers], N[kMaxLayers];
    int64_t offW[kMaxLayers];    // flat offset of W or V
    int64_t offS[kMaxLayers];    // flat offset of s (RWF) or -1
    int64_t offB[kMaxLayers];    // flat offset of b
    int64_t dW[kMaxLayers];      // offset into the materialised weight arena
    int64_t dB[kMaxLayers];      // offset into the bias arena
};

// wamax (optional): per layer, max |W| as float bits (3xFP16 weight-image scale)
static __global__ void k_prep(const float* __restrict__ params, LayerTab t, float* __restrict__ W,
                       float* __restrict__ Wt, float* __restrict__ bias, unsigned* __restrict__ wamax = nullptr) {
    const int l = blockIdx.y;
    if (l >= t.n) return;
    const int K = t.K[l], N = t.N[l];
    const int64_t total = (int64_t)K * N;
    unsigned mx = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total + N;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < total) {
            const int k = (int)(i / N), n = (int)(i % N);
            float w = params[t.offW[l] + i];
            if (t.offS[l] >= 0) w = w * expf(params[t.offS[l] + n]);
            W[t.dW[l] + i] = w;
            Wt[t.dW[l] + (int64_t)n * K + k] = w;
            mx = max(mx, __float_as_uint(fabsf(w)));
        } else {
            const int n = (int)(i - total);
            bias[t.dB[l] + n] = params[t.offB[l] + n];
        }
    }
    if (wamax) {
        mx = __reduce_max_sync(0xffffffffu, mx);
        if ((threadIdx.x & 31) == 0) atomicMax(wamax + l, mx);
    }
}

// ---------------------------------------------------------------------------
// input features: coordinate embedding (model.cpp:134-154) + RFF (:157-161),
// evaluated in float64 from float64 coordinates, stored as float32 jets.
// ---------------------------------------------------------------------------
struct InputArgs {
    const double* coords;   // [d][ld] float64, global rows
    int64_t ld;             // leading dimension of coords
    int64_t row0;           // first global row of this chunk
    int nrows, Rpad;
    int in_dim;
    int periodic[kMaxAxes];
    double period[kMaxAxes];
    int64_t period_off[kMaxAxes];  // flat param offset of a trainable period, else -1
    const float* params;
    int E;                  // embedded width
    int rff_w;              // 0 = off
    const double* rffB;     // [E][rff_w]
    int K0;                 // feature width written (E or 2*rff_w)
    float* Hin;             // [S][Rpad][K0]
    unsigned* amax_out;     // k_input: per-stream max |Hin| (float bits, atomicMax), or null
};

// embedding jets e[s][c] (c < E) for one row, float64
template <int L>
__device__ __forceinline__ void embed_row(const InputArgs& a, int64_t g, double (*e)[2 * kMaxAxes]) {
    using St = Streams<L>;
    constexpr int S = St::S;
    int c = 0;
    for (int ax = 0; ax < a.in_dim; ++ax) {
        const double x = a.coords[(int64_t)ax * a.ld + g];
        if (!a.periodic[ax]) {
#pragma unroll
            for (int s = 0; s < S; ++s)
                e[s][c] = (s == 0) ? x : ((St::order(s) == 1 && St::axis(s) == ax) ? 1.0 : 0.0);
            c += 1;
            continue;
        }
        double kappa, phi;
        if (a.period_off[ax] >= 0) {  // phase = affine(scale(x, P^-1), 2pi) (model.cpp:144-147)
            const double P = (double)a.params[a.period_off[ax]];
            kappa = 2.0 * CUDART_PI * (1.0 / P);
            phi = 2.0 * CUDART_PI * (x * (1.0 / P));
        } else {  // affine(x, 2pi/P) (model.cpp:149)
            kappa = 2.0 * CUDART_PI / a.period[ax];
            phi = x * kappa;
        }
        double sp, cp;
        sincos(phi, &sp, &cp);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            double C = 0.0, Sn = 0.0;
            if (s == 0) {
                C = cp;
                Sn = sp;
            } else if (St::axis(s) == ax) {
                if (St::order(s) == 1) {
                    C = -sp * kappa;
                    Sn = cp * kappa;
                } else {
                    C = -cp * kappa * kappa;
                    Sn = -sp * kappa * kappa;
                }
            }
            e[s][c] = C;
            e[s][c + 1] = Sn;
        }
        c += 2;
    }
}

// m[s] = sum_k e[s][k] B[k][col] for one row without materialising e (a local
// array indexed by the runtime embedding layout lived in local memory): the
// same terms in the same order as embed_row followed by the dot product
template <int L>
__device__ __forceinline__ void embed_dot(const InputArgs& a, int64_t g, int col, double (&m)[Streams<L>::S]) {
    using St = Streams<L>;
    constexpr int S = St::S;
#pragma unroll
    for (int s = 0; s < S; ++s) m[s] = 0.0;
    int k = 0;
#pragma unroll
    for (int ax = 0; ax < kMaxAxes; ++ax) {
        if (ax >= a.in_dim) break;
        const double x = a.coords[(int64_t)ax * a.ld + g];
        if (!a.periodic[ax]) {
            const double b = a.rffB[(int64_t)k * a.rff_w + col];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const double e = (s == 0) ? x : ((St::order(s) == 1 && St::axis(s) == ax) ? 1.0 : 0.0);
                m[s] += e * b;
            }
            k += 1;
            continue;
        }
        double kappa, phi;
        if (a.period_off[ax] >= 0) {  // as embed_row (model.cpp:144-149)
            const double P = (double)a.params[a.period_off[ax]];
            kappa = 2.0 * CUDART_PI * (1.0 / P);
            phi = 2.0 * CUDART_PI * (x * (1.0 / P));
        } else {
            kappa = 2.0 * CUDART_PI / a.period[ax];
            phi = x * kappa;
        }
        double sp, cp;
        sincos(phi, &sp, &cp);
        const double b0 = a.rffB[(int64_t)k * a.rff_w + col], b1 = a.rffB[(int64_t)(k + 1) * a.rff_w + col];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            double C = 0.0, Sn = 0.0;
            if (s == 0) {
                C = cp;
                Sn = sp;
            } else if (St::axis(s) == ax) {
                if (St::order(s) == 1) {
                    C = -sp * kappa;
                    Sn = cp * kappa;
                } else {
                    C = -cp * kappa * kappa;
                    Sn = -sp * kappa * kappa;
                }
            }
            m[s] += C * b0;
            m[s] += Sn * b1;
        }
        k += 2;
    }
}

template <int L>
static __global__ void k_input(InputArgs a) {
    using St = Streams<L>;
    constexpr int S = St::S;
    // per-stream bounds of the written features (3xFP16 operand scales of layer 0)
    float mx[S];
#pragma unroll
    for (int s = 0; s < S; ++s) mx[s] = 0.0f;
    const int per_row = a.rff_w > 0 ? a.rff_w : 1;
    const int64_t total = (int64_t)a.Rpad * per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / per_row), c = (int)(i % per_row);
        const int64_t RK = (int64_t)a.Rpad * a.K0;
        float* out = a.Hin + (int64_t)r * a.K0;
        if (r >= a.nrows) {  // zero padding rows so they stay finite downstream
            if (a.rff_w > 0) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    out[s * RK + c] = 0.0f;
                    out[s * RK + a.rff_w + c] = 0.0f;
                }
            } else {
                for (int s = 0; s < S; ++s)
                    for (int k = 0; k < a.K0; ++k) out[s * RK + k] = 0.0f;
            }
            continue;
        }
        if (a.rff_w == 0) {
            double e[S][2 * kMaxAxes];
            embed_row<L>(a, a.row0 + r, e);
#pragma unroll
            for (int s = 0; s < S; ++s)
                for (int k = 0; k < a.E; ++k) {
                    out[s * RK + k] = (float)e[s][k];
                    mx[s] = fmaxf(mx[s], fabsf((float)e[s][k]));
                }
            continue;
        }
        // m = e B  (B frozen, float64), then [cos m, sin m] jets
        double m[S];
        embed_dot<L>(a, a.row0 + r, c, m);
        double sm, cm;
        sincos(m[0], &sm, &cm);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            double C, Sn;
            if (s == 0) {
                C = cm;
                Sn = sm;
            } else if (St::order(s) == 1) {
                C = -sm * m[s];
                Sn = cm * m[s];
            } else {
                const double ma = m[St::partner(s)];
                C = -sm * m[s] - cm * ma * ma;
                Sn = cm * m[s] - sm * ma * ma;
            }
            out[s * RK + c] = (float)C;
            out[s * RK + a.rff_w + c] = (float)Sn;
            mx[s] = fmaxf(mx[s], fmaxf(fabsf((float)C), fabsf((float)Sn)));
        }
    }
    if (a.amax_out) {  // warp, then block maxima: one atomic per block and stream
        __shared__ unsigned bm[32][S];
        const int w = threadIdx.x >> 5;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const unsigned v = __reduce_max_sync(0xffffffffu, __float_as_uint(mx[s]));
            if ((threadIdx.x & 31) == 0) bm[w][s] = v;
        }
        __syncthreads();
        if (threadIdx.x < S) {
            unsigned v = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) v = max(v, bm[k][threadIdx.x]);
            atomicMax(a.amax_out + threadIdx.x, v);
        }
    }
}

// Layer 0 for narrow embeddings (no RFF, K0 <= 8) fused with the input jets:
// Z0[s] = e[s] W0 + [s==0] b0 with e recomputed in float64 per row; no Hin in HBM.
constexpr int L0_ROWS = 32;

template <int L, int ACT>
__global__ void __launch_bounds__(256) k_layer0_fwd(InputArgs a, const float* __restrict__ W0,
                                                   const float* __restrict__ b0, float* __restrict__ Z0, int H,
                                                   unsigned* __restrict__ amax = nullptr) {
    using St = Streams<L>;
    constexpr int S = St::S;
    __shared__ float E[L0_ROWS][S][2 * kMaxAxes];
    __shared__ float Ws[2 * kMaxAxes * 512];
    const int K0 = a.E;
    for (int i = threadIdx.x; i < K0 * H; i += blockDim.x) Ws[i] = W0[i];
    const int64_t RH = (int64_t)a.Rpad * H;
    unsigned mx[S];  // |z| bound per stream (3xFP16 operand scales of the next layer)
#pragma unroll
    for (int s = 0; s < S; ++s) mx[s] = 0;
    for (int rb = blockIdx.x * L0_ROWS; rb < a.Rpad; rb += gridDim.x * L0_ROWS) {
        __syncthreads();
        if (threadIdx.x < L0_ROWS) {
            const int r = rb + threadIdx.x;
            if (r < a.nrows) {
                double e[S][2 * kMaxAxes];
                embed_row<L>(a, a.row0 + r, e);
                for (int s = 0; s < S; ++s)
                    for (int k = 0; k < K0; ++k) E[threadIdx.x][s][k] = (float)e[s][k];
            } else {
                for (int s = 0; s < S; ++s)
                    for (int k = 0; k < K0; ++k) E[threadIdx.x][s][k] = 0.0f;
            }
        }
        __syncthreads();
        const int nch = H / 4;
        for (int item = threadIdx.x; item < L0_ROWS * nch; item += blockDim.x) {
            const int rr = item / nch, n = (item % nch) * 4;
            float z[S][4];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int j = 0; j < 4; ++j) z[s][j] = 0.0f;
            for (int k = 0; k < K0; ++k) {
                const float4 w = *reinterpret_cast<const float4*>(&Ws[k * H + n]);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const float e = E[rr][s][k];
                    z[s][0] = fmaf(e, w.x, z[s][0]);
                    z[s][1] = fmaf(e, w.y, z[s][1]);
                    z[s][2] = fmaf(e, w.z, z[s][2]);
                    z[s][3] = fmaf(e, w.w, z[s][3]);
                }
            }
            const float4 bb = *reinterpret_cast<const float4*>(b0 + n);
            z[0][0] = store_value<ACT>(z[0][0] + bb.x);
            z[0][1] = store_value<ACT>(z[0][1] + bb.y);
            z[0][2] = store_value<ACT>(z[0][2] + bb.z);
            z[0][3] = store_value<ACT>(z[0][3] + bb.w);
            float* dst = Z0 + (int64_t)(rb + rr) * H + n;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                *reinterpret_cast<float4*>(dst + s * RH) = make_float4(z[s][0], z[s][1], z[s][2], z[s][3]);
#pragma unroll
                for (int j = 0; j < 4; ++j) mx[s] = max(mx[s], __float_as_uint(fabsf(z[s][j])));
            }
        }
    }
    if (amax) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const unsigned v = __reduce_max_sync(0xffffffffu, mx[s]);
            if ((threadIdx.x & 31) == 0) atomicMax(amax + s, v);
        }
    }
}

// Layer-0 weight gradient for narrow embeddings: part[blk][k*H + n] +=
// sum_rows sum_s e[s][row][k] Zb0[s][row][n], part[blk][K0*H + n] += sum_rows Zb0[0][row][n].
// Streams Zb0 once (coalesced), recomputes e; FP32 per 32-row tile, FP64 across tiles.
template <int L>
__global__ void __launch_bounds__(256) k_layer0_wgrad(InputArgs a, const float* __restrict__ Zb0, int H,
                                                     double* __restrict__ part) {
    using St = Streams<L>;
    constexpr int S = St::S;
    constexpr int KM = 2 * kMaxAxes;
    __shared__ float E[L0_ROWS][S][KM];
    __shared__ double red[KM + 1][512];
    const int K0 = a.E;
    const int nch = H / 4;           // <= 128 chunks (H <= 512)
    const int lanes = 256 / nch;     // row lanes per block (H=256: 4)
    const int rl = threadIdx.x / nch, c = threadIdx.x % nch, n = c * 4;
    const bool active = rl < lanes && c < nch;
    double acc[KM + 1][4];
#pragma unroll
    for (int k = 0; k <= KM; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[k][j] = 0.0;
    const int64_t RH = (int64_t)a.Rpad * H;
    for (int rb = blockIdx.x * L0_ROWS; rb < a.nrows; rb += gridDim.x * L0_ROWS) {
        __syncthreads();
        if (threadIdx.x < L0_ROWS) {
            const int r = rb + threadIdx.x;
            double e[S][2 * kMaxAxes];
            if (r < a.nrows) embed_row<L>(a, a.row0 + r, e);
            for (int s = 0; s < S; ++s)
                for (int k = 0; k < K0; ++k) E[threadIdx.x][s][k] = r < a.nrows ? (float)e[s][k] : 0.0f;
        }
        __syncthreads();
        if (!active) continue;
        float t32[KM + 1][4];
#pragma unroll
        for (int k = 0; k <= KM; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) t32[k][j] = 0.0f;
        for (int rr = rl; rr < L0_ROWS; rr += lanes) {
            const int r = rb + rr;
            if (r >= a.nrows) break;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float4 z = *reinterpret_cast<const float4*>(Zb0 + s * RH + (int64_t)r * H + n);
                if (s == 0) {
                    t32[KM][0] += z.x; t32[KM][1] += z.y; t32[KM][2] += z.z; t32[KM][3] += z.w;
                }
#pragma unroll
                for (int k = 0; k < KM; ++k) {
                    if (k >= K0) break;
                    const float e = E[rr][s][k];
                    t32[k][0] = fmaf(e, z.x, t32[k][0]);
                    t32[k][1] = fmaf(e, z.y, t32[k][1]);
                    t32[k][2] = fmaf(e, z.z, t32[k][2]);
                    t32[k][3] = fmaf(e, z.w, t32[k][3]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k <= KM; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[k][j] += (double)t32[k][j];
    }
    // fixed-order reduction over the row lanes (lane 0 first), then one partial per block
    for (int l2 = 0; l2 < lanes; ++l2) {
        __syncthreads();
        if (active && rl == l2)
            for (int k = 0; k <= KM; ++k)
                for (int j = 0; j < 4; ++j) red[k][c * 4 + j] = (l2 == 0 ? 0.0 : red[k][c * 4 + j]) + acc[k][j];
    }
    __syncthreads();
    double* dst = part + (int64_t)blockIdx.x * ((int64_t)K0 * H + H);
    for (int i = threadIdx.x; i < (K0 + 1) * H; i += blockDim.x) {
        const int k = i / H, nn = i % H;
        dst[(int64_t)k * H + nn] += red[k < K0 ? k : KM][nn];
    }
}

// Layer-0 weight gradient, streaming version (H = 32*NC):
//   dW0[k][n] = sum_rows sum_s E[s][row][k] Zb0[s][row][n],  db0[n] = sum_rows Zb0[0][row][n]
// Each warp owns a contiguous row chunk; lane owns NC consecutive columns, so a
// row of a stream is one fully coalesced warp load. The FP64 input-feature jets
// of 32 rows are computed once (lane = row) and broadcast by shuffles. FP32
// accumulation per warp chunk, then the block folds its 8 warps into FP64 in
// fixed order and adds one partial slice (same layout as k_layer0_wgrad).
template <int L, int K0C, int NC>
__global__ void __launch_bounds__(256) k_layer0_wgrad_stream(InputArgs a, const float* __restrict__ Zb0, int H,
                                                            int rows_per_warp, double* __restrict__ part) {
    using St = Streams<L>;
    constexpr int S = St::S;
    __shared__ double red[(K0C + 1) * 32 * NC];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * 8 + wid;
    const int rbeg = gw * rows_per_warp, rend = min(a.nrows, rbeg + rows_per_warp);
    const int K0 = a.E;
    const int64_t RH = (int64_t)a.Rpad * H;
    float acc[K0C + 1][NC];
#pragma unroll
    for (int k = 0; k <= K0C; ++k)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[k][c] = 0.0f;
    for (int g0 = rbeg; g0 < rend; g0 += 32) {
        float e[S][K0C];
        {
            double ed[S][2 * kMaxAxes];
            const int r = g0 + lane;
            if (r < rend) embed_row<L>(a, a.row0 + r, ed);
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int k = 0; k < K0C; ++k) e[s][k] = (r < rend && k < K0) ? (float)ed[s][k] : 0.0f;
        }
        const int nr = min(32, rend - g0);
#pragma unroll 2
        for (int rr = 0; rr < nr; ++rr) {
            const float* zp = Zb0 + (int64_t)(g0 + rr) * H + lane * NC;
            float4 z[S][NC / 4];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c4 = 0; c4 < NC / 4; ++c4) z[s][c4] = __ldg(reinterpret_cast<const float4*>(zp + s * RH) + c4);
#pragma unroll
            for (int s = 0; s < S; ++s) {
#pragma unroll
                for (int k = 0; k < K0C; ++k) {
                    const float ek = __shfl_sync(0xffffffffu, e[s][k], rr);
#pragma unroll
                    for (int c4 = 0; c4 < NC / 4; ++c4) {
                        acc[k][4 * c4 + 0] = fmaf(ek, z[s][c4].x, acc[k][4 * c4 + 0]);
                        acc[k][4 * c4 + 1] = fmaf(ek, z[s][c4].y, acc[k][4 * c4 + 1]);
                        acc[k][4 * c4 + 2] = fmaf(ek, z[s][c4].z, acc[k][4 * c4 + 2]);
                        acc[k][4 * c4 + 3] = fmaf(ek, z[s][c4].w, acc[k][4 * c4 + 3]);
                    }
                }
                if (s == 0)
#pragma unroll
                    for (int c4 = 0; c4 < NC / 4; ++c4) {
                        acc[K0C][4 * c4 + 0] += z[0][c4].x;
                        acc[K0C][4 * c4 + 1] += z[0][c4].y;
                        acc[K0C][4 * c4 + 2] += z[0][c4].z;
                        acc[K0C][4 * c4 + 3] += z[0][c4].w;
                    }
            }
        }
    }
    // fold the block's warps in fixed order (warp 0 first) into FP64
    for (int w = 0; w < 8; ++w) {
        __syncthreads();
        if (wid == w)
#pragma unroll
            for (int k = 0; k <= K0C; ++k)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    double& d = red[k * 32 * NC + lane * NC + c];
                    d = (w == 0 ? 0.0 : d) + (double)acc[k][c];
                }
    }
    __syncthreads();
    double* dst = part + (int64_t)blockIdx.x * ((int64_t)K0 * H + H);
    for (int i = threadIdx.x; i < (K0 + 1) * H; i += blockDim.x) {
        const int k = i / H, nn = i % H;
        dst[(int64_t)k * H + nn] += red[(k < K0 ? k : K0C) * H + nn];
    }
}

// Trainable-period gradient: given Hbar_in [S][Rpad][K0] (adjoint of the input
// features), back through RFF (B frozen) and the embedding to each trainable
// period: d phi/dP = -phi/P, d kappa/dP = -kappa/P.
template <int L>
static __global__ void k_input_bwd(InputArgs a, const float* __restrict__ Hb, double* __restrict__ partP) {
    using St = Streams<L>;
    constexpr int S = St::S;
    double accP[kMaxAxes] = {0.0, 0.0, 0.0, 0.0};
    const int64_t RK = (int64_t)a.Rpad * a.K0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.nrows; r += gridDim.x * blockDim.x) {
        double e[S][2 * kMaxAxes];
        embed_row<L>(a, a.row0 + r, e);
        double eb[S][2 * kMaxAxes];
#pragma unroll
        for (int s = 0; s < S; ++s)
            for (int k = 0; k < a.E; ++k) eb[s][k] = 0.0;
        const float* hb = Hb + (int64_t)r * a.K0;
        if (a.rff_w == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s)
                for (int k = 0; k < a.E; ++k) eb[s][k] = hb[s * RK + k];
        } else {
            for (int c = 0; c < a.rff_w; ++c) {
                double m[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    double acc = 0.0;
                    for (int k = 0; k < a.E; ++k) acc += e[s][k] * a.rffB[(int64_t)k * a.rff_w + c];
                    m[s] = acc;
                }
                double sm, cm;
                sincos(m[0], &sm, &cm);
                double Cb[S], Sb[S], mb[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    Cb[s] = hb[s * RK + c];
                    Sb[s] = hb[s * RK + a.rff_w + c];
                    mb[s] = 0.0;
                }
                double cmb = Cb[0], smb = Sb[0];
#pragma unroll
                for (int s = 1; s < S; ++s) {
                    if (St::order(s) == 1) {
                        cmb += Sb[s] * m[s];
                        smb += -Cb[s] * m[s];
                        mb[s] += -sm * Cb[s] + cm * Sb[s];
                    } else {
                        const int p = St::partner(s);
                        const double ma = m[p], maa = m[s];
                        cmb += -Cb[s] * ma * ma + Sb[s] * maa;
                        smb += -Cb[s] * maa - Sb[s] * ma * ma;
                        mb[p] += -2.0 * cm * ma * Cb[s] - 2.0 * sm * ma * Sb[s];
                        mb[s] += -sm * Cb[s] + cm * Sb[s];
                    }
                }
                mb[0] += -sm * cmb + cm * smb;
#pragma unroll
                for (int s = 0; s < S; ++s)
                    for (int k = 0; k < a.E; ++k) eb[s][k] += mb[s] * a.rffB[(int64_t)k * a.rff_w + c];
            }
        }
        // embedding transpose, trainable periods only
        int col = 0;
        for (int ax = 0; ax < a.in_dim; ++ax) {
            if (!a.periodic[ax]) {
                col += 1;
                continue;
            }
            if (a.period_off[ax] >= 0) {
                const double x = a.coords[(int64_t)ax * a.ld + a.row0 + r];
                const double P = (double)a.params[a.period_off[ax]];
                const double kappa = 2.0 * CUDART_PI * (1.0 / P);
                const double phi = 2.0 * CUDART_PI * (x * (1.0 / P));
                double sp, cp;
                sincos(phi, &sp, &cp);
                double phib = -sp * eb[0][col] + cp * eb[0][col + 1], kb = 0.0;
#pragma unroll
                for (int s = 1; s < S; ++s) {
                    if (St::axis(s) != ax) continue;
                    const double Cb = eb[s][col], Sbv = eb[s][col + 1];
                    if (St::order(s) == 1) {
                        phib += -cp * kappa * Cb - sp * kappa * Sbv;
                        kb += -sp * Cb + cp * Sbv;
                    } else {
                        phib += sp * kappa * kappa * Cb - cp * kappa * kappa * Sbv;
                        kb += -2.0 * cp * kappa * Cb - 2.0 * sp * kappa * Sbv;
                    }
                }
                accP[ax] += phib * (-phi / P) + kb * (-kappa / P);
            }
            col += 2;
        }
    }
    // block reduction (fixed order) -> partP[block][axis]
    __shared__ double red[kMaxAxes][256];
    for (int ax = 0; ax < kMaxAxes; ++ax) red[ax][threadIdx.x] = accP[ax];
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off)
            for (int ax = 0; ax < kMaxAxes; ++ax) red[ax][threadIdx.x] += red[ax][threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int ax = 0; ax < kMaxAxes; ++ax) partP[blockIdx.x * kMaxAxes + ax] += red[ax][0];
}

// ---------------------------------------------------------------------------
// Tiled FFMA GEMM over all streams with fused jet prologue / epilogue.
//   C[s] = PRO(A[s]) (Rpad x K) * B (K x N)
//   EPI_BIAS : out[s] = C[s] + [s==0] bias           (forward layer)
//   EPI_ACTT : out[s] = act^T(Zlow; C)[s]            (reverse layer)
//   EPI_RAW  : out[s] = C[s]
// ---------------------------------------------------------------------------
enum Epi : int { EPI_BIAS = 0, EPI_ACTT = 1, EPI_RAW = 2 };

struct GemmArgs {
    const float* A;   // [S][Rpad][K]
    const float* B;   // [K][N]
    const float* bias;
    const float* Zlow;  // [S][Rpad][N] (EPI_ACTT)
    float* out;       // [S][Rpad][N]
    int Rpad, K, N;
    float w0;
};

constexpr int GT_M = 64, GT_N = 64, GT_K = 16;

template <int L, int PRO, int EPI, int EACT>
__global__ void __launch_bounds__(256) k_gemm(GemmArgs g) {
    constexpr int S = Streams<L>::S;
    __shared__ __align__(16) float As[S][GT_K][GT_M + 4];
    __shared__ __align__(16) float Bs[GT_K][GT_N + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int r0 = blockIdx.x * GT_M, n0 = blockIdx.y * GT_N;
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * g.N;
    float acc[S][4][4];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[s][i][j] = 0.0f;

    for (int k0 = 0; k0 < g.K; k0 += GT_K) {
#pragma unroll
        for (int e = 0; e < (GT_M * GT_K) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int r = idx / GT_K, k = idx % GT_K;
            float z[S], h[S];
            if (k0 + k < g.K) {
                const float* p = g.A + (int64_t)(r0 + r) * g.K + k0 + k;
#pragma unroll
                for (int s = 0; s < S; ++s) z[s] = p[s * RK];
                act_fwd<L, PRO>(z, h, g.w0);
            } else {
#pragma unroll
                for (int s = 0; s < S; ++s) h[s] = 0.0f;
            }
#pragma unroll
            for (int s = 0; s < S; ++s) As[s][k][r] = h[s];
        }
#pragma unroll
        for (int e = 0; e < (GT_K * GT_N) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int k = idx / GT_N, n = idx % GT_N;
            Bs[k][n] = (k0 + k < g.K && n0 + n < g.N) ? g.B[(int64_t)(k0 + k) * g.N + n0 + n] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GT_K; ++kk) {
            const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
            const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float4 a4 = *reinterpret_cast<const float4*>(&As[s][kk][ty * 4]);
                const float a[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[s][i][j] = fmaf(a[i], b[j], acc[s][i][j]);
            }
        }
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + ty * 4 + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= g.N) continue;
            const int64_t o = (int64_t)r * g.N + n;
            if constexpr (EPI == EPI_BIAS) {  // EACT: activation of this layer's output
                g.out[o] = store_value<EACT>(acc[0][i][j] + g.bias[n]);
#pragma unroll
                for (int s = 1; s < S; ++s) g.out[s * RN + o] = acc[s][i][j];
            } else if constexpr (EPI == EPI_RAW) {
#pragma unroll
                for (int s = 0; s < S; ++s) g.out[s * RN + o] = acc[s][i][j];
            } else {
                float z[S], hb[S], zb[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    z[s] = g.Zlow[s * RN + o];
                    hb[s] = acc[s][i][j];
                }
                act_bwd<L, EACT>(z, hb, zb, g.w0);
#pragma unroll
                for (int s = 0; s < S; ++s) g.out[s * RN + o] = zb[s];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Weight gradient: part[split][k][n] += sum_s sum_r PRO(A[s][r][k]) Bm[s][r][n]
// (FP32 over a 16-row block, FP64 across blocks; deterministic split order).
// blockIdx.y == 0 CTAs also produce db[n] = sum_r Bm[0][r][n].
// ---------------------------------------------------------------------------
struct WgradArgs {
    const float* A;   // [S][Rpad][K]
    const float* Bm;  // [S][Rpad][N]
    double* part;     // [splits][K*N + N]
    int Rpad, nrows_valid, K, N, rows_per_split;
    float w0;
};

constexpr int WT_R = 16;

template <int L, int PRO>
__global__ void __launch_bounds__(256) k_wgrad(WgradArgs g) {
    constexpr int S = Streams<L>::S;
    __shared__ __align__(16) float As[S][WT_R][64 + 4];
    __shared__ __align__(16) float Bs[S][WT_R][64 + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int n0 = blockIdx.x * 64, k0 = blockIdx.y * 64;
    const int rbeg = blockIdx.z * g.rows_per_split;
    const int rend = min(g.nrows_valid, rbeg + g.rows_per_split);
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * g.N;
    double dacc[4][4];
    double dbias[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dacc[i][j] = 0.0;

    for (int rb = rbeg; rb < rend; rb += WT_R) {
#pragma unroll
        for (int e = 0; e < (WT_R * 64) / 256; ++e) {
            const int idx = tid + 256 * e;
            const int r = idx / 64, c = idx % 64;
            const bool rv = rb + r < rend;
            float z[S], h[S];
            if (rv && k0 + c < g.K) {
                const float* p = g.A + (int64_t)(rb + r) * g.K + k0 + c;
#pragma unroll
                for (int s = 0; s < S; ++s) z[s] = p[s * RK];
                act_fwd<L, PRO>(z, h, g.w0);
            } else {
#pragma unroll
                for (int s = 0; s < S; ++s) h[s] = 0.0f;
            }
#pragma unroll
            for (int s = 0; s < S; ++s) As[s][r][c] = h[s];
            const bool cv = rv && n0 + c < g.N;
            const float* q = g.Bm + (int64_t)(rb + r) * g.N + n0 + c;
#pragma unroll
            for (int s = 0; s < S; ++s) Bs[s][r][c] = cv ? q[s * RN] : 0.0f;
        }
        __syncthreads();
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
        float bsum[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int r = 0; r < WT_R; ++r) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float4 a4 = *reinterpret_cast<const float4*>(&As[s][r][ty * 4]);
                const float4 b4 = *reinterpret_cast<const float4*>(&Bs[s][r][tx * 4]);
                const float a[4] = {a4.x, a4.y, a4.z, a4.w};
                const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
                if (s == 0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) bsum[j] += b[j];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dacc[i][j] += (double)acc[i][j];
#pragma unroll
        for (int j = 0; j < 4; ++j) dbias[j] += (double)bsum[j];
        __syncthreads();
    }
    double* part = g.part + (int64_t)blockIdx.z * ((int64_t)g.K * g.N + g.N);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = k0 + ty * 4 + i;
        if (k >= g.K) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n < g.N) part[(int64_t)k * g.N + n] += dacc[i][j];
        }
    }
    if (blockIdx.y == 0 && ty == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n < g.N) part[(int64_t)g.K * g.N + n] += dbias[j];
        }
    }
}

// ---------------------------------------------------------------------------
// Head: last linear layer + residual / data losses + seeds + first reverse
// step, one warp per row (losses.cpp:77-144, trainer.cpp:234-236).
// ---------------------------------------------------------------------------
constexpr int kHeadMaxJ = 16;  // hidden width <= 512
constexpr int kHeadWarps = 8;
constexpr int kHeadBlocks = 2;  // resident head blocks per SM (grid = kHeadBlocks x SMs; 3 is slower)

struct HeadArgs {
    const float* Z;      // [S][Rpad][H]
    float* Zb;           // [S][Rpad][H]
    unsigned* zb_amax;   // optional: per-stream |Zb| bound (float bits, 3xFP16 scales)
    const float* W;      // [H][F]
    const float* b;      // [F]
    int H, Rpad, nrows;
    int64_t row0;        // global row of chunk row 0
    // global row segments: [bca0,bca1) [bcb0,bcb1) [ic0,ic1) [int0,int1)
    int64_t bca0, bca1, bcb0, bcb1, ic0, ic1, int0, int1;
    int bc_mode;
    const float* ic_t;   // [F][n_ic]
    const float* bc_t;   // [F][n_bc]
    const float* bc_vals;  // periodic: [2][n_pairs][F]
    float w_pde, w_ic, w_bc;  // 2*lambda/n per term
    PdeConst pc;
    float w0;
    double* loss_part;   // [grid][3]
    double* head_part;   // [grid][H*F + F]
    int* bad;            // [3] first non-finite interior index per component
    float* resid_out;    // optional [K][n_int] (interior residuals, diagnostics)
    int values_only;     // periodic prepass: write O[0] of bc rows to bc_vals
    float* vals_out;
    int rbeg;            // first chunk row this launch visits
    // stats pre-pass (stats = 1): no seeds; per-block FP64 sums for the two
    // objective terms whose seeds need global reductions first
    int stats;
    // temporal causality (trainer.cpp:156-177, losses.cpp:163-185): interior rows
    // bucketed by their last coordinate; seeds scaled per segment by seg_w
    int seg_M;
    double seg_tlo, seg_span;
    const double* tcoord;  // last-axis coordinate of every global row
    const float* seg_w;    // [M] 2 lambda_pde omega_i / (M n_i)
    double* seg_part;      // [grid][M] sum of r^2 per segment (stats)
    // Poynting penalty rows [poy0, poy1): poy_T samples of poy_n2 nodes each
    int64_t poy0, poy1;
    int poy_T, poy_n2;
    const float* poy_g;    // [T][3] seed multipliers for (Ez, Hx, Hy)
    double* poy_part;      // [grid][T][2] sum Ez^2, sum Hx^2 + Hy^2 (stats)
};
constexpr int kStatMax = 64;  // max causality segments / Poynting time samples

template <int P, int ACT, int J>
__global__ void __launch_bounds__(32 * kHeadWarps, kHeadBlocks) k_head(HeadArgs a) {
    using Tr = PdeTraits<P>;
    constexpr int L = Tr::L, F = Tr::F, K = Tr::K;
    constexpr int S = Streams<L>::S;
    constexpr int FLUSH = 16;  // rows accumulated in FP32 before the FP64 flush
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * kHeadWarps + wid, nw = gridDim.x * kHeadWarps;
    const int64_t RH = (int64_t)a.Rpad * a.H;
    // lane owns features k = lane + 32 j (coalesced per j); W_L in shared memory
    __shared__ float Ws[512 * 3];
    extern __shared__ double head_dyn[];  // per-warp FP64 dW_L / db_L: [kHeadWarps][H*F + F]
    const int acc_ld = a.H * F + F;
    double* accw = head_dyn + (int64_t)wid * acc_ld;
    for (int i = threadIdx.x; i < a.H * F; i += blockDim.x) Ws[i] = a.W[i];
    for (int i = lane; i < acc_ld; i += 32) accw[i] = 0.0;
    __syncthreads();

    unsigned zmx[S];
#pragma unroll
    for (int s = 0; s < S; ++s) zmx[s] = 0;
    float accW[J][F];
    float accB[F];
#pragma unroll
    for (int j = 0; j < J; ++j)
#pragma unroll
        for (int f = 0; f < F; ++f) accW[j][f] = 0.0f;
#pragma unroll
    for (int f = 0; f < F; ++f) accB[f] = 0.0f;
    double lpde = 0.0, lic = 0.0, lbc = 0.0;
    int since_flush = 0;

    auto load_row = [&](int r, float (*zz)[J]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
#pragma unroll
            for (int s = 0; s < S; ++s) zz[s][j] = (k < a.H) ? __ldg(a.Z + s * RH + (int64_t)r * a.H + k) : 0.0f;
        }
    };
    auto flush = [&]() {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
            if (k < a.H)
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    accw[k * F + f] += (double)accW[j][f];
                    accW[j][f] = 0.0f;
                }
        }
        if (lane == 0)
#pragma unroll
            for (int f = 0; f < F; ++f) accw[a.H * F + f] += (double)accB[f];
#pragma unroll
        for (int f = 0; f < F; ++f) accB[f] = 0.0f;
        since_flush = 0;
    };

    // stats pre-pass accumulators (lane 0 of each warp; fixed-order block fold)
    __shared__ double sacc[kHeadWarps][3 * kStatMax];
    if (a.stats) {
        for (int i = lane; i < 3 * kStatMax; i += 32) sacc[wid][i] = 0.0;
        __syncwarp();
    }
    // one row per warp iteration, no register prefetch of the next row: the
    // prefetch pushed the kernel into local-memory spills (2.5 -> 2.0 ms at C5
    // without it; occupancy hides the load latency)
    float z[S][J];
    int r = a.rbeg + gw;
    for (; r < a.nrows; r += nw) {
        load_row(r, z);
        const int64_t g = a.row0 + r;
        float o[S * F];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int f = 0; f < F; ++f) o[s * F + f] = 0.0f;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
            float zz[S], hh[S];
#pragma unroll
            for (int s = 0; s < S; ++s) zz[s] = z[s][j];
            act_fwd<L, ACT>(zz, hh, a.w0);
#pragma unroll
            for (int f = 0; f < F; ++f) {
                const float w = (k < a.H) ? Ws[k * F + f] : 0.0f;
#pragma unroll
                for (int s = 0; s < S; ++s) o[s * F + f] = fmaf(hh[s], w, o[s * F + f]);
            }
        }
#pragma unroll
        for (int i = 0; i < S * F; ++i) {
            float v = o[i];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            o[i] = v;
        }
#pragma unroll
        for (int f = 0; f < F; ++f) o[f] += a.b[f];

        if (a.stats) {
            if (lane == 0) {
                if (a.seg_M > 0 && g >= a.int0 && g < a.int1) {
                    float res[K];
                    residual<P>(o, res, a.pc);
                    double sq = 0.0;
#pragma unroll
                    for (int k = 0; k < K; ++k) sq += (double)res[k] * (double)res[k];
                    const double frac = (a.tcoord[g] - a.seg_tlo) / a.seg_span;
                    const int sg = min(a.seg_M - 1, max(0, (int)(frac * a.seg_M)));
                    sacc[wid][sg] += sq;
                } else if (g >= a.poy0 && g < a.poy1) {
                    const int j = (int)((g - a.poy0) / a.poy_n2);
                    sacc[wid][kStatMax + 2 * j] += (double)o[0] * (double)o[0];
                    sacc[wid][kStatMax + 2 * j + 1] += (double)o[1] * (double)o[1] + (double)o[2] * (double)o[2];
                }
            }
        } else if (a.values_only) {
            if (lane == 0) {
                int64_t slot = -1;
                if (g >= a.bca0 && g < a.bca1) slot = g - a.bca0;
                else if (g >= a.bcb0 && g < a.bcb1) slot = (a.bca1 - a.bca0) + (g - a.bcb0);
                if (slot >= 0)
                    for (int f = 0; f < F; ++f) a.vals_out[slot * F + f] = o[f];
            }
        } else {
            float ob[S * F];
#pragma unroll
            for (int i = 0; i < S * F; ++i) ob[i] = 0.0f;
            if (g >= a.int0 && g < a.int1) {
                float res[K], rb[K];
                residual<P>(o, res, a.pc);
                float sq = 0.0f;
                float wr = a.w_pde;
                if (a.seg_M > 0) {  // causality: per-segment weight (losses.cpp:173-185)
                    const double frac = (a.tcoord[g] - a.seg_tlo) / a.seg_span;
                    wr = a.seg_w[min(a.seg_M - 1, max(0, (int)(frac * a.seg_M)))];
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    sq += res[k] * res[k];
                    rb[k] = wr * res[k];
                    if (lane == 0 && !isfinite(res[k])) atomicMin(&a.bad[k], (int)(g - a.int0));
                }
                if (a.resid_out && lane == 0) {
                    const int64_t n_int = a.int1 - a.int0;
#pragma unroll
                    for (int k = 0; k < K; ++k) a.resid_out[k * n_int + (g - a.int0)] = res[k];
                }
                lpde += (double)sq;
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
                lic += (double)sq;
            } else if (a.bc_mode == 2 && g >= a.bca0 && g < a.bca1) {
                const int64_t i = g - a.bca0, n = a.bca1 - a.bca0;
                float sq = 0.0f;
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    const float d = o[f] - a.bc_t[f * n + i];
                    sq += d * d;
                    ob[f] = a.w_bc * d;
                }
                lbc += (double)sq;
            } else if (a.bc_mode == 1 && g >= a.bca0 && g < a.bca1) {
                const int64_t i = g - a.bca0, np = a.bca1 - a.bca0;
                float sq = 0.0f;
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    const float d = o[f] - a.bc_vals[(np + i) * F + f];
                    sq += d * d;
                    ob[f] = a.w_bc * d;
                }
                lbc += (double)sq;
            } else if (a.bc_mode == 1 && g >= a.bcb0 && g < a.bcb1) {
                const int64_t i = g - a.bcb0;
#pragma unroll
                for (int f = 0; f < F; ++f) ob[f] = -a.w_bc * (a.bc_vals[i * F + f] - o[f]);
            } else if (g >= a.poy0 && g < a.poy1) {
                // Poynting nodes: value-stream seeds weight * dpen/dE_j * dE_j/dfield
                const int j = (int)((g - a.poy0) / a.poy_n2);
#pragma unroll
                for (int f = 0; f < F; ++f) ob[f] = (f < 3 ? a.poy_g[3 * j + f] : 0.0f) * o[f];
            }
            // reverse through the head: hbar = Obar W^T, dW_L += h^T Obar
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int k = lane + 32 * j;
                float w[F];
#pragma unroll
                for (int f = 0; f < F; ++f) w[f] = (k < a.H) ? Ws[k * F + f] : 0.0f;
                float zz[S], hh[S], hb[S], zb[S];
#pragma unroll
                for (int s = 0; s < S; ++s) zz[s] = z[s][j];
                act_fwd<L, ACT>(zz, hh, a.w0);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    float v = 0.0f;
#pragma unroll
                    for (int f = 0; f < F; ++f) v = fmaf(ob[s * F + f], w[f], v);
                    hb[s] = v;
                }
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    float v = accW[j][f];
#pragma unroll
                    for (int s = 0; s < S; ++s) v = fmaf(hh[s], ob[s * F + f], v);
                    accW[j][f] = v;
                }
                if (k < a.H) {
                    act_bwd<L, ACT>(zz, hb, zb, a.w0);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        a.Zb[s * RH + (int64_t)r * a.H + k] = zb[s];
                        zmx[s] = max(zmx[s], __float_as_uint(fabsf(zb[s])));
                    }
                }
            }
#pragma unroll
            for (int f = 0; f < F; ++f) accB[f] += ob[f];
            if (++since_flush == FLUSH) flush();
        }

    }
    if (a.stats) {  // fixed-order fold of the warps' sums, one partial per block
        __syncthreads();
        for (int i = threadIdx.x; i < 3 * kStatMax; i += blockDim.x) {
            double v = 0.0;
            for (int w = 0; w < kHeadWarps; ++w) v += sacc[w][i];
            // accumulate: the buffers are zeroed per step and several chunks may contribute
            if (i < kStatMax) {
                if (i < a.seg_M) a.seg_part[(int64_t)blockIdx.x * a.seg_M + i] += v;
            } else if (i - kStatMax < 2 * a.poy_T) {
                a.poy_part[(int64_t)blockIdx.x * 2 * a.poy_T + (i - kStatMax)] += v;
            }
        }
        return;
    }
    if (a.values_only) return;
    flush();
    if (a.zb_amax) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const unsigned v = __reduce_max_sync(0xffffffffu, zmx[s]);
            if (lane == 0) atomicMax(a.zb_amax + s, v);
        }
    }
    // pad rows of the chunk: zero adjoints so they contribute nothing
    for (int r2 = a.nrows + gw; r2 < a.Rpad; r2 += nw)
        for (int k = lane; k < a.H; k += 32)
#pragma unroll
            for (int s = 0; s < S; ++s) a.Zb[s * RH + (int64_t)r2 * a.H + k] = 0.0f;

    // deterministic block reduction: warps in order
    __shared__ double lsum[kHeadWarps][3];
    if (lane == 0) {
        lsum[wid][0] = lpde;
        lsum[wid][1] = lic;
        lsum[wid][2] = lbc;
    }
    __syncthreads();
    const int nWF = a.H * F;
    double* hp = a.head_part + (int64_t)blockIdx.x * (nWF + F);
    for (int i = threadIdx.x; i < nWF + F; i += blockDim.x) {
        double v = 0.0;
        for (int w = 0; w < kHeadWarps; ++w) v += head_dyn[(int64_t)w * acc_ld + i];
        hp[i] += v;
    }
    if (threadIdx.x < 3) {
        double v = 0.0;
        for (int w = 0; w < kHeadWarps; ++w) v += lsum[w][threadIdx.x];
        a.loss_part[blockIdx.x * 3 + threadIdx.x] += v;
    }
}

// ---------------------------------------------------------------------------
// finalize: fixed-order reduction of partials -> flat float32 gradient in
// trainable() order (RWF: dV = dW*exp(s), ds = exp(s)*colsum(dW*V)), losses.
// ---------------------------------------------------------------------------
struct FinalArgs {
    LayerTab t;
    const double* part[kMaxLayers];  // per layer: [nsplit][K*N + N]
    int nsplit[kMaxLayers];
    const float* params;
    float* grad;                     // flat
    double* dWscratch;               // max(K*N + N) doubles
};

// reduce splits of layer l into dWscratch (double)
// out[i] = sum_p part[p][i] in a fixed order: a 32 x 8 block takes 32 consecutive
// entries; thread row y sums the splits p = y, y + 8, ... into four interleaved
// partials (loads in flight), the rows are folded in order y = 0..7. Many
// splits of a short vector (the head's per-block partials) and few splits of a
// long one both keep every SM busy.
constexpr int kRsX = 32, kRsY = 8;
static __global__ void __launch_bounds__(kRsX* kRsY) k_reduce_splits(const double* __restrict__ part, int nsplit,
                                                                   int64_t len, double* __restrict__ out) {
    __shared__ double acc[kRsY][kRsX];
    const int x = threadIdx.x % kRsX, y = threadIdx.x / kRsX;
    for (int64_t i0 = (int64_t)blockIdx.x * kRsX; i0 < len; i0 += (int64_t)gridDim.x * kRsX) {
        const int64_t i = i0 + x;
        double s[4] = {0.0, 0.0, 0.0, 0.0};
        if (i < len) {
            int p = y;
            for (; p + 3 * kRsY < nsplit; p += 4 * kRsY) {
#pragma unroll
                for (int u = 0; u < 4; ++u) s[u] += part[(int64_t)(p + u * kRsY) * len + i];
            }
            for (int u = 0; p < nsplit; p += kRsY, ++u) s[u] += part[(int64_t)p * len + i];
        }
        acc[y][x] = (s[0] + s[1]) + (s[2] + s[3]);
        __syncthreads();
        if (y == 0 && i < len) {
            double t = acc[0][x];
#pragma unroll
            for (int r = 1; r < kRsY; ++r) t += acc[r][x];
            out[i] = t;
        }
        __syncthreads();
    }
}
inline unsigned reduce_splits_grid(int64_t len) {
    const int64_t b = (len + kRsX - 1) / kRsX;
    return (unsigned)(b < 4096 ? b : 4096);
}

// write layer l's flat grads from the reduced dW (K*N) + db (N)
static __global__ void k_write_layer_grad(const double* __restrict__ red, const float* __restrict__ params,
                                   int K, int N, int64_t offW, int64_t offS, int64_t offB, float scale,
                                   float* __restrict__ grad) {
    const int64_t total = (int64_t)K * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total + N;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < total) {
            const int n = (int)(i % N);
            double v = red[i];
            if (offS >= 0) v *= exp((double)params[offS + n]);
            grad[offW + i] = (float)(v * scale);
        } else {
            const int n = (int)(i - total);
            grad[offB + n] = (float)(red[total + n] * scale);
        }
    }
}

// RWF scale gradient ds_n = exp(s_n) * sum_k dW[k][n] V[k][n] (model.cpp:117-126):
// one warp per n, lanes stride k, a fixed shuffle tree
static __global__ void k_write_rwf_ds(const double* __restrict__ red, const float* __restrict__ params, int K, int N,
                                      int64_t offW, int64_t offS, float scale, float* __restrict__ grad) {
    const int lane = threadIdx.x & 31;
    for (int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < N; n += gridDim.x * (blockDim.x >> 5)) {
        double acc = 0.0;
        for (int k = lane; k < K; k += 32) acc += red[(int64_t)k * N + n] * (double)params[offW + (int64_t)k * N + n];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) grad[offS + n] = (float)(exp((double)params[offS + n]) * acc * scale);
    }
}

// Causality weights from the stats pass (losses.cpp:163-185): L_i = S_i / n_i
// (0 for empty segments), omega_0 = 1, omega_i = exp(-eps sum_{j<i} L_j);
// seeds 2 lambda omega_i / (M n_i); l_pde = (1/M) sum omega_i L_i.
static __global__ void k_causality_weights(const double* __restrict__ seg_part, int nblk, int M,
                                           const double* __restrict__ cnt, double eps, double lam,
                                           float* __restrict__ seg_w, double* __restrict__ lpde) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double acc = 0.0, tot = 0.0;
    for (int i = 0; i < M; ++i) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += seg_part[(int64_t)b * M + i];
        const double Li = cnt[i] > 0.0 ? s / cnt[i] : 0.0;
        const double om = i == 0 ? 1.0 : exp(-eps * acc);
        acc += Li;
        tot += om * Li;
        seg_w[i] = cnt[i] > 0.0 ? (float)(2.0 * lam * om / ((double)M * cnt[i])) : 0.0f;
    }
    *lpde = tot / (double)M;
}

// Poynting penalty from the stats pass (losses.cpp:187-223):
// E_j = cell/2 (eps sum Ez^2 + mu sum (Hx^2 + Hy^2)), pen = mean_j (E_{j+1} - E_j)^2;
// g[j] = weight * dpen/dE_j * cell * (eps, mu, mu) multiplies (Ez, Hx, Hy).
static __global__ void k_poynting_weights(const double* __restrict__ poy_part, int nblk, int T, double cell,
                                          double eps, double mu, double weight, float* __restrict__ g,
                                          double* __restrict__ pen) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double E[kStatMax];
    for (int j = 0; j < T; ++j) {
        double se = 0.0, sh = 0.0;
        for (int b = 0; b < nblk; ++b) {
            se += poy_part[((int64_t)b * T + j) * 2];
            sh += poy_part[((int64_t)b * T + j) * 2 + 1];
        }
        E[j] = 0.5 * cell * (eps * se + mu * sh);
    }
    double p = 0.0;
    for (int j = 0; j + 1 < T; ++j) p += (E[j + 1] - E[j]) * (E[j + 1] - E[j]);
    *pen = p / (double)(T - 1);
    for (int j = 0; j < T; ++j) {
        double dE = 0.0;
        if (j > 0) dE += 2.0 * (E[j] - E[j - 1]) / (double)(T - 1);
        if (j + 1 < T) dE -= 2.0 * (E[j + 1] - E[j]) / (double)(T - 1);
        g[3 * j + 0] = (float)(weight * dE * cell * eps);
        g[3 * j + 1] = (float)(weight * dE * cell * mu);
        g[3 * j + 2] = (float)(weight * dE * cell * mu);
    }
}

static __global__ void k_write_scalar_grads(const double* __restrict__ partP, int nblk, const int64_t* offs,
                                     int naxes, float scale, float* __restrict__ grad,
                                     const double* __restrict__ loss_part, int nloss_blk,
                                     const double* inv_n, double* __restrict__ losses_out,
                                     const double* __restrict__ pde_override = nullptr) {
    // one warp per sum (warps 0-2: the loss terms, 3..: the period axes): lanes
    // stride the blocks, then a fixed shuffle tree (launched with 32 * (3 + kMaxAxes) threads)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (blockIdx.x != 0) return;
    if (w < 3) {
        if (!losses_out) return;
        double s = 0.0;
        for (int b = lane; b < nloss_blk; b += 32) s += loss_part[b * 3 + w];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) losses_out[w] = (w == 0 && pde_override) ? *pde_override : s * inv_n[w];
    } else if (w - 3 < naxes) {
        const int ax = w - 3;
        if (offs[ax] < 0) return;
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += partP[b * kMaxAxes + ax];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) grad[offs[ax]] = (float)(s * scale);
    }
}
constexpr int kScalarGradThreads = 32 * (3 + kMaxAxes);

// ---------------------------------------------------------------------------
// Adam (optim.cpp:7-41) fused with the 1/W average (trainer.cpp:278-280)
// ---------------------------------------------------------------------------
// Non-finite gradients (optim.cpp:16-22: "adam: non-finite gradient for
// parameter <name> at step t" aborts before any update): k_any_nonfinite first
// records the smallest bad index in bad[0]; the update kernels then skip the
// whole step (bad[0] != kBadNone) and note its step number in bad[1]; the host
// reports both at the next pnx_check (the flags are sticky until read).
constexpr int kBadNone = 0x7f7f7f7f;
static __global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps,
                       float bc1, float bc2, float gscale, int* __restrict__ bad, int t) {
    if (*(volatile int*)bad != kBadNone) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(bad + 1, kBadNone, t);
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float gi = g[i] * gscale;
        const float mi = b1 * m[i] + (1.0f - b1) * gi;
        const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    }
}

// Same update with the step count t and the epoch in device memory (state[0] =
// steps taken, state[1] = epoch): bias corrections and lr = lr0 gamma^epoch
// (ExponentialLr::at, optim.cpp:71-73) are formed on the device, so a captured
// CUDA graph replays correct updates; k_adam_tick advances both after the update
// (the step count only when the update ran).
static __global__ void k_adam_state(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                    float* __restrict__ v, int64_t n, const double* __restrict__ state, double lr0,
                                    double gamma, double b1d, double b2d, float eps, float gscale,
                                    int* __restrict__ bad) {
    const double t = state[0] + 1.0;
    if (*(volatile int*)bad != kBadNone) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(bad + 1, kBadNone, (int)t);
        return;
    }
    const float lr = (float)(lr0 * pow(gamma, state[1]));
    const float bc1 = (float)(1.0 - pow(b1d, t)), bc2 = (float)(1.0 - pow(b2d, t));
    const float b1 = (float)b1d, b2 = (float)b2d;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float gi = g[i] * gscale;
        const float mi = b1 * m[i] + (1.0f - b1) * gi;
        const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    }
}
static __global__ void k_adam_tick(double* state, const int* __restrict__ bad) {
    if (*bad == kBadNone) state[0] += 1.0;
    state[1] += 1.0;
}

static __global__ void k_f64_to_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

static __global__ void k_any_nonfinite(const float* __restrict__ g, int64_t n, int* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(g[i])) atomicMin(flag, (int)i);
}

}  // namespace pnx
