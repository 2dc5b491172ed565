// tc_gemm.cuh -- the hidden-layer contractions of the jet train step on sm_100a
// 5th-generation tensor cores: tcgen05.mma kind::tf32 with FP32 accumulators
// in TMEM and 3xTF32 split accumulation (x = hi + lo, D += Ah*Bh + Ah*Bl + Al*Bh)
// to hold FP32 accuracy.
//
//   k_tc_fwd   Z_out[s] = act(Z_in)[s] W + [s==0] b          (model.cpp:163-175)
//   k_tc_bwd   Zb_in[s] = act^T(Zb_out[s] W^T ; Z_in)         (graph.cpp:468-502)
//   k_tc_wgrad dW = sum_s act(Z_in)[s]^T Zb_out[s] per row tile, + db
//
// One CTA per SM (TMEM: 512 columns). Operands live in shared memory as
// K-major 32-byte-swizzled tiles (K = 8 fp32 per stage = one MMA K step):
// all 8 warps produce a stage (load -> jet activation -> hi/lo split ->
// swizzled st.shared), thread 0 issues the 3 MMAs per accumulator and commits
// to the stage's mbarrier, so production of stage i+1 overlaps the tensor
// core on stage i. Weights are pre-split and pre-swizzled once per step into
// "stage images" (k_tc_prep_images) and copied 16 B at a time.
#pragma once
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>

#include "jets.cuh"
#include "kernels_simt.cuh"
#include "tc_common.cuh"

namespace pnx {

constexpr int TC_M = 128;          // rows per MMA / per CTA tile
constexpr int TC_TILE_BYTES = 4096;  // 128 rows x 8 fp32 (one SW32 K-major tile)
constexpr int TC_SMEM = 200 * 1024;
constexpr int TC_WROWS = 512;      // rows per weight-gradient tile (FP32 partial)

struct TcWorkspace {
    float* img = nullptr;          // weight stage images, all layers
    int64_t img_cap = 0;
    int64_t img_fwd[kMaxLayers] = {};
    int64_t img_bwd[kMaxLayers] = {};
    float* wpart = nullptr;        // [n_wtiles][K*N] FP32 partials
    int64_t wpart_cap = 0;
    double* dbpart = nullptr;      // [n_wtiles][N]
    int64_t dbpart_cap = 0;
    double* red = nullptr;         // [TC_WRED_G][K*N + N] first-level reduction
    int64_t red_cap = 0;
    bool attrs_set = false;
};

// NT: output columns per CTA so that S * NT <= 512 TMEM columns.
__host__ __device__ constexpr int tc_nt(int S) { return S <= 4 ? 128 : 64; }

// ---------------------------------------------------------------------------
// weight images: img[(ntile * (K/8) + kb)] = {hi tile, lo tile}, NT x 8 each,
// element (n, k) of B at sw32_off(n % NT, k % 8). fwd: B(n,k) = W[k][n];
// bwd: B(n = k_in, k = n_out) = W[n][k].
// ---------------------------------------------------------------------------
static __global__ void k_tc_prep_image(const float* __restrict__ W, int K, int N, int transpose_b, int NT,
                                float* __restrict__ img) {
    // B is (rowsB x KB): fwd rowsB = N, KB = K ; bwd rowsB = K, KB = N
    const int rowsB = transpose_b ? K : N, KB = transpose_b ? N : K;
    const int64_t total = (int64_t)rowsB * KB;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i / KB), k = (int)(i % KB);
        const float w = transpose_b ? W[(int64_t)n * N + k] : W[(int64_t)k * N + n];
        float hi, lo;
        tc::split3(w, hi, lo);
        const int nt = n / NT, kb = k / 8;
        const int64_t blk = ((int64_t)nt * (KB / 8) + kb) * (2 * NT * 8);
        const uint32_t off = tc::sw32_off((uint32_t)(n % NT), (uint32_t)(k % 8)) / 4;
        img[blk + off] = hi;
        img[blk + NT * 8 + off] = lo;
    }
}

// 3xFP16 weight images: per 16-wide K block kb, {hi, lo} tiles of NT rows x 16
// fp16 (32 B rows, SW32 like the tf32 tiles), element (n, k) at
// sw32h_off(n % NT, k % 16); W is scaled by 2^e, e = f16_exp_bits(*wamax).
static __global__ void k_tc_prep_image16(const float* __restrict__ W, int K, int N, int transpose_b, int NT,
                                         const unsigned* __restrict__ wamax, uint16_t* __restrict__ img) {
    const int rowsB = transpose_b ? K : N, KB = transpose_b ? N : K;
    const float sc = ldexpf(1.0f, tc::f16_exp_bits(*wamax));
    const int64_t total = (int64_t)rowsB * KB;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int n = (int)(i / KB), k = (int)(i % KB);
        const float w = (transpose_b ? W[(int64_t)n * N + k] : W[(int64_t)k * N + n]) * sc;
        const __half hi = __float2half_rn(w);
        const __half lo = __float2half_rn(w - __half2float(hi));
        const int nt = n / NT, kb = k / 16;
        const int64_t blk = ((int64_t)nt * (KB / 16) + kb) * (2 * NT * 16);
        const uint32_t off = tc::sw32h_off((uint32_t)(n % NT), (uint32_t)(k % 16)) / 2;
        img[blk + off] = __half_as_ushort(hi);
        img[blk + NT * 16 + off] = __half_as_ushort(lo);
    }
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts128u(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint32_t lds32u(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// streaming operand loads (read once per stage): policy selectable for experiments
__device__ __forceinline__ float4 ldg4(const float* p) {
#if defined(PNX_LD_CG)
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
#elif defined(PNX_LD_NA)
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
#else
    return __ldg(reinterpret_cast<const float4*>(p));
#endif
}
// truncation split: hi = x with the 13 low mantissa bits cleared (exact TF32),
// lo = x - hi (exact FP32, the MMA reads its TF32 part): two integer / FP ops per
// element instead of two cvt. Measured at parity in the general backward
// (k_tc2_bwd: C3 3.04 -> 2.71 ms/step); the other TF32 producers keep the
// rounding split (in the pair forward / decoupled backward / weight gradient the
// truncation measured 1.2e-4 against the oracle at C4 -- not investigated further)
__device__ __forceinline__ void split4_trunc(float4 v, float4& hi, float4& lo) {
    const float4 h = make_float4(__uint_as_float(__float_as_uint(v.x) & 0xffffe000u),
                                 __uint_as_float(__float_as_uint(v.y) & 0xffffe000u),
                                 __uint_as_float(__float_as_uint(v.z) & 0xffffe000u),
                                 __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
    hi = h;
    lo = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}
__device__ __forceinline__ void split4(float4 v, float4& hi, float4& lo) {
    tc::split3(v.x, hi.x, lo.x);
    tc::split3(v.y, hi.y, lo.y);
    tc::split3(v.z, hi.z, lo.z);
    tc::split3(v.w, hi.w, lo.w);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// jet activation of 4 consecutive features for all streams (z: S float4)
template <int L, int PRO>
__device__ __forceinline__ void act4(const float4* z, float4* h) {
    constexpr int S = Streams<L>::S;
    float zz[S], hh[S];
#define ACT4_LANE(c)                                         \
    _Pragma("unroll") for (int s = 0; s < S; ++s) zz[s] = z[s].c; \
    act_fwd<L, PRO>(zz, hh, 1.0f);                           \
    _Pragma("unroll") for (int s = 0; s < S; ++s) h[s].c = hh[s];
    ACT4_LANE(x) ACT4_LANE(y) ACT4_LANE(z) ACT4_LANE(w)
#undef ACT4_LANE
}

// ---------------------------------------------------------------------------
// shared skeleton bits
// ---------------------------------------------------------------------------
struct TcGemmArgs {
    const float* A;     // [S][Rpad][K] (fwd: Z_in / Hin ; bwd: Zb_out)
    const float* img;   // weight stage images
    const float* bias;  // fwd
    const float* Zlow;  // bwd: Z_in [S][Rpad][N]
    float* out;         // [S][Rpad][N]
    int Rpad, K, N;
    // 3xFP16: |A| bounds per stream and the |W| bound (float bits) recorded by the
    // producers; amax_out (optional) records this kernel's output bounds per stream
    int f16;  // 1: 3xFP16 operands (fp16 weight image at img)
    const unsigned* amax_in;
    const unsigned* amax_w;
    unsigned* amax_out;
    CUtensorMap tmA;    // pair kernels: A as [S][Rpad][K], box {32, 128, 1}, 128 B swizzle
    CUtensorMap tmB;    // pair kernels: weight image as rows of 8 fp32, box {8, 128}
    CUtensorMap tmO;    // forward pair kernel: out as [S][Rpad][N], box {32, 32, 1}, 128 B swizzle
};

// ---------------------------------------------------------------------------
// weight gradient: per row tile of TC_WROWS rows,
//   wpart[tile][k][n] = sum_{rows, s} act(Z_in)[s][row][k] * Zb[s][row][n]
//   dbpart[tile][n]   = sum_rows Zb[0][row][n]
// M = k_in (MT tiles of 128), N = n_out, K = 8 rows of one stream per stage.
// Operands are written transposed (K-major: k = row) into SW32 tiles.
// ---------------------------------------------------------------------------
struct TcWgradArgs {
    const float* A;   // Z_in / Hin [S][Rpad][Kin]
    const float* Bm;  // Zb_out [S][Rpad][N]
    // 3xFP16 mode: per-stream |Z_in| and |Zb_out| bounds (float bits) recorded
    // by the producing kernels; one power-of-two scale per operand (the whole
    // reduction over rows and streams accumulates into one TMEM accumulator)
    const unsigned* amaxA;
    const unsigned* amaxB;
    int f16;
    CUtensorMap tmA;  // A as [S][Rpad][Kin], box {128, 8, S}
    CUtensorMap tmB;  // Bm as [S][Rpad][N], box {N, 8, S}
    float* wpart;
    double* dbpart;
    int Rpad, nrows, Kin, N;
};

// Host: fp32 tensor map over [d2][d1][d0] (d0 contiguous; d2 = 1 for 2-D), box
// {b0, b1, b2}. sw128: 128 B swizzle (16 B chunk c of box row r stored at c ^ (r % 8)),
// else the box lands in smem as a dense [b2][b1][b0] array.
int tc_make_tmap(CUtensorMap* map, const float* base, int rank, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                 uint32_t b1, uint32_t b2, bool sw128);
inline int tc_make_tmap_3d(CUtensorMap* map, const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                           uint32_t b1, uint32_t b2) {
    return tc_make_tmap(map, base, 3, d0, d1, d2, b0, b1, b2, false);
}

// Two-level fixed-order reduction of the weight-gradient tile partials:
//   level 1: group y sums tiles [y*T/G, (y+1)*T/G) in order (float4 loads, FP64)
//   level 2: part[i] += sum_y red[y][i] in y order
// (deterministic for a given tile count; replaces the one-pass k_tc_wreduce).
constexpr int TC_WRED_G = 16;
static __global__ void k_tc_wreduce1(const float* __restrict__ wpart, const double* __restrict__ dbpart, int ntiles,
                                     int K, int N, double* __restrict__ red) {
    const int64_t KN = (int64_t)K * N, len = KN + N;
    const int y = blockIdx.y;
    const int t0 = (int)((int64_t)ntiles * y / TC_WRED_G), t1 = (int)((int64_t)ntiles * (y + 1) / TC_WRED_G);
    for (int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i4 * 4 < len;
         i4 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i4 * 4;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (i < KN) {  // KN is a multiple of 4 (N % 4 == 0)
            int t = t0;
            for (; t + 4 <= t1; t += 4) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(wpart + (int64_t)(t + u) * KN + i));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    s0 += (double)v[u].x;
                    s1 += (double)v[u].y;
                    s2 += (double)v[u].z;
                    s3 += (double)v[u].w;
                }
            }
            for (; t < t1; ++t) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(wpart + (int64_t)t * KN + i));
                s0 += (double)v.x;
                s1 += (double)v.y;
                s2 += (double)v.z;
                s3 += (double)v.w;
            }
        } else {
            for (int t = t0; t < t1; ++t) {
                const double* d = dbpart + (int64_t)t * N + (i - KN);
                s0 += d[0];
                s1 += d[1];
                s2 += d[2];
                s3 += d[3];
            }
        }
        double* r = red + (int64_t)y * len + i;
        r[0] = s0;
        r[1] = s1;
        r[2] = s2;
        r[3] = s3;
    }
}
static __global__ void k_tc_wreduce2(const double* __restrict__ red, int64_t len, double* __restrict__ part) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int y = 0; y < TC_WRED_G; ++y) s += red[(int64_t)y * len + i];
        part[i] += s;
    }
}


// ---------------------------------------------------------------------------
// Persistent weight gradient (k_tc2_wgrad): G groups of MT = Kin/128 CTAs (one
// CTA per SM), each over a contiguous row range; the FP32 TMEM accumulator is
// drained into the group's slot every tc_wgrad_seg() rows. The truncating FP32
// accumulation error grows linearly with the rows per drain (DESIGN.md §4:
// 1024 rows 1.5e-5, 512 rows 8.8e-6 gradient rel-L2 at 1M points), so 256 rows
// keep the headline gradient well inside the north_star ~1e-5.
inline int tc_wgrad_seg() {
    static const int force = getenv("PNX_WG_SEG") ? atoi(getenv("PNX_WG_SEG")) : 0;  // A/B override
    return force >= 8 && force % 8 == 0 ? force : 256;
}
inline int tc_wgrad_groups(int64_t Rpad, int Kin, int nsm) {
    const int mt = Kin / 128;
    const int64_t g = nsm / mt > 1 ? nsm / mt : 1;
    return (int)(g < Rpad / 8 ? g : Rpad / 8);
}
constexpr int TC_WG_MAX_GROUPS = 256;  // slots allocated (>= SM count)

// the decoupled N=256 backward (k_tc5_bwd): first-order tanh layouts whose
// backward GEMM writes 256 features (PNX_TC5_OFF=1 falls back to k_tc2_bwd)
inline bool tc5_bwd_ok(int L, int nout, int kred) {
    static const bool off = getenv("PNX_TC5_OFF") != nullptr;
    return !off && (L == LAY_XT || L == LAY_MX) && nout == 256 && kred % 8 == 0;
}

// the CTA-pair forward (k_tc4_fwd) runs this layer (PNX_FWD_NOPAIR=1 disables it)
inline bool tc4_fwd_ok(int K, int N) {
    static const bool off = getenv("PNX_FWD_NOPAIR") != nullptr;
    return !off && N == 256 && K % 32 == 0;
}

inline bool tc_layer_ok(int S, int K, int N) {
    const int NT = tc_nt(S);
    return S <= 5 && K % 32 == 0 && K >= 32 && K <= 256 && N % NT == 0 && N <= 256 && (K == 128 || K == 256);
}

inline bool tc_enabled(int engine, int H, int S, int act) {
    if (engine == 1) return false;  // PNX_ENGINE_FFMA
    return (H == 128 || H == 256) && S <= 5 && act == ACT_TANH;
}

// extra_bytes: allocated past every buffer (the context's PNX_GUARD tails)
inline int tc_workspace_alloc(TcWorkspace& ws, int, int64_t Rpad, int H, int K0, size_t extra_bytes = 0) {
    {
        const int64_t kmax0 = H > K0 ? H : K0;
        const int64_t need_red = (int64_t)TC_WRED_G * (kmax0 * H + H);
        if (need_red > ws.red_cap) {
            if (ws.red) cudaFree(ws.red);
            if (cudaMalloc(&ws.red, need_red * sizeof(double) + extra_bytes) != cudaSuccess) return -2;
            ws.red_cap = need_red;
        }
    }
    (void)Rpad;
    const int64_t tiles = TC_WG_MAX_GROUPS;  // one FP32 slot per weight-gradient group
    const int64_t kmax = H > K0 ? H : K0;
    const int64_t need = tiles * kmax * H;
    if (need > ws.wpart_cap) {
        if (ws.wpart) cudaFree(ws.wpart);
        if (cudaMalloc(&ws.wpart, need * sizeof(float) + extra_bytes) != cudaSuccess) return -2;
        ws.wpart_cap = need;
    }
    if (tiles * H > ws.dbpart_cap) {
        if (ws.dbpart) cudaFree(ws.dbpart);
        if (cudaMalloc(&ws.dbpart, tiles * H * sizeof(double) + extra_bytes) != cudaSuccess) return -2;
        ws.dbpart_cap = tiles * H;
    }
    return 0;
}
inline void tc_workspace_free(TcWorkspace& ws) {
    if (ws.red) cudaFree(ws.red);
    if (ws.img) cudaFree(ws.img);
    if (ws.wpart) cudaFree(ws.wpart);
    if (ws.dbpart) cudaFree(ws.dbpart);
    ws = TcWorkspace{};
}


// ===========================================================================
// v2: warp-specialized kernels with split ("big" | "small") accumulators.
//
// Accumulating the 3xTF32 correction products (hi*lo, lo*hi) into the same
// FP32 TMEM accumulator as hi*hi truncates them against the large running sum
// (measured: 5.2e-7 vs 1.5e-7 rel. error for FP32 FMA at K=64). Keeping them in
// a separate "small" accumulator restores FP32-level accuracy (1.9e-7); the
// epilogue adds big + small. N=256 MMAs with the A operand reused by two
// consecutive MMAs keep the SMEM operand traffic under the tensor pipe's rate.
//
// Roles (416 threads): warps 0-7 produce stages, warp 8 issues tcgen05.mma
// (lane 0) and owns TMEM, warps 9-12 drain TMEM (epilogue; warp%4 = lane quarter).
// ===========================================================================
// Optional role-timing instrumentation (compile with -DPNX_TC_TRACE): per CTA,
// [0] MMA waits on full stages, [1] MMA waits on TMEM-empty, [2] producer waits
// on empty stages (warp 0), [3] epilogue busy cycles (warp 9), [4] kernel cycles.
#ifdef PNX_TC_TRACE
__device__ unsigned long long g_tc_trace[8];
#define TC_T0() long long _t0 = clock64()
#define TC_ACC(i) atomicAdd(&g_tc_trace[i], (unsigned long long)(clock64() - _t0))
#else
#define TC_T0()
#define TC_ACC(i)
#endif
constexpr int TC2_THREADS = 416;
constexpr int TCW_THREADS = 704;  // 16 converter + MMA + loader + 4 epilogue warps
constexpr int TC3_THREADS = 544;  // 8 producer + 1 MMA + 8 epilogue warps
constexpr int TC2_PROD = 256;

template <int NF>
struct Tc2FwdCfg {
    static constexpr int A_T = TC_TILE_BYTES;  // 128 rows x 8 fp32
    static constexpr int B_T = NF * 32;
    static constexpr int STAGE = 2 * A_T + 2 * B_T;
    static constexpr int NST = (TC_SMEM - 1024) / STAGE > 8 ? 8 : (TC_SMEM - 1024) / STAGE;
    static constexpr int NBUF = 4 * NF <= 512 ? 2 : 1;  // TMEM buffers of (big | small)
};

// forward: Z_out[p] = act(Z_in)[p] W + [p==0] b, one stream p per pass.
//
// Memory access is organised around 128 B lines (the L1 request rate, not DRAM
// bandwidth, bounded the first version): producers read a 32-feature group
// (4 MMA k-steps) per row with 8 lanes per line and write it into four stages;
// the epilogue transposes each warp's 32 rows x 32 columns through a padded
// smem tile so global stores are full-line as well.
template <int NF>
struct Tc3FwdCfg {
    static constexpr int A_T = TC_TILE_BYTES;
    static constexpr int B_T = NF * 32;
    static constexpr int STAGE = 2 * A_T + 2 * B_T;
    static constexpr int EPI_ROW = 144;                     // 128 B + 16 B pad
    static constexpr int EPI_BYTES = 8 * 32 * EPI_ROW;      // 8 epilogue warps
    static constexpr int NST = (TC_SMEM + 20 * 1024 - 1024 - EPI_BYTES) / STAGE > 8
                                   ? 8
                                   : (TC_SMEM + 20 * 1024 - 1024 - EPI_BYTES) / STAGE;
    static constexpr int NBUF = 4 * NF <= 512 ? 2 : 1;
    static constexpr int SMEM = NST * STAGE + EPI_BYTES + 1024;
};

// F16: 3xFP16 operands (kind::f16, K = 16 per stage: two stages per 32-feature
// group), scaled by the recorded bounds like the pair forward.
template <int L, int PRO, int NF, bool F16 = false>
__global__ void __launch_bounds__(TC3_THREADS, 1) k_tc2_fwd(TcGemmArgs g) {
    using St = Streams<L>;
    constexpr int S = St::S;
    using Cfg = Tc3FwdCfg<NF>;
    constexpr int NST = Cfg::NST, NBUF = Cfg::NBUF;
    constexpr bool SECOND = (St::order(S - 1) == 2);  // layout has order-2 streams
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[8], empty[8], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = blockIdx.x * TC_M;
    constexpr int KS = F16 ? 16 : 8, SPG = 32 / KS;  // K per stage, stages per 32-feature group
    const int nkb = g.K / KS, ngrp = g.K / 32;
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * NF;
    // 3xFP16 operand scale exponent of stream p's A (|act(Z_in)[p]| bound)
    auto a_exp = [&](int p) -> int {
        if (PRO != ACT_NONE && p == 0) return tc::f16_scale_exp(1.0f);
        float b = __uint_as_float(g.amax_in[p]);
        if (PRO != ACT_NONE && St::order(p) == 2) {
            const float a = __uint_as_float(g.amax_in[St::partner(p)]);
            b = b + 2.0f * a * a;
        }
        return tc::f16_exp_bits(__float_as_uint(b * 1.001f));
    };
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], 9);  // 8 producer warps + 1 expect_tx
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < NBUF; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], 8);
        }
        tc::fence_barrier_init();
    }
    if (warp == 8) tc::tmem_alloc<512>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t sbase = tc::smem_u32(smem);

    if (warp < 8) {
        // ---------------- producers ----------------
        // lane -> (row quad offset rq = lane/8, 16 B chunk c = lane%8 of a 128 B
        // group line); warp w covers rows 16w .. 16w+15 as rq + 4i, i = 0..3.
        const int rq = lane >> 3, c = lane & 7;
        // k-step of the group this lane feeds and its place in that step's 32 B row:
        // tf32: 4 of 8 features (16 B chunk); fp16: 4 of 16 halves (8 B in a 16 B chunk)
        const int j_own = F16 ? c >> 2 : c >> 1;
        const int kc = (c & 1) * 4;
        const float* base = g.A + (int64_t)(r0 + warp * 16 + rq) * g.K + c * 4;
        uint32_t aoff[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t row = (uint32_t)(warp * 16 + rq + 4 * i);
            aoff[i] = F16 ? tc::sw32_chunk(row, (uint32_t)((c & 3) >> 1)) + (uint32_t)(c & 1) * 8u
                          : tc::sw32_off(row, (uint32_t)kc);
        }
        float4 t4[4], z4[4], p4[SECOND ? 4 : 1];
        auto load = [&](int grp, float4* tt, float4* zz, float4* pp) {
#ifdef PNX_EXP_NOLOAD
#pragma unroll
            for (int i = 0; i < 4; ++i) tt[i] = zz[i] = pp[SECOND ? i : 0] = make_float4(0.1f * grp, 0.2f, 0.3f, 0.4f);
            return;
#endif
            const int p = grp / ngrp, off = (grp % ngrp) * 32;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float* q = base + (int64_t)(4 * i) * g.K + off;
                if constexpr (PRO == ACT_NONE) {
                    tt[i] = ldg4(q + p * RK);
                } else {
                    tt[i] = ldg4(q);
                    if (p > 0) zz[i] = ldg4(q + p * RK);
                    if constexpr (SECOND) {
                        if (St::order(p) == 2) pp[i] = ldg4(q + St::partner(p) * RK);
                    }
                }
            }
        };
        const int ngt = S * ngrp;
        load(0, t4, z4, p4);
        for (int gi = 0; gi < ngt; ++gi) {
            float4 tc4[4], zc4[4], pc4[SECOND ? 4 : 1];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                tc4[i] = t4[i];
                zc4[i] = z4[i];
                if constexpr (SECOND) pc4[i] = p4[i];
            }
            if (gi + 1 < ngt) load(gi + 1, t4, z4, p4);  // prefetch one group ahead
            const int p = gi / ngrp;
            const float sc = F16 ? ldexpf(1.0f, a_exp(p)) : 1.0f;
            // activation + split for this lane's 4 rows (used at stage j_own)
            float4 hi[4], lo[4];
            uint2 hi16[4], lo16[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float4 h;
                if constexpr (PRO == ACT_NONE) {
                    h = tc4[i];
                } else {
                    const float4 t = tc4[i], z = zc4[i];
                    if (p == 0) {
                        h = t;
                    } else if (St::order(p) == 1) {
                        h = make_float4((1.f - t.x * t.x) * z.x, (1.f - t.y * t.y) * z.y, (1.f - t.z * t.z) * z.z,
                                        (1.f - t.w * t.w) * z.w);
                    } else {
                        float4 za = make_float4(0.f, 0.f, 0.f, 0.f);
                        if constexpr (SECOND) za = pc4[i];
                        h = make_float4((1.f - t.x * t.x) * (z.x - 2.f * t.x * za.x * za.x),
                                        (1.f - t.y * t.y) * (z.y - 2.f * t.y * za.y * za.y),
                                        (1.f - t.z * t.z) * (z.z - 2.f * t.z * za.z * za.z),
                                        (1.f - t.w * t.w) * (z.w - 2.f * t.w * za.w * za.w));
                    }
                }
                if constexpr (F16) {
                    tc::split_h2(h.x * sc, h.y * sc, hi16[i].x, lo16[i].x);
                    tc::split_h2(h.z * sc, h.w * sc, hi16[i].y, lo16[i].y);
                } else {
                    split4(h, hi[i], lo[i]);
                }
            }
#pragma unroll
            for (int j = 0; j < SPG; ++j) {
                const int it = gi * SPG + j, st = it % NST, kb = it % nkb;
                const uint32_t stage = sbase + st * Cfg::STAGE;
                {
                    TC_T0();
                    tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                    if (tid == 0) TC_ACC(2);
                }
                if (tid == 0) {
#ifdef PNX_EXP_NOB
                    tc::mbar_arrive(&full[st]);
                    (void)kb;
#else
                    tc::mbar_arrive_expect_tx(&full[st], 2 * Cfg::B_T);
                    tc::bulk_g2s(stage + 2 * Cfg::A_T, g.img + (int64_t)kb * (2 * Cfg::B_T / 4), 2 * Cfg::B_T,
                                 &full[st]);
#endif
                }
                if (j == j_own) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if constexpr (F16) {
                            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(stage + aoff[i]), "r"(hi16[i].x),
                                         "r"(hi16[i].y));
                            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(stage + Cfg::A_T + aoff[i]),
                                         "r"(lo16[i].x), "r"(lo16[i].y));
                        } else {
                            sts128(stage + aoff[i], hi[i]);
                            sts128(stage + Cfg::A_T + aoff[i], lo[i]);
                        }
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&full[st]);
            }
        }
    } else if (warp == 8) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = F16 ? tc::make_idesc_f16(TC_M, NF, 0, 0) : tc::make_idesc_tf32(TC_M, NF, 0, 0);
            for (int p = 0; p < S; ++p) {
                const int buf = p % NBUF, use = p / NBUF;
                {
                    TC_T0();
                    tc::mbar_wait(&tempty[buf], ((uint32_t)use & 1u) ^ 1u);
                    TC_ACC(1);
                }
                tc::tc_fence_after();
                const uint32_t dbig = tmem + (uint32_t)(buf * 2 * NF), dsmall = dbig + NF;
                for (int kb = 0; kb < nkb; ++kb) {
                    const int it = p * nkb + kb, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                        TC_ACC(0);
                    }
                    tc::tc_fence_after();
                    const uint64_t ah = tc::make_sdesc(stage, 16, 256, 6), al = tc::make_sdesc(stage + Cfg::A_T, 16, 256, 6);
                    const uint64_t bh = tc::make_sdesc(stage + 2 * Cfg::A_T, 16, 256, 6);
                    const uint64_t bl = tc::make_sdesc(stage + 2 * Cfg::A_T + Cfg::B_T, 16, 256, 6);
                    if constexpr (F16) {
                        tc::mma_f16(dbig, ah, bh, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_f16(dsmall, ah, bl, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_f16(dsmall, al, bh, idesc, 1u);
                    } else {
                        tc::mma_tf32(dbig, ah, bh, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_tf32(dsmall, ah, bl, idesc, kb > 0 ? 1u : 0u);
                        tc::mma_tf32(dsmall, al, bh, idesc, 1u);
                    }
                    tc::mma_commit(&empty[st]);
                }
                tc::mma_commit(&tfull[buf]);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (8 warps: lane quarter warp%4, column half) ----------------
        const int q = warp & 3, half = (warp - 9) >> 2;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t stg = sbase + NST * Cfg::STAGE + (uint32_t)(warp - 9) * 32 * Cfg::EPI_ROW;
        for (int p = 0; p < S; ++p) {
            const int buf = p % NBUF, use = p / NBUF;
            float mx = 0.0f;  // |z| bound of this stream (consumers' 3xFP16 scales)
            const float usA = F16 ? ldexpf(1.0f, -a_exp(p)) : 1.0f;
            const float usW = F16 ? ldexpf(1.0f, -tc::f16_exp_bits(*g.amax_w)) : 1.0f;
            tc::mbar_wait(&tfull[buf], (uint32_t)use & 1u);
            tc::tc_fence_after();
            TC_T0();
#pragma unroll 1
            for (int c = half * (NF / 2); c < (half + 1) * (NF / 2); c += 32) {
                float a[32], b[32];
                tc::tmem_ld16(tl + (uint32_t)(buf * 2 * NF + c), a);
                tc::tmem_ld16(tl + (uint32_t)(buf * 2 * NF + c + 16), a + 16);
                tc::tmem_ld16(tl + (uint32_t)(buf * 2 * NF + NF + c), b);
                tc::tmem_ld16(tl + (uint32_t)(buf * 2 * NF + NF + c + 16), b + 16);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] += b[j];
                if constexpr (F16) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) a[j] = a[j] * usA * usW;
                }
                if (p == 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) a[j] = store_value<ACT_TANH>(a[j] + __ldg(g.bias + c + j));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fabsf(a[j]));
                }
                // row `lane` of this warp's 32 x 32 block -> padded smem
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    sts128(stg + lane * Cfg::EPI_ROW + j * 4, make_float4(a[j], a[j + 1], a[j + 2], a[j + 3]));
                __syncwarp();
                // full-line stores: instruction k writes rows 4k .. 4k+3 (8 lanes x 16 B each)
                float* dst = g.out + p * RN + (int64_t)(r0 + q * 32) * NF + c;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int rr = 4 * k + (lane >> 3), cc = (lane & 7) * 4;
                    float4 v;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                                 : "r"(stg + rr * Cfg::EPI_ROW + cc * 4));
#ifdef PNX_EXP_NOSTORE
                    if (v.x == 12345.f)
#endif
                    *reinterpret_cast<float4*>(dst + (int64_t)rr * NF + cc) = v;
                }
                __syncwarp();
            }
            if (p > 0 && g.amax_out) tc::warp_amax(g.amax_out + p, __float_as_uint(mx));
            tc::tc_fence_before();
            __syncwarp();
            if (warp == 9 && lane == 0) TC_ACC(3);
            if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 8) tc::tmem_dealloc<512>(tmem);
}

// Forward, CTA pair (NF = 256): a 2-CTA cluster owns 256 rows; the leader issues
// M=256 x N=256 cta_group::2 MMAs, each CTA holding its 128 rows of A and
// HALF of the weight columns (B), so per-SM weight traffic and operand smem
// reads drop by a third. Per CTA:
//   warp 8  : TMEM owner; lane 0 streams raw A (32-feature x 128-row boxes of the
//             streams a pass needs, 128 B swizzled) into a ring by tensor-map TMA
//   warp 17 : lane 0 streams this CTA's weight-image half into the MMA stages,
//             completing on the leader's full barrier (.cta_group::2 TMA)
//   warps 0-7  : converters -- jet activation + hi/lo split of a whole 4-k-step
//                group per thread, SW32 stores, one proxy fence per group
//   warps 9-16 : epilogue
//   warp 18 : lane 0 of the leader issues the MMAs
template <int L>
struct Tc4FwdCfg {
    using St = Streams<L>;
    static constexpr bool SECOND = St::order(St::S - 1) == 2;
    static constexpr int NF = 256, NFL = 128;
    static constexpr int A_T = TC_TILE_BYTES;  // 128 rows x 8 fp32
    static constexpr int B_T = NFL * 32;       // 128 weight columns x 8 fp32
    static constexpr int STAGE = 2 * A_T + 2 * B_T;
    static constexpr int BOX = 128 * 32 * 4;   // 128 rows x 32 features
    static constexpr int NBOX = SECOND ? 3 : 2;
    static constexpr int RAW = NBOX * BOX;
    // raw ring depth: 3 groups in flight for first-order layouts (2 for second-order,
    // whose 3-box groups leave no room); tools/trace_fwd4.cu: 3 slots + the MMA warp
    // cut the 3xFP16 forward by 5.5%
    static constexpr int NR = SECOND ? 2 : 3;
    static constexpr int EPI_TILE = 32 * 128;       // 32 rows x 32 fp32, 128 B swizzled (TMA store box)
    static constexpr int EPI_BYTES = 8 * 2 * EPI_TILE;  // 8 warps x 2 buffers
    static constexpr int BUDGET = 226 * 1024;
    static constexpr int NST0 = (BUDGET - NR * RAW - EPI_BYTES) / STAGE;
    static constexpr int NST = NST0 > 8 ? 8 : NST0;
    static constexpr int SMEM = NR * RAW + NST * STAGE + EPI_BYTES + 1024;
    static_assert(NST >= 4, "forward stage ring");
};
// warp 18 issues the MMAs, so stream p+1 starts as soon as the epilogue warps
// have read stream p's accumulators (not after an epilogue warp's own stores)
constexpr int TC4_THREADS = 608;  // 19 warps

// F16: 3xFP16 operands (kind::f16, K = 16 per stage) scaled by the recorded
// bounds g.amax_in / g.amax_w; the epilogue unscales and records g.amax_out.
template <int L, int PRO, bool F16 = false>
__global__ void __launch_bounds__(TC4_THREADS, 1) k_tc4_fwd(const __grid_constant__ TcGemmArgs g) {
    using St = Streams<L>;
    constexpr int S = St::S;
    using Cfg = Tc4FwdCfg<L>;
    constexpr int NST = Cfg::NST, NR = Cfg::NR, NF = Cfg::NF, NFL = Cfg::NFL;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[8], empty[8], rfull[NR], rempty[NR], tfull, tempty;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = tc::cluster_ctarank();
    // persistent: pair `pair` owns 256-row tiles pair, pair + npairs, ...; every ring
    // and accumulator barrier keeps counting across tiles, so the converters and
    // loaders run into the next tile while the epilogue drains the previous one
    const int npairs = (int)(gridDim.x >> 1), pair = (int)(blockIdx.x >> 1), ntiles = g.Rpad / 256;
    const int nloc = pair < ntiles ? (ntiles - 1 - pair) / npairs + 1 : 0;
    auto row0 = [&](int i) { return (pair + i * npairs) * 256 + (int)rank * 128; };
    constexpr int KS = F16 ? 16 : 8;   // K per stage (one MMA)
    constexpr int SPG = 32 / KS;       // stages per 32-feature raw group
    const int nkb = g.K / KS, ngrp = g.K / 32;
    // 3xFP16 operand scale exponent of stream p's A (|act(Z_in)[p]| bound)
    auto a_exp = [&](int p) -> int {
        if (PRO != ACT_NONE && p == 0) return tc::f16_scale_exp(1.0f);
        float b = __uint_as_float(g.amax_in[p]);
        if (PRO != ACT_NONE && St::order(p) == 2) {
            const float a = __uint_as_float(g.amax_in[St::partner(p)]);
            b = b + 2.0f * a * a;
        }
        return tc::f16_exp_bits(__float_as_uint(b * 1.001f));
    };
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], 17);  // 2 x 8 converter warps + the leader's expect_tx
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < NR; ++i) {
            tc::mbar_init(&rfull[i], 1);
            tc::mbar_init(&rempty[i], 8);
        }
        tc::mbar_init(&tfull, 1);
        tc::mbar_init(&tempty, 16);
        tc::fence_barrier_init();
    }
    if (warp == 8) tc::tmem_alloc_pair<512>(&tmem_base);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t sraw = tc::smem_u32(smem);
    const uint32_t sbase = sraw + NR * Cfg::RAW;
    const uint32_t sepi = sbase + NST * Cfg::STAGE;
    const uint32_t full0 = tc::mapa(tc::smem_u32(&full[0]), 0);
    const uint32_t tempty0 = tc::mapa(tc::smem_u32(&tempty), 0);
    // raw boxes a pass needs: [0] = stream 0 (t), [1] = stream p, [2] = partner
    auto nbox = [](int p) { return PRO == ACT_NONE ? 1 : (p == 0 ? 1 : (St::order(p) == 2 ? 3 : 2)); };

    // MMAs of the ps-th (tile, stream) item (one elected thread of the pair leader)
    auto issue_stream = [&](int ps) {
        constexpr uint32_t idesc =
            F16 ? tc::make_idesc_f16(2 * TC_M, NF, 0, 0) : tc::make_idesc_tf32(2 * TC_M, NF, 0, 0);
        {
            TC_T0();
            tc::mbar_wait(&tempty, ((uint32_t)ps & 1u) ^ 1u);
            TC_ACC(1);
        }
        tc::tc_fence_after();
        const uint32_t dbig = tmem, dsmall = tmem + NF;
        for (int kb = 0; kb < nkb; ++kb) {
            const int it = ps * nkb + kb, st = it % NST;
            const uint32_t stage = sbase + st * Cfg::STAGE;
            {
                TC_T0();
                tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                TC_ACC(0);
            }
            tc::tc_fence_after();
            const uint64_t ah = tc::make_sdesc(stage, 16, 256, 6), al = tc::make_sdesc(stage + Cfg::A_T, 16, 256, 6);
            const uint64_t bh = tc::make_sdesc(stage + 2 * Cfg::A_T, 16, 256, 6);
            const uint64_t bl = tc::make_sdesc(stage + 2 * Cfg::A_T + Cfg::B_T, 16, 256, 6);
            if constexpr (F16) {
                tc::mma_f16_pair(dbig, ah, bh, idesc, kb > 0 ? 1u : 0u);
                tc::mma_f16_pair(dsmall, ah, bl, idesc, kb > 0 ? 1u : 0u);
                tc::mma_f16_pair(dsmall, al, bh, idesc, 1u);
            } else {
                tc::mma_tf32_pair(dbig, ah, bh, idesc, kb > 0 ? 1u : 0u);
                tc::mma_tf32_pair(dsmall, ah, bl, idesc, kb > 0 ? 1u : 0u);
#ifndef PNX_EXP_TWO_MMA  // timing experiment only: drops a product
                tc::mma_tf32_pair(dsmall, al, bh, idesc, 1u);
#endif
            }
            tc::mma_commit_pair(&empty[st], 3);
        }
        tc::mma_commit_pair(&tfull, 3);
    };

    if (warp < 8) {
        // ---------------- converters ----------------
        const int row = tid >> 1, c = tid & 1;
        const uint32_t aoff = tc::sw32_off((uint32_t)row, (uint32_t)(c * 4));
        const uint32_t rrow = (uint32_t)row * 128;
        const uint32_t rsw = (uint32_t)(row & 7);
        // activation jet of stream p for the 4 features in raw 16 B chunk `off`
        auto act_h = [&](uint32_t raw, uint32_t off, int p) -> float4 {
            if (PRO == ACT_NONE || p == 0) return lds128(raw + off);
            const float4 t = lds128(raw + off), z = lds128(raw + Cfg::BOX + off);
            if (St::order(p) == 1)
                return make_float4((1.f - t.x * t.x) * z.x, (1.f - t.y * t.y) * z.y, (1.f - t.z * t.z) * z.z,
                                   (1.f - t.w * t.w) * z.w);
            const float4 za = lds128(raw + 2 * Cfg::BOX + off);
            return make_float4((1.f - t.x * t.x) * (z.x - 2.f * t.x * za.x * za.x),
                               (1.f - t.y * t.y) * (z.y - 2.f * t.y * za.y * za.y),
                               (1.f - t.z * t.z) * (z.z - 2.f * t.z * za.z * za.z),
                               (1.f - t.w * t.w) * (z.w - 2.f * t.w * za.w * za.w));
        };
        for (int ps = 0; ps < nloc * S; ++ps) {
            const int p = ps % S;
            const float sc = F16 ? ldexpf(1.0f, a_exp(p)) : 1.0f;
            for (int gi = 0; gi < ngrp; ++gi) {
                const int gq = ps * ngrp + gi, rs = gq % NR;
                const uint32_t raw = sraw + rs * Cfg::RAW;
                {
                    TC_T0();
                    tc::mbar_wait(&rfull[rs], (uint32_t)(gq / NR) & 1u);
                    if (tid == 0) TC_ACC(5);
                }
                if constexpr (F16) {
                    // stage j = features [16j, 16j+16) of the group; this thread: chunk c
                    uint4 hi[2], lo[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        float h[8];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const float4 v = act_h(raw, rrow + ((((uint32_t)(4 * j + 2 * c + u)) ^ rsw) << 4), p);
                            h[4 * u] = v.x;
                            h[4 * u + 1] = v.y;
                            h[4 * u + 2] = v.z;
                            h[4 * u + 3] = v.w;
                        }
                        tc::split_h8(h, sc, hi[j], lo[j]);
                    }
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&rempty[rs]);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int it = gq * 2 + j, st = it % NST;
                        const uint32_t stage = sbase + st * Cfg::STAGE;
                        TC_T0();
                        tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        if (tid == 0) TC_ACC(2);
                        sts128u(stage + aoff, hi[j]);
                        sts128u(stage + Cfg::A_T + aoff, lo[j]);
                    }
                } else {
                    float4 hi[4], lo[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        split4(act_h(raw, rrow + ((((uint32_t)(2 * j + c)) ^ rsw) << 4), p), hi[j], lo[j]);
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&rempty[rs]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int it = gq * 4 + j, st = it % NST;
                        const uint32_t stage = sbase + st * Cfg::STAGE;
                        tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        sts128(stage + aoff, hi[j]);
                        sts128(stage + Cfg::A_T + aoff, lo[j]);
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < SPG; ++j) tc::mbar_arrive_cluster(full0 + ((gq * SPG + j) % NST) * 8);
                }
            }
        }
    } else if (warp == 8) {
        // ---------------- raw A loader ----------------
        if (lane == 0) {
            for (int ps = 0; ps < nloc * S; ++ps) {
                const int p = ps % S, r0 = row0(ps / S);
                const int nb = nbox(p);
                const int s1 = PRO == ACT_NONE ? p : 0;
                for (int gi = 0; gi < ngrp; ++gi) {
                    const int gq = ps * ngrp + gi, rs = gq % NR;
                    const uint32_t raw = sraw + rs * Cfg::RAW;
                    tc::mbar_wait(&rempty[rs], ((uint32_t)(gq / NR) & 1u) ^ 1u);
                    tc::mbar_arrive_expect_tx(&rfull[rs], nb * Cfg::BOX);
                    tc::tma_load_3d(raw, &g.tmA, gi * 32, r0, s1, &rfull[rs]);
                    if (nb > 1) tc::tma_load_3d(raw + Cfg::BOX, &g.tmA, gi * 32, r0, p, &rfull[rs]);
                    if (nb > 2) tc::tma_load_3d(raw + 2 * Cfg::BOX, &g.tmA, gi * 32, r0, St::partner(p), &rfull[rs]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 17) {
        // ---------------- weight-half loader ----------------
        if (lane == 0) {
            const int nit = nloc * S * nkb;
            for (int it = 0; it < nit; ++it) {
                const int st = it % NST, kb = it % nkb;
                const uint32_t stage = sbase + st * Cfg::STAGE;
                tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                if (rank == 0) tc::mbar_arrive_expect_tx(&full[st], 2 * 2 * Cfg::B_T);
                const int rowb = kb * 2 * NF + (int)rank * NFL;  // image rows (8 fp32 each)
                tc::tma_load_2d_pair(stage + 2 * Cfg::A_T, &g.tmB, 0, rowb, full0 + st * 8);
                tc::tma_load_2d_pair(stage + 2 * Cfg::A_T + Cfg::B_T, &g.tmB, 0, rowb + NF, full0 + st * 8);
            }
        }
        __syncwarp();
    } else if (warp == 18) {
        if (lane == 0 && rank == 0)
            for (int ps = 0; ps < nloc * S; ++ps) issue_stream(ps);
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 9-16) ----------------
        // Epilogue: TMEM -> registers -> 128 B-swizzled staging tile (row r, 16 B chunk c
        // at r*128 + ((c ^ r%8) << 4): conflict-free) -> one TMA tensor store per
        // 32 x 32 block; TMEM is released as soon as it is read, the stores drain
        // asynchronously (double-buffered staging, bulk_wait_read before reuse).
        const int q = warp & 3, half = (warp - 9) >> 2;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t stg0 = sepi + (uint32_t)(warp - 9) * 2 * Cfg::EPI_TILE;
        int nst = 0;  // stores issued by this warp (buffer = nst & 1)
        for (int ps = 0; ps < nloc * S; ++ps) {
            const int p = ps % S, r0 = row0(ps / S);
            // 3xFP16 unscale 2^-(eA+eW): one multiply while the power of two is a normal
            // float (always, in practice), else two
            float usA = 1.0f, usW = 1.0f;
            if constexpr (F16) {
                const int e = a_exp(p) + tc::f16_exp_bits(*g.amax_w);
                if (e > -120 && e < 120) {
                    usA = ldexpf(1.0f, -e);
                } else {
                    usA = ldexpf(1.0f, -a_exp(p));
                    usW = ldexpf(1.0f, -tc::f16_exp_bits(*g.amax_w));
                }
            }
            float mx = 0.0f;  // |z| bound of this stream (fmax with |.|: one FMNMX per element)
            tc::mbar_wait(&tfull, (uint32_t)ps & 1u);
            tc::tc_fence_after();
            TC_T0();
#pragma unroll 1
            for (int c = half * (NF / 2); c < (half + 1) * (NF / 2); c += 32) {
                float a[32], b[32];
                tc::tmem_ld16(tl + (uint32_t)c, a);
                tc::tmem_ld16(tl + (uint32_t)(c + 16), a + 16);
                tc::tmem_ld16(tl + (uint32_t)(NF + c), b);
                tc::tmem_ld16(tl + (uint32_t)(NF + c + 16), b + 16);
                tc::tmem_ld_wait();
                if (c + 32 >= (half + 1) * (NF / 2)) {  // last TMEM read of this pass: release it
                    tc::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(tempty0);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] += b[j];
                if constexpr (F16) {
                    if (usW != 1.0f) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) a[j] = a[j] * usA * usW;
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) a[j] *= usA;
                    }
                }
                if (p == 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) a[j] = store_value<ACT_TANH>(a[j] + __ldg(g.bias + c + j));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fabsf(a[j]));
                }
                const uint32_t stg = stg0 + (uint32_t)(nst & 1) * Cfg::EPI_TILE;
                if (lane == 0) tc::bulk_wait_read<1>();  // the store that last used this buffer has read it
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    sts128(stg + lane * 128 + (((uint32_t)j ^ (uint32_t)(lane & 7)) << 4),
                           make_float4(a[4 * j], a[4 * j + 1], a[4 * j + 2], a[4 * j + 3]));
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tc::tma_store_3d(&g.tmO, c, r0 + q * 32, p, stg);
                    tc::bulk_commit();
                }
                ++nst;
            }
            if (p > 0 && g.amax_out) tc::warp_amax(g.amax_out + p, __float_as_uint(mx));
            if (warp == 9 && lane == 0) TC_ACC(3);
        }
        if (lane == 0) tc::bulk_wait<0>();
        __syncwarp();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 8) tc::tmem_dealloc_pair<512>(tmem);
}

// Weight gradient, bulk-fed. One thread (an epilogue warp's lane 0; those warps
// are idle until the accumulators are final) streams raw 8-row blocks of every
// stream -- Z_in rows of this M tile and Zb_out rows -- into a ring with one
// tensor-map TMA per operand, so load latency is covered by the ring depth
// instead of producer registers. Two groups of 8 converter warps take alternate
// k-steps: jet activation of the layer input, hi/lo split, swizzled store.
//
// PAIR (Kin = 256): a 2-CTA cluster covers both 128-feature M tiles of a row
// block with cta_group::2 MMAs (M = 256). Each CTA converts its own A rows and
// HALF of the B columns, so the B work the two single-CTA M tiles used to
// duplicate is shared, and per-SM operand smem reads drop by a third.
template <int S, int NF, bool PAIR>
struct Tc2WgCfg {
    static constexpr int NFL = PAIR ? NF / 2 : NF;  // B columns staged by this CTA
    static constexpr int A_T = 8 * 128 * 4;         // 8 rows x 128 k_in (one stream)
    static constexpr int B_T = 8 * NFL * 4;         // 8 rows x NFL
    static constexpr int STAGE = 2 * A_T + 2 * B_T;
    static constexpr int RAW_A = S * A_T;
    static constexpr int RAW = RAW_A + S * B_T;  // one 8-row block, all streams
    static constexpr int BUDGET = 226 * 1024;
    static constexpr int NR0 = (BUDGET - 4 * STAGE) / RAW;
    static constexpr int NR = NR0 > 4 ? 4 : NR0;
    static constexpr int NST0 = (BUDGET - NR * RAW) / STAGE;
    static constexpr int NST = NST0 > 8 ? 8 : NST0;
    static constexpr int SMEM = NR * RAW + NST * STAGE + 1024;
    static_assert(NR >= 2 && NST >= 2, "weight-gradient rings");
    static_assert(NR * RAW >= 2 * 8 * NFL * 8, "db reduction reuses the raw ring");
};

// F16: 3xFP16 operands. A stage is one kind::f16 K = 16 step: the same 8 rows
// of two streams (k-rows 0-7 stream s, 8-15 stream s+1; a group's odd last
// stream pads with zeros), fp16 MN-major 128 B-swizzled tiles of the same byte
// size as the tf32 ones.
//
// Persistent: CTA group `grp` (one CTA, or the pair / the MT m-tiles of a row
// block) walks the contiguous 8-row blocks [NB*grp/G, NB*(grp+1)/G) and drains
// the "big" accumulator every `segrows` rows into its FP32 slot g.wpart[grp]
// (zeroed before the launch; round-to-nearest red.add, L2-resident: G x Kin x N
// x 4 B), so the FP32 TMEM
// accumulation (which truncates, DESIGN.md §4 accuracy) never spans more than
// `segrows` rows; the "small" accumulator (the hi*lo + lo*hi corrections, 2^-11
// of the result) keeps accumulating over the whole range and joins the slot at
// the end. The MMA issuer pauses only for the big drain; loader and converters
// run ahead through it.
template <int L, int PRO, int NF, bool PAIR, bool F16 = false>
__global__ void __launch_bounds__(TCW_THREADS, 1) k_tc2_wgrad(const __grid_constant__ TcWgradArgs g, int segrows,
                                                             int G) {
    using St = Streams<L>;
    constexpr int S = St::S;
    constexpr int SG = (S + 1) / 2;                                   // streams of converter group 0
    constexpr int NSTG = F16 ? (SG + 1) / 2 + (S - SG + 1) / 2 : S;  // MMA stages per 8-row block
    using Cfg = Tc2WgCfg<S, NF, PAIR>;
    constexpr int NST = Cfg::NST, NR = Cfg::NR, NFL = Cfg::NFL;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[8], empty[8], rfull[4], rempty[4], tfull, tempty;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int MT = g.Kin / 128;
    const int tile = blockIdx.x / MT, mt = blockIdx.x % MT;  // group; PAIR: mt == cluster rank
    const int NB = g.Rpad / 8;
    const int blk0 = (int)((int64_t)NB * tile / G), blk1 = (int)((int64_t)NB * (tile + 1) / G);
    const int rbeg = blk0 * 8;
    const int nblk = blk1 - blk0;
    const int nit = nblk * NSTG;
    const int segit = (segrows / 8) * NSTG;  // MMA k-steps per big-accumulator segment
    const int nseg = (nit + segit - 1) / segit;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], PAIR ? 16 : 8);  // the converter group(s) filling stage i
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < NR; ++i) {
            tc::mbar_init(&rfull[i], 1);
            tc::mbar_init(&rempty[i], 16);
        }
        tc::mbar_init(&tfull, 1);
        tc::mbar_init(&tempty, PAIR ? 8 : 4);  // the epilogue warps (of both CTAs) drained big
        tc::fence_barrier_init();
    }
    if (warp == 16) {
        if constexpr (PAIR) tc::tmem_alloc_pair<512>(&tmem_base);
        else tc::tmem_alloc<512>(&tmem_base);
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t sraw = tc::smem_u32(smem);
    const uint32_t sbase = sraw + NR * Cfg::RAW;
    // F16: operand scales 2^sA, 2^sB from the largest per-stream bound
    // (|act(z)[s]| <= 1 (value), |z_s| (first order), |z_aa| + 2 z_a^2 (second))
    int sA = 0, sB = 0;
    if constexpr (F16) {
        float ma = 0.0f, mb = 0.0f;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            float b = __uint_as_float(g.amaxA[s]);
            if (PRO != ACT_NONE && s == 0) b = 1.0f;
            if (PRO != ACT_NONE && St::order(s) == 2) {
                const float a = __uint_as_float(g.amaxA[St::partner(s)]);
                b = b + 2.0f * a * a;
            }
            ma = fmaxf(ma, b);
            mb = fmaxf(mb, __uint_as_float(g.amaxB[s]));
        }
        sA = tc::f16_exp_bits(__float_as_uint(ma * 1.001f));
        sB = tc::f16_exp_bits(__float_as_uint(mb));
    }
    const float scA = ldexpf(1.0f, sA), scB = ldexpf(1.0f, sB);

    if (warp < 16) {
        // A: thread -> (row ar, features 4*ac); B: up to 2 chunks of 4 columns
        const int grp = tid >> 8, gtid = tid & 255;
        const int ar = gtid >> 5, ac = gtid & 31;
        const uint32_t aoff = tc::mn32_off((uint32_t)ar, (uint32_t)(ac * 4), 128u);
        const uint32_t araw = (uint32_t)((ar * 128 + ac * 4) * 4);
        constexpr int BCH = NFL / 4;  // float4 chunks per row
        constexpr int NB = (8 * BCH + 255) / 256;
        int brow[2];
        uint32_t boff[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int idx = gtid + 256 * j;
            brow[j] = j < NB ? idx / BCH : 8;
            boff[j] = tc::mn32_off((uint32_t)(brow[j] & 7), (uint32_t)((idx % BCH) * 4), (uint32_t)NFL);
        }
        const uint32_t full0 = PAIR ? tc::mapa(tc::smem_u32(&full[0]), 0) : tc::smem_u32(&full[0]);
        double dbacc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        for (int b = 0; b < nblk; ++b) {
            const int rs = b % NR;
            const uint32_t raw = sraw + rs * Cfg::RAW;
            {
                TC_T0();
                tc::mbar_wait(&rfull[rs], (uint32_t)(b / NR) & 1u);
                if (tid == 0) TC_ACC(1);
            }
            const float4 t = lds128(raw + araw);
            // group 0 converts streams [0, SG), group 1 streams [SG, S) of this
            // block: independent k-steps interleave (ILP) and share one fence
            auto convert = [&](auto lo_c, auto hi_c) {
                constexpr int SLO = decltype(lo_c)::value, SHI = decltype(hi_c)::value, NS = SHI - SLO;
#ifdef PNX_TC_TRACE
                long long _tc = clock64();
#endif
                float4 ahi[NS], bhi[NS][2];
                [[maybe_unused]] float4 alo[NS], blo[NS][2];  // tf32 split only
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    const int s = SLO + i;
                    float4 h;
                    if constexpr (PRO == ACT_NONE) {
                        h = s == 0 ? t : lds128(raw + s * Cfg::A_T + araw);
                    } else if (s == 0) {
                        h = t;
                    } else {
                        const float4 z = lds128(raw + s * Cfg::A_T + araw);
                        const int par = St::partner(s);
                        if (par < 0) {
                            h = make_float4((1.f - t.x * t.x) * z.x, (1.f - t.y * t.y) * z.y,
                                            (1.f - t.z * t.z) * z.z, (1.f - t.w * t.w) * z.w);
                        } else {
                            const float4 za = lds128(raw + par * Cfg::A_T + araw);
                            h = make_float4((1.f - t.x * t.x) * (z.x - 2.f * t.x * za.x * za.x),
                                            (1.f - t.y * t.y) * (z.y - 2.f * t.y * za.y * za.y),
                                            (1.f - t.z * t.z) * (z.z - 2.f * t.z * za.z * za.z),
                                            (1.f - t.w * t.w) * (z.w - 2.f * t.w * za.w * za.w));
                        }
                    }
                    if constexpr (F16) ahi[i] = h;
                    else split4(h, ahi[i], alo[i]);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        if (brow[j] >= 8) continue;
                        const float4 bv = lds128(raw + Cfg::RAW_A + s * Cfg::B_T + (gtid + 256 * j) * 16);
                        if (s == 0) {
                            dbacc[j][0] += bv.x;
                            dbacc[j][1] += bv.y;
                            dbacc[j][2] += bv.z;
                            dbacc[j][3] += bv.w;
                        }
                        if constexpr (F16) bhi[i][j] = bv;
                        else split4(bv, bhi[i][j], blo[i][j]);
                    }
                }
#ifdef PNX_TC_TRACE
                if (tid == 0) atomicAdd(&g_tc_trace[5], (unsigned long long)(clock64() - _tc));
#endif
                if constexpr (F16) {
                    // stage (b, SOFF + i/2): k-rows 8*(i&1) + row of stream SLO + i
                    constexpr int SOFF = SLO == 0 ? 0 : (SG + 1) / 2;
                    auto st_h = [](uint32_t addr, float4 v, float sc, uint32_t lo_addr) {
                        uint32_t h0, l0, h1, l1;
                        tc::split_h2(v.x * sc, v.y * sc, h0, l0);
                        tc::split_h2(v.z * sc, v.w * sc, h1, l1);
                        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(h0), "r"(h1));
                        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(lo_addr), "r"(l0), "r"(l1));
                    };
                    auto st_z = [](uint32_t addr) {
                        asm volatile("st.shared.v2.b32 [%0], {%1, %1};" ::"r"(addr), "r"(0u));
                    };
#pragma unroll
                    for (int i = 0; i < NS; ++i) {
                        const int it = b * NSTG + SOFF + (i >> 1), st = it % NST, pos = i & 1;
                        const uint32_t stage = sbase + st * Cfg::STAGE;
                        if (pos == 0) tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        // (ahi, alo) hold the unsplit values in the F16 mode
                        const uint32_t ao = tc::mn16_off((uint32_t)(ar + 8 * pos), (uint32_t)(ac * 4), 128u);
                        st_h(stage + ao, ahi[i], scA, stage + Cfg::A_T + ao);
                        const bool pad = pos == 0 && i + 1 == NS;  // odd tail: zero k-rows 8-15
                        if (pad) {
                            const uint32_t az = tc::mn16_off((uint32_t)(ar + 8), (uint32_t)(ac * 4), 128u);
                            st_z(stage + az);
                            st_z(stage + Cfg::A_T + az);
                        }
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            if (brow[j] >= 8) continue;
                            const int idx = gtid + 256 * j;
                            const uint32_t bo = tc::mn16_off((uint32_t)(brow[j] + 8 * pos), (uint32_t)((idx % BCH) * 4),
                                                             (uint32_t)NFL);
                            st_h(stage + 2 * Cfg::A_T + bo, bhi[i][j], scB, stage + 2 * Cfg::A_T + Cfg::B_T + bo);
                            if (pad) {
                                const uint32_t bz = tc::mn16_off((uint32_t)(brow[j] + 8), (uint32_t)((idx % BCH) * 4),
                                                                 (uint32_t)NFL);
                                st_z(stage + 2 * Cfg::A_T + bz);
                                st_z(stage + 2 * Cfg::A_T + Cfg::B_T + bz);
                            }
                        }
                    }
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int i = 0; i < NS; i += 2) {
                            const int st = (b * NSTG + SOFF + (i >> 1)) % NST;
                            if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                            else tc::mbar_arrive(&full[st]);
                        }
                    }
                } else {
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    const int it = b * S + SLO + i;
                    const int st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        if (tid == 0) TC_ACC(2);
                    }
#ifdef PNX_TC_TRACE
                    _tc = clock64();
#endif
                    sts128(stage + aoff, ahi[i]);
                    sts128(stage + Cfg::A_T + aoff, alo[i]);
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        if (brow[j] >= 8) continue;
                        sts128(stage + 2 * Cfg::A_T + boff[j], bhi[i][j]);
                        sts128(stage + 2 * Cfg::A_T + Cfg::B_T + boff[j], blo[i][j]);
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < NS; ++i) {
                        const int st = (b * S + SLO + i) % NST;
                        if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                        else tc::mbar_arrive(&full[st]);
                    }
                }
                }
#ifdef PNX_TC_TRACE
                if (tid == 0) atomicAdd(&g_tc_trace[6], (unsigned long long)(clock64() - _tc));
#endif
            };
            constexpr int SG = (S + 1) / 2;
            if (grp == 0) convert(std::integral_constant<int, 0>{}, std::integral_constant<int, SG>{});
            else convert(std::integral_constant<int, SG>{}, std::integral_constant<int, S>{});
            __syncwarp();  // raw block fully read by this warp
            if (lane == 0) tc::mbar_arrive(&rempty[rs]);
        }
        // db (one CTA per column range): fixed-order sum over [group][row slot],
        // staged in the (now idle: every block was consumed) raw ring
        if (PAIR || mt == 0) {
            double* dbred = reinterpret_cast<double*>(smem);  // [grp][8 row slots][NFL]
            asm volatile("bar.sync 1, 512;");
            for (int i = tid; i < 2 * 8 * NFL; i += 512) dbred[i] = 0.0;
            asm volatile("bar.sync 1, 512;");
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (brow[j] >= 8) continue;
                const int idx = gtid + 256 * j;
                double* d = dbred + (grp * 8 + idx / BCH) * NFL + (idx % BCH) * 4;
                for (int c = 0; c < 4; ++c) d[c] += dbacc[j][c];
            }
            asm volatile("bar.sync 1, 512;");
            const int c0 = PAIR ? mt * NFL : 0;
            for (int n = tid; n < NFL; n += 512) {
                double v[16];
                for (int i = 0; i < 16; ++i) v[i] = dbred[i * NFL + n];
                g.dbpart[(int64_t)tile * NF + c0 + n] =
                    (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
                    (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + (v[14] + v[15])));
            }
        }
    } else {
        // warp 16 lane 0 issues the MMAs, warp 17 lane 0 streams the raw blocks,
        // warps 18-21 drain TMEM (warp % 4 = lane quarter) once per segment
        if (warp == 16 && lane == 0 && (!PAIR || mt == 0)) {
            constexpr uint32_t idesc = tc::make_idesc_tf32(PAIR ? 2 * TC_M : TC_M, NF, 1, 1);
            const uint32_t dbig = tmem, dsmall = tmem + NF;
            for (int it = 0; it < nit; ++it) {
                const int st = it % NST, sit = it % segit;
                if (sit == 0 && it > 0) {  // the epilogue drained the previous segment's big
                    tc::mbar_wait(&tempty, (uint32_t)((it / segit - 1) & 1));
                    tc::tc_fence_after();
                }
                const uint32_t stage = sbase + st * Cfg::STAGE;
                {
                    TC_T0();
                    tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                    TC_ACC(0);
                }
                tc::tc_fence_after();
                const uint32_t accb = sit > 0 ? 1u : 0u, accs = it > 0 ? 1u : 0u;
                const uint64_t ah = tc::make_sdesc(stage, 512, 4 * 512, 1);
                const uint64_t al = tc::make_sdesc(stage + Cfg::A_T, 512, 4 * 512, 1);
                const uint64_t bh = tc::make_sdesc(stage + 2 * Cfg::A_T, 512, (NFL / 32) * 512, 1);
                const uint64_t bl = tc::make_sdesc(stage + 2 * Cfg::A_T + Cfg::B_T, 512, (NFL / 32) * 512, 1);
                if constexpr (F16) {
                    // fp16 MN-major SW128 tiles: LBO 1024 (next 64 MN), SBO = next 8 k-rows
                    constexpr uint32_t idesc16 = tc::make_idesc_f16(PAIR ? 2 * TC_M : TC_M, NF, 1, 1);
                    const uint64_t a16h = tc::make_sdesc(stage, 1024, 2 * 1024, 2);
                    const uint64_t a16l = tc::make_sdesc(stage + Cfg::A_T, 1024, 2 * 1024, 2);
                    const uint64_t b16h = tc::make_sdesc(stage + 2 * Cfg::A_T, 1024, (NFL / 64) * 1024, 2);
                    const uint64_t b16l = tc::make_sdesc(stage + 2 * Cfg::A_T + Cfg::B_T, 1024, (NFL / 64) * 1024, 2);
                    if constexpr (PAIR) {
                        tc::mma_f16_pair(dbig, a16h, b16h, idesc16, accb);
                        tc::mma_f16_pair(dsmall, a16h, b16l, idesc16, accs);
                        tc::mma_f16_pair(dsmall, a16l, b16h, idesc16, 1u);
                        tc::mma_commit_pair(&empty[st], 3);
                    } else {
                        tc::mma_f16(dbig, a16h, b16h, idesc16, accb);
                        tc::mma_f16(dsmall, a16h, b16l, idesc16, accs);
                        tc::mma_f16(dsmall, a16l, b16h, idesc16, 1u);
                        tc::mma_commit(&empty[st]);
                    }
                } else if constexpr (PAIR) {
                    tc::mma_tf32_pair(dbig, ah, bh, idesc, accb);
                    tc::mma_tf32_pair(dsmall, ah, bl, idesc, accs);
                    tc::mma_tf32_pair(dsmall, al, bh, idesc, 1u);
                    tc::mma_commit_pair(&empty[st], 3);
                } else {
                    tc::mma_tf32(dbig, ah, bh, idesc, accb);
                    tc::mma_tf32(dsmall, ah, bl, idesc, accs);
                    tc::mma_tf32(dsmall, al, bh, idesc, 1u);
                    tc::mma_commit(&empty[st]);
                }
                if (sit == segit - 1 || it == nit - 1) {
                    if constexpr (PAIR) tc::mma_commit_pair(&tfull, 3);
                    else tc::mma_commit(&tfull);
                }
            }
        }
        if (warp == 17 && lane == 0) {
            // raw-block loader: two tensor-map copies per 8-row block
            for (int b = 0; b < nblk; ++b) {
                const int rs = b % NR;
                const uint32_t raw = sraw + rs * Cfg::RAW;
                tc::mbar_wait(&rempty[rs], ((uint32_t)(b / NR) & 1u) ^ 1u);
                tc::mbar_arrive_expect_tx(&rfull[rs], Cfg::RAW);
                const int row0 = rbeg + b * 8;
                tc::tma_load_3d(raw, &g.tmA, mt * 128, row0, 0, &rfull[rs]);
                tc::tma_load_3d(raw + Cfg::RAW_A, &g.tmB, PAIR ? mt * NFL : 0, row0, 0, &rfull[rs]);
            }
        }
        if (warp >= 18) {
            const int q = warp & 3;
            const int m = q * 32 + lane;
            const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
            float* dst = g.wpart + ((int64_t)tile * g.Kin + mt * 128 + m) * NF;
            const uint32_t tempty0 = PAIR ? tc::mapa(tc::smem_u32(&tempty), 0) : tc::smem_u32(&tempty);
            float us = 1.0f;
            if constexpr (F16) us = ldexpf(1.0f, -sA) * ldexpf(1.0f, -sB);
            // the slot is re-read by every segment drain: keep it in L2 while the
            // operand stream passes through (ncu: without the hint the slot lines were
            // evicted and written back, ~1 GB of DRAM writes + 1 GB of reads per launch)
            uint64_t keep;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
            for (int seg = 0; seg < nseg; ++seg) {
                const bool last = seg + 1 == nseg;
                tc::mbar_wait(&tfull, (uint32_t)(seg & 1));
                tc::tc_fence_after();
                // big (and, after the last segment, small) in 64-column chunks: four
                // tcgen05.ld in flight per wait, then 16 fire-and-forget vector
                // reductions into the L2-resident slot (zeroed before the launch).
                // Only this thread updates these addresses, so the adds apply in
                // program (= row, then big-before-small) order: deterministic.
#pragma unroll 1
                for (int pass = 0; pass < (last ? 2 : 1); ++pass) {
#pragma unroll 1
                    for (int c = 0; c < NF; c += 64) {
                        float a[64];
#pragma unroll
                        for (int u = 0; u < 4; ++u) tc::tmem_ld16(tl + (uint32_t)(pass * NF + c + 16 * u), a + 16 * u);
                        tc::tmem_ld_wait();
                        if constexpr (F16) {
#pragma unroll
                            for (int j = 0; j < 64; ++j) a[j] *= us;
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(
                                             dst + c + 4 * j),
                                         "f"(a[4 * j]), "f"(a[4 * j + 1]), "f"(a[4 * j + 2]), "f"(a[4 * j + 3]), "l"(keep)
                                         : "memory");
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR) tc::mbar_arrive_cluster(tempty0);
                    else tc::mbar_arrive(&tempty);
                }
            }
        }
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    if (warp == 16) {
        if constexpr (PAIR) tc::tmem_dealloc_pair<512>(tmem);
        else tc::tmem_dealloc<512>(tmem);
    }
}

// Backward for first-order tanh jets (LAY_XT S=3, LAY_MX S=4), N = 256.
// The jet transpose decouples there:
//   zb_s = d hb_s (s >= 1),   zb_0 = d (hb_0 - 2 t P),   P = sum_{s>=1} z_s hb_s,
// so the streams need not share TMEM. Two passes of two streams each
// ({1,2} then {3,0}; XT: {1,2} then {0}) run N=256 MMAs into two interleaved
// accumulators (the tensor pipe's full-rate pattern, tools/rate_probe.cu) and
// each stream's A tile is converted once (the N=128 n-tiled kernel converted it
// per n-tile). P (128 rows x 256 features, FP32) lives in shared memory
// between the passes, accumulated in the same order as act_bwd.
// Producers start a pass only after the previous epilogue released the stage
// ring, which the epilogue reuses as its Z_in staging.
// PAIR: a 2-CTA cluster covers 256 rows (cta_group::2, M = 256); each CTA
// stages half of the weight rows, which halves the stage and leaves room for a
// fourth one (the single-CTA ring is too shallow to hide the weight copies).
template <int L, bool PAIR = false>
struct Tc5BwdCfg {
    static constexpr int S = Streams<L>::S;
    static constexpr int NF = 256;
    static constexpr int NFL = PAIR ? NF / 2 : NF;  // weight rows staged by this CTA
    static constexpr int A_T = TC_TILE_BYTES;    // 128 rows x 8 fp32
    static constexpr int B_T = NFL * 32;         // weight rows x 8 fp32
    static constexpr int STAGE = 4 * A_T + 2 * B_T;  // 2 streams x (hi, lo) + B (hi, lo)
    static constexpr int NST = PAIR ? 4 : 3;
    static constexpr int TILE = 32 * 16 * 4;     // 32-row x 16-col staging tile, 16 B chunks XOR-swizzled
    static constexpr int EPI_BYTES = 8 * 2 * 3 * TILE;  // 8 warps x 2 buffers x {t, zA, zB}
    static constexpr int P_BYTES = 128 * NF * 4;
    static constexpr int SMEM = NST * STAGE + P_BYTES + 1024;
    static_assert(NST * STAGE >= EPI_BYTES, "epilogue staging must fit in the stage ring");
    static_assert(SMEM <= 227 * 1024, "tc5 bwd shared memory");
    static_assert(NST >= 3, "two k-steps per producer iteration need a third stage in flight");
    // pass -> streams (second = -1: single accumulator)
    __host__ __device__ static constexpr int sa(int pass) { return pass == 0 ? 1 : (S == 4 ? 3 : 0); }
    __host__ __device__ static constexpr int sb(int pass) { return pass == 0 ? 2 : (S == 4 ? 0 : -1); }
};

// F16: 3xFP16 operands (kind::f16, K = 16 per stage) scaled by the recorded
// |Zb_out| bounds g.amax_in and |W| bound g.amax_w; the epilogue unscales and
// records the |Zb_in| bounds in g.amax_out.
template <int L, bool PAIR, bool F16 = false>
__global__ void __launch_bounds__(TC3_THREADS, 1) k_tc5_bwd(const __grid_constant__ TcGemmArgs g) {
    using Cfg = Tc5BwdCfg<L, PAIR>;
    constexpr int NST = Cfg::NST, NF = Cfg::NF;
    constexpr int NEW = 8;              // epilogue warps (9-16)
    constexpr int ECOLS = 4 * NF / NEW;  // columns per epilogue warp and pass: 128
    constexpr int NCH = ECOLS / 16;      // 16-column chunks per warp and pass
    constexpr int NBUF = 2;              // staging buffers per warp
    static_assert(L == LAY_XT || L == LAY_MX, "first-order layouts only");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[NST], empty[NST], tfull, tempty, tempty_all;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
    // persistent: group `grp` (a CTA, or a pair) walks tiles grp, grp + ngrp, ...;
    // every ring / accumulator barrier keeps counting across tiles (pass index
    // gp = 2 * local tile + pass), so the producers prefetch the next tile's
    // operands into registers while the epilogue drains the current one
    const int ngrp = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x, grp = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ntiles = g.Rpad / (PAIR ? 256 : TC_M);
    const int nloc = grp < ntiles ? (ntiles - 1 - grp) / ngrp + 1 : 0;
    auto row0 = [&](int lt) { return PAIR ? (grp + lt * ngrp) * 256 + (int)rank * 128 : (grp + lt * ngrp) * TC_M; };
    const int nkb = g.K / (F16 ? 16 : 8);
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * NF;
    // weight stage copy of k-step kk into `stage` (tid 0 of the producers)
    auto load_w = [&](int kk, int st, uint32_t stage, uint32_t full0) {
        if constexpr (PAIR) {
            // image rows (32 B each) of k-step kk: [hi: 256 rows][lo: 256 rows]
            const int rowb = kk * 2 * NF + (int)rank * Cfg::NFL;
            if (rank == 0) tc::mbar_arrive_expect_tx(&full[st], 2 * 2 * Cfg::B_T);
            tc::tma_load_2d_pair(stage + 4 * Cfg::A_T, &g.tmB, 0, rowb, full0 + st * 8);
            tc::tma_load_2d_pair(stage + 4 * Cfg::A_T + Cfg::B_T, &g.tmB, 0, rowb + NF, full0 + st * 8);
        } else {
            tc::mbar_arrive_expect_tx(&full[st], 2 * Cfg::B_T);
            tc::bulk_g2s(stage + 4 * Cfg::A_T, g.img + (int64_t)kk * (2 * Cfg::B_T / 4), 2 * Cfg::B_T, &full[st]);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], PAIR ? 17 : 9);  // producer warps (both CTAs) + expect_tx
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(&tfull, 1);
        tc::mbar_init(&tempty, NEW);                      // this CTA's epilogue -> its producers
        tc::mbar_init(&tempty_all, PAIR ? 2 * NEW : NEW);  // both epilogues -> the MMA issuer
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
    const uint32_t full0 = PAIR ? tc::mapa(tc::smem_u32(&full[0]), 0) : tc::smem_u32(&full[0]);
    const uint32_t tempty_all0 = PAIR ? tc::mapa(tc::smem_u32(&tempty_all), 0) : tc::smem_u32(&tempty_all);

    // ---------------- epilogue: 16-column chunks, Z_in staged by cp.async ----------------
    // staging tiles: row r, 16 B chunk c at r*64 + ((c ^ ((r>>1)&3)) << 4): conflict-free
    // for both the row-per-lane reads and the 8-rows-per-instruction copies.
    // Double-buffered: the tiles of chunk i+1 are in flight while chunk i computes.
    // Epilogue warp e = warp - 9: TMEM lane quarter warp % 4, column block cq.
    // (Measured and dropped: the producer warps joining the epilogue -- 16 warps,
    // 64 columns each, single-buffered staging -- bwd 16.9 -> 17.7 ms/step.)
    auto run_epilogue = [&](int pass, int gp, int r0) {
        const int ew = warp - 9;
        const int q = warp & 3, cq = (warp - 9) >> 2;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t stg0 = sbase + (uint32_t)ew * NBUF * 3 * Cfg::TILE;
        const uint32_t pbuf = sP + (uint32_t)ew * ECOLS * 32 * 4;  // [col/4][lane][4]: one 16 B access per 4 columns
        const int64_t rbase = (int64_t)(r0 + q * 32) * NF;
        const int lr = lane >> 2, lcv = lane & 3;
        auto soff = [](int r, int c) { return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4)); };
        const int s0 = Cfg::sa(pass), s1 = Cfg::sb(pass);
        // Z_in tiles this pass needs: t (stream 0) and z of its first-order streams
        const int zA = s0 > 0 ? s0 : -1, zB = s1 > 0 ? s1 : -1;
        auto issue = [&](int cch) {
            const uint32_t stg = stg0 + (uint32_t)(cch % NBUF) * 3 * Cfg::TILE;
            const int c0 = cq * ECOLS + cch * 16;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int sz = u == 0 ? 0 : (u == 1 ? zA : zB);
                if (sz < 0) continue;
                const float* src = g.Zlow + sz * RN + rbase + c0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    cp_async16(stg + u * Cfg::TILE + soff(8 * k + lr, lcv), src + (int64_t)(8 * k + lr) * NF + lcv * 4);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        float usa = 1.0f, usb = 1.0f;  // 3xFP16 unscale of the two accumulators
        if constexpr (F16) {
            const float usw = ldexpf(1.0f, -tc::f16_exp_bits(*g.amax_w));
            usa = usw * ldexpf(1.0f, -tc::f16_exp_bits(g.amax_in[s0]));
            if (s1 >= 0) usb = usw * ldexpf(1.0f, -tc::f16_exp_bits(g.amax_in[s1]));
        }
        float mxa = 0.0f, mxb = 0.0f;
        tc::mbar_wait(&tfull, (uint32_t)gp & 1u);
        tc::tc_fence_after();
        TC_T0();
        issue(0);
#pragma unroll 1
        for (int cch = 0; cch < NCH; ++cch) {
            const int c0 = cq * ECOLS + cch * 16;
            const uint32_t stg = stg0 + (uint32_t)(cch % NBUF) * 3 * Cfg::TILE;
            float ha[16], hb[16];
            tc::tmem_ld16(tl + (uint32_t)c0, ha);
            if (s1 >= 0) tc::tmem_ld16(tl + (uint32_t)(NF + c0), hb);
            if (NBUF == 2 && cch + 1 < NCH) {
                issue(cch + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncwarp();
            tc::tmem_ld_wait();
            if constexpr (F16) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    ha[j] *= usa;
                    hb[j] *= usb;
                }
            }
#pragma unroll
            for (int j4 = 0; j4 < 16; j4 += 4) {
                const uint32_t ro = soff(lane, j4 >> 2);
                const float4 t4 = lds128(stg + ro);
                const float tt[4] = {t4.x, t4.y, t4.z, t4.w};
                float za[4] = {0.f, 0.f, 0.f, 0.f}, zb2[4] = {0.f, 0.f, 0.f, 0.f}, pp[4] = {0.f, 0.f, 0.f, 0.f};
                if (zA >= 0) {
                    const float4 v = lds128(stg + Cfg::TILE + ro);
                    za[0] = v.x; za[1] = v.y; za[2] = v.z; za[3] = v.w;
                }
                if (zB >= 0) {
                    const float4 v = lds128(stg + 2 * Cfg::TILE + ro);
                    zb2[0] = v.x; zb2[1] = v.y; zb2[2] = v.z; zb2[3] = v.w;
                }
                if (pass == 1) {
                    const float4 v = lds128(pbuf + (uint32_t)((((cch * 16 + j4) >> 2) * 32 + lane) * 16));
                    pp[0] = v.x; pp[1] = v.y; pp[2] = v.z; pp[3] = v.w;
                }
                float oa[4], ob[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int j = j4 + e;
                    const float t = tt[e];
                    const float d = 1.0f - t * t;
                    if (pass == 0) {
                        // streams 1, 2: zb_s = d hb_s ; P = z_1 hb_1 + z_2 hb_2
                        oa[e] = d * ha[j];
                        ob[e] = d * hb[j];
                        float P = 0.0f;
                        P += za[e] * ha[j];
                        P += zb2[e] * hb[j];
                        pp[e] = P;
                    } else if (Streams<L>::S == 4) {
                        // streams 3, 0: zb_3 = d hb_3 ; zb_0 = d (hb_0 - 2 t (P + z_3 hb_3))
                        oa[e] = d * ha[j];
                        float P = pp[e];
                        P += za[e] * ha[j];
                        float tbar = hb[j];
                        tbar += -2.0f * t * P;
                        ob[e] = d * tbar;
                    } else {
                        // XT stream 0: zb_0 = d (hb_0 - 2 t P)
                        float tbar = ha[j];
                        tbar += -2.0f * t * pp[e];
                        oa[e] = d * tbar;
                        ob[e] = 0.0f;
                    }
                }
                if (pass == 0)
                    sts128(pbuf + (uint32_t)((((cch * 16 + j4) >> 2) * 32 + lane) * 16),
                           make_float4(pp[0], pp[1], pp[2], pp[3]));
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    mxa = fmaxf(mxa, fabsf(oa[e]));
                    mxb = fmaxf(mxb, fabsf(ob[e]));
                }
                // outputs in place: stream s0 -> its z tile (the t tile when s0 = 0),
                // stream s1 -> its z tile (the t tile when s1 = 0)
                sts128(stg + (zA >= 0 ? Cfg::TILE : 0) + ro, make_float4(oa[0], oa[1], oa[2], oa[3]));
                if (s1 >= 0) sts128(stg + (zB >= 0 ? 2 * Cfg::TILE : 0) + ro, make_float4(ob[0], ob[1], ob[2], ob[3]));
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int so = u == 0 ? s0 : s1;
                if (so < 0) continue;
                const int slot = u == 0 ? (zA >= 0 ? 1 : 0) : (zB >= 0 ? 2 : 0);
                float* dst = g.out + so * RN + rbase + c0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 v = lds128(stg + slot * Cfg::TILE + soff(8 * k + lr, lcv));
                    *reinterpret_cast<float4*>(dst + (int64_t)(8 * k + lr) * NF + lcv * 4) = v;
                }
            }
            __syncwarp();
        }
        if (g.amax_out) {
            tc::warp_amax(g.amax_out + s0, __float_as_uint(mxa));
            if (s1 >= 0) tc::warp_amax(g.amax_out + s1, __float_as_uint(mxb));
        }
        if (warp == 9 && lane == 0) TC_ACC(3);
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            tc::mbar_arrive(&tempty);
            if constexpr (PAIR) tc::mbar_arrive_cluster(tempty_all0);
            else tc::mbar_arrive(&tempty_all);
        }
    };

    if (F16 && warp < 8) {
        // ---------------- producers (3xFP16): one 16-wide k-step per stage ----------------
        const int prow = tid >> 1, pc = tid & 1;
        const uint32_t aoff = tc::sw32_chunk((uint32_t)prow, (uint32_t)pc);
#pragma unroll 1
        for (int gp = 0; gp < 2 * nloc; ++gp) {
            const int pass = gp & 1;
            const float* asrc = g.A + (int64_t)(row0(gp >> 1) + prow) * g.K + pc * 8;
            const int s0 = Cfg::sa(pass), s1 = Cfg::sb(pass);
            const float sc0 = ldexpf(1.0f, tc::f16_exp_bits(g.amax_in[s0]));
            const float sc1 = s1 >= 0 ? ldexpf(1.0f, tc::f16_exp_bits(g.amax_in[s1])) : 1.0f;
            constexpr int D = 2;  // k-steps of A prefetched in registers (3 or 4: slower, trace_bwd5)
            float4 ra[D][2], rb[D][2];
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    ra[d][u] = d < nkb ? ldg4(asrc + s0 * RK + d * 16 + 4 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
                    rb[d][u] = (s1 >= 0 && d < nkb) ? ldg4(asrc + s1 * RK + d * 16 + 4 * u)
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            if (gp > 0) tc::mbar_wait(&tempty, (uint32_t)(gp - 1) & 1u);  // the epilogue released the stage ring
#pragma unroll 1
            for (int kb0 = 0; kb0 < nkb; kb0 += D)
#pragma unroll
                for (int cur = 0; cur < D; ++cur) {
                    const int kb = kb0 + cur;
                    if (kb >= nkb) break;
                    uint4 ahi, alo, bhi, blo;
                    {
                        const float ha[8] = {ra[cur][0].x, ra[cur][0].y, ra[cur][0].z, ra[cur][0].w,
                                             ra[cur][1].x, ra[cur][1].y, ra[cur][1].z, ra[cur][1].w};
                        const float hb[8] = {rb[cur][0].x, rb[cur][0].y, rb[cur][0].z, rb[cur][0].w,
                                             rb[cur][1].x, rb[cur][1].y, rb[cur][1].z, rb[cur][1].w};
                        tc::split_h8(ha, sc0, ahi, alo);
                        tc::split_h8(hb, sc1, bhi, blo);
                    }
                    if (kb + D < nkb) {
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            ra[cur][u] = ldg4(asrc + s0 * RK + (kb + D) * 16 + 4 * u);
                            if (s1 >= 0) rb[cur][u] = ldg4(asrc + s1 * RK + (kb + D) * 16 + 4 * u);
                        }
                    }
                    const int it = gp * nkb + kb, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                    if (tid == 0) load_w(kb, st, stage, full0);
                    sts128u(stage + aoff, ahi);
                    sts128u(stage + Cfg::A_T + aoff, alo);
                    if (s1 >= 0) {
                        sts128u(stage + 2 * Cfg::A_T + aoff, bhi);
                        sts128u(stage + 3 * Cfg::A_T + aoff, blo);
                    }
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                        else tc::mbar_arrive(&full[st]);
                    }
                }
        }
    } else if (warp < 8) {
        // ---------------- producers: A tiles of the pass's two streams ----------------
        const int prow = tid >> 1, pc = tid & 1;
        const uint32_t aoff = tc::sw32_off((uint32_t)prow, (uint32_t)(pc * 4));
#pragma unroll 1
        for (int gp = 0; gp < 2 * nloc; ++gp) {
            const int pass = gp & 1;
            const float* asrc = g.A + (int64_t)(row0(gp >> 1) + prow) * g.K + pc * 4;
            const int s0 = Cfg::sa(pass), s1 = Cfg::sb(pass);
            constexpr int D = 4;  // k-steps of A prefetched in registers
            float4 ra[D], rb[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                ra[d] = d < nkb ? ldg4(asrc + s0 * RK + d * 8) : make_float4(0.f, 0.f, 0.f, 0.f);
                rb[d] = (s1 >= 0 && d < nkb) ? ldg4(asrc + s1 * RK + d * 8) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (gp > 0) tc::mbar_wait(&tempty, (uint32_t)(gp - 1) & 1u);  // the epilogue released the stage ring
            // two k-steps per iteration: their stores share one proxy fence
#pragma unroll 1
            for (int kb0 = 0; kb0 < nkb; kb0 += D)
#pragma unroll
            for (int cur = 0; cur < D; cur += 2) {
                const int kb = kb0 + cur;
                if (kb >= nkb) break;
                float4 h[2][4];  // per k-step: A hi, A lo, B hi, B lo
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float4 va = ra[cur + u], vb = rb[cur + u];
                    if (kb + u + D < nkb) {
                        ra[cur + u] = ldg4(asrc + s0 * RK + (kb + u + D) * 8);
                        if (s1 >= 0) rb[cur + u] = ldg4(asrc + s1 * RK + (kb + u + D) * 8);
                    }
                    split4(va, h[u][0], h[u][1]);
                    split4(vb, h[u][2], h[u][3]);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int it = gp * nkb + kb + u, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                        if (tid == 0) TC_ACC(2);
                    }
                    if (tid == 0) load_w(kb + u, st, stage, full0);
                    sts128(stage + aoff, h[u][0]);
                    sts128(stage + Cfg::A_T + aoff, h[u][1]);
                    if (s1 >= 0) {
                        sts128(stage + 2 * Cfg::A_T + aoff, h[u][2]);
                        sts128(stage + 3 * Cfg::A_T + aoff, h[u][3]);
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int st = (gp * nkb + kb + u) % NST;
                        if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                        else tc::mbar_arrive(&full[st]);
                    }
            }
        }
    } else if (warp == 8) {
        // ---------------- MMA issuer ----------------
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = F16 ? tc::make_idesc_f16(PAIR ? 2 * TC_M : TC_M, NF, 0, 0)
                                           : tc::make_idesc_tf32(PAIR ? 2 * TC_M : TC_M, NF, 0, 0);
            for (int gp = 0; gp < 2 * nloc; ++gp) {
                const int pass = gp & 1;
                const bool two = Cfg::sb(pass) >= 0;
                if (gp > 0) tc::mbar_wait(&tempty_all, (uint32_t)(gp - 1) & 1u);  // TMEM drained
                tc::tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb) {
                    const int it = gp * nkb + kb, st = it % NST;
                    const uint32_t stage = sbase + st * Cfg::STAGE;
                    {
                        TC_T0();
                        tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                        TC_ACC(0);
                    }
                    tc::tc_fence_after();
                    const uint64_t bh = tc::make_sdesc(stage + 4 * Cfg::A_T, 16, 256, 6);
                    const uint64_t bl = tc::make_sdesc(stage + 4 * Cfg::A_T + Cfg::B_T, 16, 256, 6);
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
                        if (a == 1 && !two) break;
                        const uint32_t ah = stage + (2 * a) * Cfg::A_T;
                        const uint64_t adh = tc::make_sdesc(ah, 16, 256, 6), adl = tc::make_sdesc(ah + Cfg::A_T, 16, 256, 6);
                        const uint32_t d = tmem + (uint32_t)(a * NF);
                        if constexpr (F16 && PAIR) {
                            tc::mma_f16_pair(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                            tc::mma_f16_pair(d, adh, bl, idesc, 1u);
                            tc::mma_f16_pair(d, adl, bh, idesc, 1u);
                        } else if constexpr (F16) {
                            tc::mma_f16(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                            tc::mma_f16(d, adh, bl, idesc, 1u);
                            tc::mma_f16(d, adl, bh, idesc, 1u);
                        } else if constexpr (PAIR) {
                            tc::mma_tf32_pair(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                            tc::mma_tf32_pair(d, adh, bl, idesc, 1u);
#ifndef PNX_EXP_TWO_MMA  // timing experiment only: drops a product
                            tc::mma_tf32_pair(d, adl, bh, idesc, 1u);
#endif
                        } else {
                            tc::mma_tf32(d, adh, bh, idesc, kb > 0 ? 1u : 0u);
                            tc::mma_tf32(d, adh, bl, idesc, 1u);
#ifndef PNX_EXP_TWO_MMA  // timing experiment only: drops a product
                            tc::mma_tf32(d, adl, bh, idesc, 1u);
#endif
                        }
                    }
                    if constexpr (PAIR) tc::mma_commit_pair(&empty[st], 3);
                    else tc::mma_commit(&empty[st]);
                }
                if constexpr (PAIR) tc::mma_commit_pair(&tfull, 3);
                else tc::mma_commit(&tfull);
            }
        }
        __syncwarp();
    } else {
#pragma unroll 1
        for (int gp = 0; gp < 2 * nloc; ++gp) run_epilogue(gp & 1, gp, row0(gp >> 1));
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    if (warp == 8) {
        if constexpr (PAIR) tc::tmem_dealloc_pair<512>(tmem);
        else tc::tmem_dealloc<512>(tmem);
    }
}

// PAIR: a 2-CTA cluster covers 256 rows of one n-tile with cta_group::2 MMAs
// (M = 256); each CTA stages its own 128 rows of every stream and half of the
// n-tile's weight rows (2-D tensor TMA completing on the leader's barrier).
template <int S, int NT, bool PAIR = false>
struct Tc2BwdCfg {
    static constexpr int A_BYTES = 2 * S * TC_TILE_BYTES;
    static constexpr int NTL = PAIR ? NT / 2 : NT;  // weight rows staged by this CTA
    static constexpr int B_T = NTL * 32;
    static constexpr int STAGE = A_BYTES + 2 * B_T;
    static constexpr int NST = (TC_SMEM - 1024) / STAGE > 8 ? 8 : (TC_SMEM - 1024) / STAGE;
    // the epilogue reuses the (then idle) stage ring as its staging buffer
    static constexpr int EPI_BYTES = 8 * S * 32 * 36 * 4;
    static constexpr int SMEM = (NST * STAGE > EPI_BYTES ? NST * STAGE : EPI_BYTES) + 1024;
    static_assert(SMEM <= 227 * 1024, "bwd shared memory");
};

// F16: 3xFP16 operands (non-pair only), per-stream scales from the recorded |Zb| bounds
template <int L, int NT, bool PAIR, bool F16 = false>
__global__ void __launch_bounds__(TC3_THREADS, 1) k_tc2_bwd(const __grid_constant__ TcGemmArgs g) {
    using St = Streams<L>;
    constexpr int S = St::S;
    using Cfg = Tc2BwdCfg<S, NT, PAIR>;
    constexpr int NST = Cfg::NST;
    static_assert(!(F16 && PAIR), "3xFP16 general backward: single CTA");
    constexpr int D = F16 ? 1 : 2;  // k-steps of A in registers (F16 steps carry twice the features)
    constexpr int KS = F16 ? 16 : 8;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    __shared__ uint64_t full[8], empty[8], tfull;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntiles = g.N / NT;
    const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
    const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // (row tile, n tile) of this CTA / pair
    const int rt = cid / ntiles, nt = cid % ntiles;
    const int r0 = PAIR ? rt * 256 + (int)rank * 128 : rt * TC_M, n0 = nt * NT;
    const int nkb = g.K / KS;
    const int64_t RK = (int64_t)g.Rpad * g.K, RN = (int64_t)g.Rpad * g.N;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            tc::mbar_init(&full[i], PAIR ? 17 : 9);  // producer warps (both CTAs) + expect_tx
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(&tfull, 1);
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
    const float* bimg = g.img + (int64_t)nt * nkb * (2 * NT * 8);
    const uint32_t full0 = PAIR ? tc::mapa(tc::smem_u32(&full[0]), 0) : 0u;

    if (F16 && warp < 8) {
        // ---- 3xFP16 producers: 8 consecutive features per thread and k-step ----
        const int prow = tid >> 1, pc = tid & 1;
        const float* asrc = g.A + (int64_t)(r0 + prow) * g.K + pc * 8;
        const uint32_t aoff = tc::sw32_chunk((uint32_t)prow, (uint32_t)pc);
        float sc[S];
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) sc[s2] = ldexpf(1.0f, tc::f16_exp_bits(g.amax_in[s2]));
        float4 ring[S][2];
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
            ring[s2][0] = ldg4(asrc + s2 * RK);
            ring[s2][1] = ldg4(asrc + s2 * RK + 4);
        }
        for (int it = 0; it < nkb; ++it) {
            const int st = it % NST;
            const uint32_t stage = sbase + st * Cfg::STAGE;
            uint4 hi[S], lo[S];
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                const float h[8] = {ring[s2][0].x, ring[s2][0].y, ring[s2][0].z, ring[s2][0].w,
                                    ring[s2][1].x, ring[s2][1].y, ring[s2][1].z, ring[s2][1].w};
                tc::split_h8(h, sc[s2], hi[s2], lo[s2]);
            }
            if (it + 1 < nkb)
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) {
                    ring[s2][0] = ldg4(asrc + s2 * RK + (it + 1) * 16);
                    ring[s2][1] = ldg4(asrc + s2 * RK + (it + 1) * 16 + 4);
                }
            tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
            if (tid == 0) {
                tc::mbar_arrive_expect_tx(&full[st], 2 * Cfg::B_T);
                tc::bulk_g2s(stage + Cfg::A_BYTES, bimg + (int64_t)it * (2 * Cfg::B_T / 4), 2 * Cfg::B_T, &full[st]);
            }
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                sts128u(stage + (2 * s2) * TC_TILE_BYTES + aoff, hi[s2]);
                sts128u(stage + (2 * s2 + 1) * TC_TILE_BYTES + aoff, lo[s2]);
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[st]);
        }
    } else if (warp < 8) {
        const int prow = tid >> 1, pc = tid & 1;
        const float* asrc = g.A + (int64_t)(r0 + prow) * g.K + pc * 4;
        const uint32_t aoff = tc::sw32_off((uint32_t)prow, (uint32_t)(pc * 4));
        float4 ring[D][S];
#pragma unroll
        for (int d = 0; d < D; ++d)
            if (d < nkb)
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) ring[d][s2] = ldg4(asrc + s2 * RK + d * 8);
        for (int it0 = 0; it0 < nkb; it0 += D) {
#pragma unroll
            for (int slot = 0; slot < D; ++slot) {
                const int it = it0 + slot;
                if (it >= nkb) break;
                const int st = it % NST;
                const uint32_t stage = sbase + st * Cfg::STAGE;
                float4 hi[S], lo[S];
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) split4_trunc(ring[slot][s2], hi[s2], lo[s2]);
                if (it + D < nkb)
#pragma unroll
                    for (int s2 = 0; s2 < S; ++s2) ring[slot][s2] = ldg4(asrc + s2 * RK + (it + D) * 8);
                tc::mbar_wait(&empty[st], ((uint32_t)(it / NST) & 1u) ^ 1u);
                if (tid == 0) {
                    if constexpr (PAIR) {
                        // image rows (8 fp32 each) of k-step it: [hi: NT rows][lo: NT rows]
                        const int rowb = (nt * nkb + it) * 2 * NT + (int)rank * Cfg::NTL;
                        if (rank == 0) tc::mbar_arrive_expect_tx(&full[st], 2 * 2 * Cfg::B_T);
                        tc::tma_load_2d_pair(stage + Cfg::A_BYTES, &g.tmB, 0, rowb, full0 + st * 8);
                        tc::tma_load_2d_pair(stage + Cfg::A_BYTES + Cfg::B_T, &g.tmB, 0, rowb + NT, full0 + st * 8);
                    } else {
                        tc::mbar_arrive_expect_tx(&full[st], 2 * Cfg::B_T);
                        tc::bulk_g2s(stage + Cfg::A_BYTES, bimg + (int64_t)it * (2 * Cfg::B_T / 4), 2 * Cfg::B_T,
                                     &full[st]);
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) {
                    sts128(stage + (2 * s2) * TC_TILE_BYTES + aoff, hi[s2]);
                    sts128(stage + (2 * s2 + 1) * TC_TILE_BYTES + aoff, lo[s2]);
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR) tc::mbar_arrive_cluster(full0 + st * 8);
                    else tc::mbar_arrive(&full[st]);
                }
            }
        }
    } else if (warp == 8) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = F16 ? tc::make_idesc_f16(TC_M, NT, 0, 0)
                                           : tc::make_idesc_tf32(PAIR ? 2 * TC_M : TC_M, NT, 0, 0);
            for (int it = 0; it < nkb; ++it) {
                const int st = it % NST;
                const uint32_t stage = sbase + st * Cfg::STAGE;
                {
                    TC_T0();
                    tc::mbar_wait(&full[st], (uint32_t)(it / NST) & 1u);
                    TC_ACC(0);
                }
                tc::tc_fence_after();
                const uint64_t bh = tc::make_sdesc(stage + Cfg::A_BYTES, 16, 256, 6);
                const uint64_t bl = tc::make_sdesc(stage + Cfg::A_BYTES + Cfg::B_T, 16, 256, 6);
                // stream-major order (tools/rate_probe.cu: 3 MMAs into one
                // accumulator then the next runs at 84% vs 56% term-major)
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) {
                    const uint32_t ah = stage + (2 * s2) * TC_TILE_BYTES;
                    const uint64_t adh = tc::make_sdesc(ah, 16, 256, 6), adl = tc::make_sdesc(ah + TC_TILE_BYTES, 16, 256, 6);
                    const uint32_t d = tmem + (uint32_t)(s2 * NT);
                    if constexpr (F16) {
                        tc::mma_f16(d, adh, bh, idesc, it > 0 ? 1u : 0u);
                        tc::mma_f16(d, adh, bl, idesc, 1u);
                        tc::mma_f16(d, adl, bh, idesc, 1u);
                    } else if constexpr (PAIR) {
                        tc::mma_tf32_pair(d, adh, bh, idesc, it > 0 ? 1u : 0u);
                        tc::mma_tf32_pair(d, adh, bl, idesc, 1u);
                        tc::mma_tf32_pair(d, adl, bh, idesc, 1u);
                    } else {
                        tc::mma_tf32(d, adh, bh, idesc, it > 0 ? 1u : 0u);
                        tc::mma_tf32(d, adh, bl, idesc, 1u);
                        tc::mma_tf32(d, adl, bh, idesc, 1u);
                    }
                }
                if constexpr (PAIR) tc::mma_commit_pair(&empty[st], 3);
                else tc::mma_commit(&empty[st]);
            }
            if constexpr (PAIR) tc::mma_commit_pair(&tfull, 3);
            else tc::mma_commit(&tfull);
        }
        __syncwarp();
    } else {
        // All MMAs have retired once tfull fires, so the stage ring is free:
        // each warp stages 32-row x 32-feature blocks of every stream there
        // and moves them to/from HBM as full 128-byte lines (8 lanes per row).
        constexpr int ROWF = 36;  // padded row (floats): conflict-free 16-B lanes
        const int q = warp & 3, half = (warp - 9) >> 2;
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t buf = sbase + (uint32_t)(warp - 9) * (S * 32 * ROWF * 4);
        const int64_t rbase = (int64_t)(r0 + q * 32) * g.N + n0;
        const int lr = lane >> 3, lc = (lane & 7) * 4;
        float mx[S];  // |Zb_in| bounds per stream (consumers' 3xFP16 scales)
        float us[S];  // 3xFP16 unscale per stream accumulator 2^-(e_s + e_W)
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
            mx[s2] = 0.0f;
            us[s2] = F16 ? ldexpf(1.0f, -tc::f16_exp_bits(g.amax_in[s2])) * ldexpf(1.0f, -tc::f16_exp_bits(*g.amax_w))
                         : 1.0f;
        }
        tc::mbar_wait(&tfull, 0);
        tc::tc_fence_after();
        TC_T0();
#pragma unroll 1
        for (int cc = 0; cc < NT / 2; cc += 32) {
            const int c0 = half * (NT / 2) + cc;
            // all S streams' lines in flight at once (cp.async: no register staging)
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                const float* src = g.Zlow + s2 * RN + rbase + c0;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    cp_async16(buf + ((s2 * 32 + 4 * k + lr) * ROWF + lc) * 4, src + (int64_t)(4 * k + lr) * g.N + lc);
            }
            cp_async_wait_all();
            __syncwarp();
#pragma unroll 1
            for (int c = 0; c < 32; c += 8) {
                float hb[S][8], z[S][8];
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) tmem_ld8(tl + (uint32_t)(s2 * NT + c0 + c), hb[s2]);
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) {
                    const uint32_t a = buf + ((s2 * 32 + lane) * ROWF + c) * 4;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(z[s2][0]), "=f"(z[s2][1]), "=f"(z[s2][2]), "=f"(z[s2][3]) : "r"(a));
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(z[s2][4]), "=f"(z[s2][5]), "=f"(z[s2][6]), "=f"(z[s2][7]) : "r"(a + 16));
                }
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float zz[S], hh[S], oo[S];
#pragma unroll
                    for (int s2 = 0; s2 < S; ++s2) {
                        zz[s2] = z[s2][j];
                        hh[s2] = F16 ? hb[s2][j] * us[s2] : hb[s2][j];
                    }
                    act_bwd<L, ACT_TANH>(zz, hh, oo, 1.0f);
#pragma unroll
                    for (int s2 = 0; s2 < S; ++s2) {
                        hb[s2][j] = oo[s2];
                        mx[s2] = fmaxf(mx[s2], fabsf(oo[s2]));
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < S; ++s2) {
                    const uint32_t a = buf + ((s2 * 32 + lane) * ROWF + c) * 4;
                    sts128(a, make_float4(hb[s2][0], hb[s2][1], hb[s2][2], hb[s2][3]));
                    sts128(a + 16, make_float4(hb[s2][4], hb[s2][5], hb[s2][6], hb[s2][7]));
                }
            }
            __syncwarp();
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                float* dst = g.out + s2 * RN + rbase + c0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    float4 v;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                                 : "r"(buf + ((s2 * 32 + 4 * k + lr) * ROWF + lc) * 4));
                    *reinterpret_cast<float4*>(dst + (int64_t)(4 * k + lr) * g.N + lc) = v;
                }
            }
            __syncwarp();
        }
        if (g.amax_out) {
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) tc::warp_amax(g.amax_out + s2, __float_as_uint(mx[s2]));
        }
        if (warp == 9 && lane == 0) TC_ACC(3);
    }
    tc::tc_fence_before();
    if constexpr (PAIR) tc::cluster_sync();
    else __syncthreads();
    if (warp == 8) {
        if constexpr (PAIR) tc::tmem_dealloc_pair<512>(tmem);
        else tc::tmem_dealloc<512>(tmem);
    }
}

}  // namespace pnx
