// pnx_capi.cu -- C ABI (include/pnx.h) and host orchestration of one worker
// step on one B200. Replaces run_worker_epoch's graph build + nested reverse
// sweeps (trainer.cpp:200-262) with a chunked pass of jet kernels:
//
//   prep -> [per chunk: input -> L fwd GEMMs -> head -> L rev GEMMs + dW]
//        -> fixed-order reductions -> flat gradient (trainable() order)
//
// Rows of a step are laid out [bc_a | bc_b | ic | interior]; the small
// replicated IC/BC sets (trainer.cpp:225-232) ride in the first chunk and carry
// value-only seeds, interior rows carry residual seeds (losses.cpp:77-95).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys) is attached

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pnx.h"
#include "kernels_simt.cuh"
#include "tc_gemm.cuh"
#include "launch.h"
#include "sampling.cuh"
#include "small_net.cuh"

using namespace pnx;

namespace {

thread_local std::string g_create_error;

int64_t roundup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace

struct pnx_ctx {
    int device = 0;
    int nsm = 148;  // SM count of `device` (grid sizing)
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    int engine = PNX_ENGINE_AUTO;

    // model (ModelSpec)
    int in_dim = 0, H = 0, depth = 0, F = 0, act = 0;
    float w0 = 1.0f;
    bool rwf = false;
    int rff_w = 0, E = 0, K0 = 0;
    int periodic[kMaxAxes] = {0, 0, 0, 0};
    double period[kMaxAxes] = {0, 0, 0, 0};
    int64_t period_off[kMaxAxes] = {-1, -1, -1, -1};
    bool train_period = false;
    // problem
    int pde = 0, bc = 0, layout = 0, S = 1, Kres = 1;
    PdeConst pc{};
    double res_eps = 1.0, res_mu = 1.0;  // ResidualSpec epsilon / mu in FP64
    // params
    int64_t P = 0;
    LayerTab tab{};
    int64_t wsize = 0, bsize = 0;

    // collocation (global rows: [bc_a | bc_b | ic | poynting | interior])
    int64_t n_bca = 0, n_bcb = 0, n_ic = 0, n_int = 0;
    std::vector<double> h_int, h_ic, h_bca, h_bcb;  // axis-major host copies
    std::vector<float> h_ic_t, h_bc_t;
    bool rows_dirty = true;
    double* d_coords = nullptr;
    int64_t ld = 0, coords_cap = 0, layout_T = -1, layout_chunk_override = -1;
    float *d_ic_t = nullptr, *d_bc_t = nullptr;
    double* d_rffB = nullptr;

    // weights / grads
    float *d_W = nullptr, *d_Wt = nullptr, *d_bias = nullptr;
    float *d_params = nullptr, *d_grad = nullptr;
    double* d_losses = nullptr;

    // activations
    int64_t chunk_rows = 0, chunk_override = 0, Rcap = 0;
    float *d_Hin = nullptr, *d_Hinb = nullptr;
    std::vector<float*> d_Z;
    float* d_Zb[2] = {nullptr, nullptr};
    // partials
    std::vector<double*> d_part;
    std::vector<int> nsplit;
    double* d_head_part = nullptr;
    int head_grid = 296;
    double* d_loss_part = nullptr;
    double* d_partP = nullptr;
    int ibwd_grid = 148;
    double* d_red = nullptr;
    float* d_bc_vals = nullptr;
    // sticky non-finite flags (first bad index, kBadNone = none), read and reset by
    // pnx_check: [0..2] residual component (losses.cpp:86-90), [3] Adam gradient
    // entry, [4] the Adam step it happened at (optim.cpp:16-22)
    int* d_bad = nullptr;
    // completion of the last step's work (recorded on the launching stream outside
    // graph capture): host-side writes to step inputs wait on it
    cudaEvent_t ev_done = nullptr;
    bool ev_pending = false;
    // PNX_GUARD=1: every context buffer carries a tail of kGuardBytes set to
    // kGuardByte, verified by pnx_check (a memcheck stand-in for out-of-bounds writes)
    std::vector<std::pair<void*, size_t>> guards;  // (buffer, payload bytes)
    // pnx_step's CUDA graph: every call that can change what a step enqueues bumps
    // state_ver; the first step after a change runs eagerly (uploads, allocations),
    // the second captures the device step, later ones replay it (same lambdas)
    uint64_t state_ver = 1, g_ver = 0, g_warm_ver = 0;
    double g_lam[3] = {0, 0, 0}, g_warm_lam[3] = {0, 0, 0};
    cudaGraphExec_t g_exec = nullptr;
    // pinned FP32 staging of the host-buffer step (pnx_step): params in, gradient out
    float* h_stage = nullptr;
    int64_t stage_cap = 0;
    // 3xFP16 operand bounds (float bits): [|W_l|] [|Z_l[s]|] [|Zb_l[s]|]
    unsigned* d_amax = nullptr;
    float* d_resid = nullptr;
    int64_t resid_cap = 0;
    bool h_int_stale = false;  // interior coordinates newer on device than in h_int
    // interior generated on the device (pnx_sample_points): no host copy; a
    // re-layout regenerates it from the design below
    bool int_on_device = false;
    SampleArgs samp{};
    int64_t int_off_prev = 0;  // first interior row of the uploaded layout
    bool capture_resid = false;
    // objective terms whose seeds need a global reduction first (trainer.cpp:209-247)
    int caus_M = 0;  // causality segments (0 = off)
    double caus_eps = 1.0, caus_tlo = 0.0, caus_thi = 1.0;
    double *d_caus_cnt = nullptr, *d_seg_part = nullptr, *d_caus_loss = nullptr;
    float* d_seg_w = nullptr;
    double poy_w = 0.0, poy_box[6] = {0, 0, 0, 0, 0, 0};
    int poy_grid = 0, poy_T = 0;
    int64_t n_poy = 0;  // Poynting quadrature rows (replicated, chunk 0)
    std::vector<double> h_poy;
    double *d_poy_part = nullptr, *d_pen = nullptr;
    float* d_poy_g = nullptr;
    bool no_penalty = false;  // per-term gradient passes exclude the penalty (trainer.cpp:256-260)
    // per-term passes 2 and 3 reuse the activations (and their operand bounds) of
    // pass 1 when the whole step is one chunk: same parameters, same points
    bool reuse_fwd = false;
    TcWorkspace tc{};
    double* d_sn_slot = nullptr;  // single-kernel narrow step: [grid][P] FP64 gradient slots
    // kernel-class timing with CUDA events on the launching stream (bench roofline)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_cls;  // class per recorded pair
    size_t ev_used = 0;
    double prof_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t prof_n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

namespace {

int fail(pnx_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

#define CK(call)                                                                     \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess)                                                       \
            return fail(ctx, PNX_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                        \
    do {                                                                             \
        ++ctx->launches;                                                             \
        cudaError_t e_ = cudaGetLastError();                                         \
        if (e_ != cudaSuccess)                                                       \
            return fail(ctx, PNX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

constexpr size_t kGuardBytes = 512;
constexpr int kGuardByte = 0xA5;
inline bool guard_on() {
    static const bool on = getenv("PNX_GUARD") && (getenv("PNX_GUARD")[0] == '1' || !strcmp(getenv("PNX_GUARD"), "poke"));
    return on;
}
// PNX_GUARD=poke: the negative control -- one byte past the end of every buffer
// is overwritten right after allocation, so the first check must report it
inline bool guard_poke() {
    static const bool on = getenv("PNX_GUARD") && !strcmp(getenv("PNX_GUARD"), "poke");
    return on;
}

// a buffer leaves the guard list before it is freed / joins it (tail set) after allocation
static void guard_forget(pnx_ctx* ctx, const void* p) {
    for (size_t i = 0; i < ctx->guards.size(); ++i)
        if (ctx->guards[i].first == p) {
            ctx->guards.erase(ctx->guards.begin() + (std::ptrdiff_t)i);
            return;
        }
}
static int guard_add(pnx_ctx* ctx, void* p, size_t bytes) {
    if (!guard_on() || !p) return PNX_OK;
    guard_forget(ctx, p);
    CK(cudaMemset(reinterpret_cast<uint8_t*>(p) + bytes, kGuardByte, kGuardBytes));
    if (guard_poke()) CK(cudaMemset(reinterpret_cast<uint8_t*>(p) + bytes, 0, 1));
    ctx->guards.emplace_back(p, bytes);
    return PNX_OK;
}

template <class T>
int dalloc(pnx_ctx* ctx, T** p, size_t n) {
    if (*p) {
        guard_forget(ctx, *p);
        cudaFree(*p);
    }
    *p = nullptr;
    if (n == 0) return PNX_OK;
    const size_t bytes = n * sizeof(T);
    CK(cudaMalloc(reinterpret_cast<void**>(p), bytes + (guard_on() ? kGuardBytes : 0)));
    return guard_add(ctx, *p, bytes);
}

// PNX_GUARD=1: every guard tail still holds its pattern (call after a device sync)
static int guard_check(pnx_ctx* ctx) {
    if (!guard_on()) return PNX_OK;
    std::vector<uint8_t> h(kGuardBytes);
    for (size_t i = 0; i < ctx->guards.size(); ++i) {
        const auto& gd = ctx->guards[i];
        CK(cudaMemcpy(h.data(), reinterpret_cast<const uint8_t*>(gd.first) + gd.second, kGuardBytes,
                      cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < kGuardBytes; ++k)
            if (h[k] != (uint8_t)kGuardByte)
                return fail(ctx, PNX_ERR_CUDA,
                            "guard: write past the end of a " + std::to_string(gd.second) + "-byte device buffer (byte " +
                                std::to_string(k) + " of its guard)");
    }
    return PNX_OK;
}

enum ProfClass { PC_INPUT = 0, PC_FWD = 1, PC_HEAD = 2, PC_BWD = 3, PC_WGRAD = 4, PC_FINAL = 5, PC_FUSED = 6 };

const char* const kClassName[8] = {"pnx input", "pnx forward GEMM", "pnx head", "pnx reverse GEMM",
                                   "pnx weight gradient", "pnx finalize", "pnx single-kernel step", "pnx"};

// NVTX range per kernel class (nsys timelines), and with profiling on a CUDA
// event pair on the launching stream around the launch.
void prof_begin(pnx_ctx* c, int cls, cudaStream_t st) {
    nvtxRangePushA(kClassName[cls & 7]);
    if (!c->prof) return;
    if (c->ev_used + 2 > c->ev_pool.size()) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            c->ev_pool.push_back(e);
        }
    }
    cudaEventRecord(c->ev_pool[c->ev_used], st);
    c->ev_cls.push_back(cls);
}
void prof_end(pnx_ctx* c, cudaStream_t st) {
    nvtxRangePop();
    if (!c->prof) return;
    cudaEventRecord(c->ev_pool[c->ev_used + 1], st);
    c->ev_used += 2;
}
void prof_collect(pnx_ctx* c) {
    for (size_t i = 0; i < c->ev_cls.size(); ++i) {
        float ms = 0.0f;
        cudaEventSynchronize(c->ev_pool[2 * i + 1]);
        cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]);
        c->prof_ms[c->ev_cls[i]] += ms;
        c->prof_n[c->ev_cls[i]] += 1;
    }
    c->ev_cls.clear();
    c->ev_used = 0;
}

int pde_layout(int pde) {
    switch (pde) {
        case PNX_PDE_ADVECTION:
        case PNX_PDE_BURGERS: return LAY_XT;
        case PNX_PDE_ALLEN_CAHN: return LAY_AC;
        case PNX_PDE_MAXWELL_TE:
        case PNX_PDE_MAXWELL_TE_EH: return LAY_MX;
        case PNX_PDE_NS_STEADY: return LAY_NS;
    }
    return -1;
}

// launch_* dispatchers: launch_simt.cu / launch_tc.cu (declared in launch.h)

// ---- buffers ---------------------------------------------------------------

constexpr int kL0Blocks = 296;
// layer 0 fused with the input jets (narrow embedding: no RFF, K0 <= 8, H % 4 == 0)
constexpr int kAmaxS = 8;
constexpr int kAmaxLen = kMaxLayers * (1 + 2 * kAmaxS) + kAmaxS;
inline unsigned* amax_w(pnx_ctx* c, int l) { return c->d_amax + l; }
inline unsigned* amax_z(pnx_ctx* c, int l) { return c->d_amax + kMaxLayers + l * kAmaxS; }
inline unsigned* amax_zb(pnx_ctx* c, int l) { return c->d_amax + kMaxLayers * (1 + kAmaxS) + l * kAmaxS; }
// bounds of the unfused input features Hin (k_input: RFF or a wide embedding)
inline unsigned* amax_hin(pnx_ctx* c) { return c->d_amax + kMaxLayers * (1 + 2 * kAmaxS); }
bool layer0_fused(const pnx_ctx* c) { return c->rff_w == 0 && c->K0 <= 8 && c->H % 4 == 0 && c->H <= 512; }

int64_t bytes_per_row(const pnx_ctx* c) {
    int64_t f = (int64_t)c->S * (c->K0 + (int64_t)c->depth * c->H + 2LL * c->H + (c->train_period ? c->K0 : 0));
    return f * 4;
}

// Points per causality segment of this shard (split_time_segments, trainer.cpp:156-177).
int causality_counts(pnx_ctx* ctx, const double* tcol, int64_t n) {
    if (ctx->caus_M <= 0) return PNX_OK;
    std::vector<double> cnt((size_t)ctx->caus_M, 0.0);
    const double span = ctx->caus_thi - ctx->caus_tlo;
    for (int64_t i = 0; i < n; ++i) {
        const double frac = (tcol[i] - ctx->caus_tlo) / span;
        const int sg = std::min(ctx->caus_M - 1, std::max(0, static_cast<int>(frac * ctx->caus_M)));
        cnt[(size_t)sg] += 1.0;
    }
    CK(cudaMemcpy(ctx->d_caus_cnt, cnt.data(), cnt.size() * 8, cudaMemcpyHostToDevice));
    return PNX_OK;
}

// [0, n) split over a few host threads when n is large (the FP64 <-> FP32
// conversions of pnx_step: ~P elements each way per step)
template <class F>
static void host_par_for(int64_t n, F&& f) {
    const int64_t kMinPerThread = 65536;
    int nt = (int)std::min<int64_t>(std::min(8u, std::max(1u, std::thread::hardware_concurrency())),
                                    n / kMinPerThread);
    if (nt <= 1) {
        f((int64_t)0, n);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t per = (n + nt - 1) / nt;
    auto range = [&](int i) { f(std::min(n, i * per), std::min(n, (i + 1) * per)); };
    int started = 1;
    try {  // no exception may cross the C ABI: ranges without a thread run here
        pool.reserve((size_t)nt - 1);
        for (; started < nt; ++started) pool.emplace_back(range, started);
    } catch (...) {
    }
    range(0);
    for (int i = started; i < nt; ++i) range(i);
    for (auto& t : pool) t.join();
}

int wait_last_step(pnx_ctx* ctx);

// generate the device design into the interior segment (rows laid out, ld set)
// and recount the causality segments on the device; synchronous on ctx->stream
int generate_interior(pnx_ctx* ctx) {
    SampleArgs a = ctx->samp;
    a.out = ctx->d_coords + ctx->int_off_prev;
    a.ld = ctx->ld;
    const unsigned grid = (unsigned)std::min<int64_t>((a.nrows + 255) / 256, 148 * 16);
    k_sample<<<grid, 256, 0, ctx->stream>>>(a);
    CK(cudaGetLastError());
    if (ctx->caus_M > 0) {
        CK(cudaMemsetAsync(ctx->d_caus_cnt, 0, (size_t)ctx->caus_M * 8, ctx->stream));
        k_segment_counts<<<grid, 256, 0, ctx->stream>>>(a.out + (int64_t)(ctx->in_dim - 1) * a.ld, a.nrows,
                                                        ctx->caus_M, ctx->caus_tlo, ctx->caus_thi - ctx->caus_tlo,
                                                        ctx->d_caus_cnt);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return PNX_OK;
}

int upload_rows(pnx_ctx* ctx) {
    if (int r = wait_last_step(ctx)) return r;
    const int d = ctx->in_dim;
    if (ctx->h_int_stale && ctx->d_coords && !ctx->int_on_device) {  // pull the fast-path interior back before re-layout
        const int64_t off = ctx->int_off_prev;
        ctx->h_int.resize((size_t)(ctx->n_int * d));  // empty when the previous interior was a device design
        for (int a = 0; a < d; ++a)
            CK(cudaMemcpy(ctx->h_int.data() + a * ctx->n_int, ctx->d_coords + a * ctx->ld + off,
                          (size_t)ctx->n_int * 8, cudaMemcpyDeviceToHost));
        ctx->h_int_stale = false;
    }
    const int64_t T = ctx->n_bca + ctx->n_bcb + ctx->n_ic + ctx->n_poy + ctx->n_int;
    ctx->ld = T;
    ctx->int_off_prev = ctx->n_bca + ctx->n_bcb + ctx->n_ic + ctx->n_poy;
    // host-assembled rows: all of them, or only the replicated ones when the
    // interior is a device design (no host copy of a 64M-point set)
    const int64_t Th = ctx->int_on_device ? T - ctx->n_int : T;
    std::vector<double> all((size_t)(d * Th));
    auto put = [&](const std::vector<double>& src, int64_t n, int64_t at) {
        for (int a = 0; a < d; ++a)
            for (int64_t i = 0; i < n; ++i) all[(size_t)(a * Th + at + i)] = src[(size_t)(a * n + i)];
    };
    put(ctx->h_bca, ctx->n_bca, 0);
    put(ctx->h_bcb, ctx->n_bcb, ctx->n_bca);
    put(ctx->h_ic, ctx->n_ic, ctx->n_bca + ctx->n_bcb);
    put(ctx->h_poy, ctx->n_poy, ctx->n_bca + ctx->n_bcb + ctx->n_ic);
    if (!ctx->int_on_device) {
        put(ctx->h_int, ctx->n_int, ctx->n_bca + ctx->n_bcb + ctx->n_ic + ctx->n_poy);
        if (int r = causality_counts(ctx, ctx->h_int.data() + (size_t)(d - 1) * ctx->n_int, ctx->n_int)) return r;
    }
    if (d * T > ctx->coords_cap) {
        if (int r = dalloc(ctx, &ctx->d_coords, (size_t)(d * T))) return r;
        ctx->coords_cap = d * T;
    }
    if (ctx->int_on_device) {  // replicated rows from the host, the interior from the device design
        for (int a = 0; a < d && Th > 0; ++a)
            CK(cudaMemcpy(ctx->d_coords + a * T, all.data() + (size_t)(a * Th), (size_t)Th * 8,
                          cudaMemcpyHostToDevice));
        if (int r = generate_interior(ctx)) return r;
    } else {
        CK(cudaMemcpy(ctx->d_coords, all.data(), all.size() * 8, cudaMemcpyHostToDevice));
    }
    if (int r = dalloc(ctx, &ctx->d_ic_t, ctx->h_ic_t.size())) return r;
    if (!ctx->h_ic_t.empty())
        CK(cudaMemcpy(ctx->d_ic_t, ctx->h_ic_t.data(), ctx->h_ic_t.size() * 4, cudaMemcpyHostToDevice));
    if (int r = dalloc(ctx, &ctx->d_bc_t, ctx->h_bc_t.size())) return r;
    if (!ctx->h_bc_t.empty())
        CK(cudaMemcpy(ctx->d_bc_t, ctx->h_bc_t.data(), ctx->h_bc_t.size() * 4, cudaMemcpyHostToDevice));
    if (int r = dalloc(ctx, &ctx->d_bc_vals, (size_t)std::max<int64_t>(1, ctx->n_bca + ctx->n_bcb) * ctx->F)) return r;
    {
        const double inv[3] = {1.0 / (double)ctx->n_int, ctx->n_ic ? 1.0 / (double)ctx->n_ic : 0.0,
                               ctx->n_bca ? 1.0 / (double)ctx->n_bca : 0.0};
        CK(cudaMemcpy(ctx->d_losses + 3, inv, sizeof(inv), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(reinterpret_cast<char*>(ctx->d_losses + 8), ctx->period_off, sizeof(ctx->period_off),
                      cudaMemcpyHostToDevice));
    }

    if (T == ctx->layout_T && ctx->chunk_override == ctx->layout_chunk_override) {
        ctx->rows_dirty = false;
        return PNX_OK;  // same row count: keep chunking, activations and partials
    }
    ctx->layout_T = T;
    ctx->layout_chunk_override = ctx->chunk_override;
    // chunking: all small rows in chunk 0
    const int64_t small = ctx->n_bca + ctx->n_bcb + ctx->n_ic + ctx->n_poy;
    int64_t ch = ctx->chunk_override;
    if (ch <= 0) {
        const int64_t budget = 48LL << 30;  // bytes of per-chunk activations
        ch = std::max<int64_t>(65536, budget / std::max<int64_t>(1, bytes_per_row(ctx)));
    }
    ch = std::max<int64_t>(ch, small + 128);
    ch = std::min<int64_t>(ch, T);
    ctx->chunk_rows = ch;
    const int64_t Rp = roundup(ch, 256);  // CTA-pair kernels tile 256 rows
    if (Rp > ctx->Rcap) {
        ctx->Rcap = Rp;
        const size_t SR = (size_t)ctx->S * Rp;
        if (int r = dalloc(ctx, &ctx->d_Hin, SR * ctx->K0)) return r;
        if (ctx->train_period)
            if (int r = dalloc(ctx, &ctx->d_Hinb, SR * ctx->K0)) return r;
        ctx->d_Z.assign(ctx->depth, nullptr);
        for (int l = 0; l < ctx->depth; ++l)
            if (int r = dalloc(ctx, &ctx->d_Z[l], SR * ctx->H)) return r;
        for (int i = 0; i < 2; ++i)
            if (int r = dalloc(ctx, &ctx->d_Zb[i], SR * ctx->H)) return r;
        CK(cudaMemset(ctx->d_Hin, 0, SR * ctx->K0 * 4));
        {
            const void* old[3] = {ctx->tc.red, ctx->tc.wpart, ctx->tc.dbpart};
            if (int r = tc_workspace_alloc(ctx->tc, (int)ctx->S, Rp, ctx->H, ctx->K0, guard_on() ? kGuardBytes : 0))
                return fail(ctx, r, "tc workspace alloc");
            void* now[3] = {ctx->tc.red, ctx->tc.wpart, ctx->tc.dbpart};
            const size_t bytes[3] = {(size_t)ctx->tc.red_cap * 8, (size_t)ctx->tc.wpart_cap * 4,
                                     (size_t)ctx->tc.dbpart_cap * 8};
            for (int i = 0; i < 3; ++i)
                if (now[i] != old[i]) {
                    guard_forget(ctx, old[i]);
                    if (int r = guard_add(ctx, now[i], bytes[i])) return r;
                }
        }
    }
    // wgrad splits per layer (fill ~4 waves of 148 SMs)
    const int L = ctx->tab.n;
    ctx->d_part.resize(L, nullptr);
    ctx->nsplit.assign(L, 1);
    for (int l = 0; l < L - 1; ++l) {
        const int tiles = (int)(((ctx->tab.N[l] + 63) / 64) * ((ctx->tab.K[l] + 63) / 64));
        int ns = std::max(1, std::min(256, (4 * 148 + tiles - 1) / tiles));
        ns = (int)std::min<int64_t>(ns, std::max<int64_t>(1, ch / 64));  // >= 64 rows per split
        if (l == 0 && layer0_fused(ctx)) ns = kL0Blocks;
        ctx->nsplit[l] = ns;
        if (int r = dalloc(ctx, &ctx->d_part[l], (size_t)ns * (ctx->tab.K[l] * (size_t)ctx->tab.N[l] + ctx->tab.N[l]))) return r;
    }
    ctx->rows_dirty = false;
    return PNX_OK;
}

// The whole step as one kernel (small_net.cuh) for narrow tanh networks: H <= 64,
// embedding only (no RFF, RWF or trainable period), first- or second-order
// 1-D / Maxwell layouts, hard or Dirichlet BC, no causality / Poynting, and the
// weights plus a 32-row tile of every layer's jets fit in shared memory.
// Taken by the default engine (AUTO); PNX_ENGINE_FFMA keeps the multi-kernel
// FFMA path (both are tested), PNX_SMALL_OFF=1 disables it (A/B).
int small_hp(const pnx_ctx* c) {
    static const bool off = getenv("PNX_SMALL_OFF") != nullptr;
    if (off || c->engine != PNX_ENGINE_AUTO) return 0;
    if (c->act != ACT_TANH || c->H > 64 || c->rff_w > 0 || c->rwf || c->train_period || c->E > SN_MAXK0) return 0;
    if (c->pde == PNX_PDE_NS_STEADY || c->bc == PNX_BC_SOFT_PERIODIC || c->caus_M > 0 || c->n_poy > 0) return 0;
    const int HP = c->H <= 32 ? 32 : 64;
    if (sn_smem_floats(HP, c->S, c->depth) * 4 > 227 * 1024) return 0;
    return HP;
}

int run_small(pnx_ctx* ctx, int HP, const float* d_params, const double lam[3], float* d_grad, double* d_losses,
              cudaStream_t st) {
    const int64_t T = ctx->ld;
    const int grid = (int)std::min<int64_t>(ctx->nsm, (T + SN_TR - 1) / SN_TR);
    if (!ctx->d_sn_slot)
        if (int r = dalloc(ctx, &ctx->d_sn_slot, (size_t)ctx->nsm * ctx->P)) return r;
    SmallArgs a{};
    a.ia.coords = ctx->d_coords;
    a.ia.ld = T;
    a.ia.in_dim = ctx->in_dim;
    for (int k = 0; k < kMaxAxes; ++k) {
        a.ia.periodic[k] = ctx->periodic[k];
        a.ia.period[k] = ctx->period[k];
        a.ia.period_off[k] = ctx->period_off[k];
    }
    a.ia.params = d_params;
    a.ia.E = ctx->E;
    a.ia.K0 = ctx->K0;
    a.params = d_params;
    a.tab = ctx->tab;
    a.D = ctx->depth;
    a.H = ctx->H;
    a.K0 = ctx->K0;
    a.T = T;
    a.bca0 = 0;
    a.bca1 = ctx->n_bca;
    a.ic0 = ctx->n_bca + ctx->n_bcb;
    a.ic1 = a.ic0 + ctx->n_ic;
    a.int0 = a.ic1 + ctx->n_poy;
    a.int1 = a.int0 + ctx->n_int;
    a.bc_mode = ctx->bc;
    a.ic_t = ctx->d_ic_t;
    a.bc_t = ctx->d_bc_t;
    a.w_pde = (float)(2.0 * lam[0] / (double)ctx->n_int);
    a.w_ic = ctx->n_ic ? (float)(2.0 * lam[1] / (double)ctx->n_ic) : 0.0f;
    a.w_bc = ctx->n_bca ? (float)(2.0 * lam[2] / (double)ctx->n_bca) : 0.0f;
    a.pc = ctx->pc;
    a.bad = ctx->d_bad;
    a.resid_out = ctx->capture_resid ? ctx->d_resid : nullptr;
    a.slot = ctx->d_sn_slot;
    a.loss_part = ctx->d_loss_part;
    a.P = ctx->P;
    prof_begin(ctx, PC_FUSED, st);
    if (launch_small(ctx->pde, HP, a, grid, st)) return fail(ctx, PNX_ERR_CUDA, "small-network step launch");
    prof_end(ctx, st);
    CKL();
    prof_begin(ctx, PC_FINAL, st);
    launch_small_finalize(ctx->d_sn_slot, grid, ctx->P, ctx->d_loss_part, ctx->d_losses + 3, d_grad,
                          d_losses ? d_losses : ctx->d_losses, st);
    prof_end(ctx, st);
    CKL();
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusNone) {
        CK(cudaEventRecord(ctx->ev_done, st));
        ctx->ev_pending = true;
    }
    return PNX_OK;
}

int run_step(pnx_ctx* ctx, const float* d_params, const double lam[3], float* d_grad, double* d_losses,
             cudaStream_t st) {
    if (ctx->n_int <= 0) return fail(ctx, PNX_ERR_STATE, "pnx_step: no interior points (call pnx_set_points)");
    if (ctx->rows_dirty)
        if (int r = upload_rows(ctx)) return r;
    ctx->launches = 0;
    if (const int HP = small_hp(ctx)) return run_small(ctx, HP, d_params, lam, d_grad, d_losses, st);
    const LayerTab& t = ctx->tab;
    const int Lw = t.n;  // linear layers
    const int S = ctx->S;
    const int L = ctx->layout;
    const int act = ctx->act;

    const bool reuse = ctx->reuse_fwd && ctx->ld <= ctx->chunk_rows;
    if (reuse)  // keep the |W| and |Z| bounds of the reused forward, reset the |Zb| ones
        CK(cudaMemsetAsync(amax_zb(ctx, 0), 0, kMaxLayers * kAmaxS * sizeof(unsigned), st));
    else
        CK(cudaMemsetAsync(ctx->d_amax, 0, kAmaxLen * sizeof(unsigned), st));
    {
        dim3 grid(64, Lw);
        k_prep<<<grid, 256, 0, st>>>(d_params, t, ctx->d_W, ctx->d_Wt, ctx->d_bias, ctx->d_amax);
        CKL();
    }
    for (int l = 0; l < Lw - 1; ++l)
        CK(cudaMemsetAsync(ctx->d_part[l], 0,
                           (size_t)ctx->nsplit[l] * (t.K[l] * (size_t)t.N[l] + t.N[l]) * 8, st));
    CK(cudaMemsetAsync(ctx->d_head_part, 0, (size_t)ctx->head_grid * (ctx->H * ctx->F + ctx->F) * 8, st));
    CK(cudaMemsetAsync(ctx->d_loss_part, 0, (size_t)ctx->head_grid * 3 * 8, st));
    CK(cudaMemsetAsync(ctx->d_partP, 0, (size_t)ctx->ibwd_grid * kMaxAxes * 8, st));

    const int64_t T = ctx->ld;
    const int64_t bca0 = 0, bca1 = ctx->n_bca, bcb0 = bca1, bcb1 = bcb0 + ctx->n_bcb;
    const int64_t ic0 = bcb1, ic1 = ic0 + ctx->n_ic, poy0 = ic1, poy1 = poy0 + ctx->n_poy, int0 = poy1,
                  int1 = int0 + ctx->n_int;
    const bool caus = ctx->caus_M > 0;
    const bool poy = ctx->n_poy > 0 && !ctx->no_penalty;
    const bool multi = T > ctx->chunk_rows;

    InputArgs ia{};
    ia.coords = ctx->d_coords;
    ia.ld = T;
    ia.in_dim = ctx->in_dim;
    for (int a = 0; a < kMaxAxes; ++a) {
        ia.periodic[a] = ctx->periodic[a];
        ia.period[a] = ctx->period[a];
        ia.period_off[a] = ctx->period_off[a];
    }
    ia.params = d_params;
    ia.E = ctx->E;
    ia.rff_w = ctx->rff_w;
    ia.rffB = ctx->d_rffB;
    ia.K0 = ctx->K0;
    ia.Hin = ctx->d_Hin;
    ia.amax_out = amax_hin(ctx);

    const bool tc_on = tc_enabled(ctx->engine, ctx->H, S, act);
    bool tc_fwd[kMaxLayers] = {}, tc_bwd[kMaxLayers] = {}, tc_wg[kMaxLayers] = {};
    // 3xFP16 per layer: the pair forward, fed by a producer that records |Z| bounds
    // (the fused layer 0 or another pair forward)
    bool f16_fwd[kMaxLayers] = {}, f16_bwd[kMaxLayers] = {}, f16_wg[kMaxLayers] = {};
    // debug/ablation: PNX_TC_MASK bit0 forward, bit1 reverse, bit2 weight-gradient (default all)
    static const int tc_mask = getenv("PNX_TC_MASK") ? atoi(getenv("PNX_TC_MASK")) : 7;
    if (tc_on) {
        const int NT = tc_nt(S);
        int64_t need = 0;
        for (int l = 0; l < ctx->depth; ++l) {
            tc_fwd[l] = tc_layer_ok(S, t.K[l], t.N[l]);
            tc_bwd[l] = l > 0 && tc_fwd[l] && t.K[l] % NT == 0 && (t.N[l] == 128 || t.N[l] == 256);
            if (tc_fwd[l]) {
                ctx->tc.img_fwd[l] = need;
                need += 2LL * t.K[l] * t.N[l];
            }
            if (tc_bwd[l]) {
                ctx->tc.img_bwd[l] = need;
                need += 2LL * t.K[l] * t.N[l];
            }
        }
        if (need > ctx->tc.img_cap) {
            if (ctx->tc.img) {
                guard_forget(ctx, ctx->tc.img);
                cudaFree(ctx->tc.img);
            }
            ctx->tc.img = nullptr;
            CK(cudaMalloc(&ctx->tc.img, need * sizeof(float) + (guard_on() ? kGuardBytes : 0)));
            if (int r = guard_add(ctx, ctx->tc.img, (size_t)need * sizeof(float))) return r;
            ctx->tc.img_cap = need;
        }
        // AUTO: 3xFP16 wherever the kernels support it, 3xTF32 elsewhere
        const bool f16 = ctx->engine == PNX_ENGINE_TC3XF16 || ctx->engine == PNX_ENGINE_AUTO;
        bool rec = layer0_fused(ctx);  // Z_{l-1} bounds recorded
        for (int l = 0; l < ctx->depth; ++l) {
            tc_wg[l] = tc_fwd[l] && (tc_mask & 4);
            if (!(tc_mask & 2)) tc_bwd[l] = false;
            // Zb_out bounds come from the head (last hidden layer) or the backward of
            // layer l+1; every tcgen05 forward / backward epilogue and the fused layer 0 / head
            // record their output bounds; every contraction kernel has a 3xFP16 variant
            // (the CTA-pair variant of the general backward does not: it is opt-in)
            const bool recb = l == ctx->depth - 1 || (tc_bwd[l + 1] && (tc_mask & 2));
            if (l > 0) {
                f16_fwd[l] = f16 && tc_fwd[l] && (tc_mask & 1) && rec;  // pair or single-CTA forward
                f16_wg[l] = f16 && tc_wg[l] && rec && recb;  // A = Z_{l-1}, B = Zb_l
                rec = tc_fwd[l] && (tc_mask & 1);
            } else if (!layer0_fused(ctx)) {
                // k_input records the bounds of the features it writes (RFF / wide embedding)
                f16_fwd[0] = f16 && tc_fwd[0] && (tc_mask & 1);
                f16_wg[0] = f16 && tc_wg[0] && recb;
                rec = tc_fwd[0] && (tc_mask & 1);  // the tcgen05 layer 0 records Z_0 bounds too
            }
            // the general (all streams in TMEM) backward gains from 3xFP16 only up to four
            // streams: at S = 5 (NS, N = 64 tiles) its producers bound it (3.04 vs 3.16 ms at C3)
            if (tc_bwd[l] && f16 && recb && (tc5_bwd_ok(L, t.K[l], t.N[l]) || S <= 4)) f16_bwd[l] = true;
            if (f16_fwd[l]) {
                k_tc_prep_image16<<<256, 256, 0, st>>>(ctx->d_W + t.dW[l], t.K[l], t.N[l], 0, t.N[l], amax_w(ctx, l),
                                                      reinterpret_cast<uint16_t*>(ctx->tc.img + ctx->tc.img_fwd[l]));
                CKL();
            } else if (tc_fwd[l]) {
                k_tc_prep_image<<<256, 256, 0, st>>>(ctx->d_W + t.dW[l], t.K[l], t.N[l], 0, t.N[l],
                                                    ctx->tc.img + ctx->tc.img_fwd[l]);
                CKL();
            }
            if (f16_bwd[l]) {
                k_tc_prep_image16<<<256, 256, 0, st>>>(ctx->d_W + t.dW[l], t.K[l], t.N[l], 1,
                                                      tc5_bwd_ok(L, t.K[l], t.N[l]) ? 256 : NT, amax_w(ctx, l),
                                                      reinterpret_cast<uint16_t*>(ctx->tc.img + ctx->tc.img_bwd[l]));
                CKL();
            } else if (tc_bwd[l]) {
                k_tc_prep_image<<<256, 256, 0, st>>>(ctx->d_W + t.dW[l], t.K[l], t.N[l], 1,
                                                    tc5_bwd_ok(L, t.K[l], t.N[l]) ? 256 : NT,
                                                    ctx->tc.img + ctx->tc.img_bwd[l]);
                CKL();
            }
        }
    }

    // forward of one chunk: input jets + hidden layers (Z_l of the chunk)
    auto forward_chunk = [&](int64_t c0, int nrows, int Rpad) -> int {
        const bool fuse0 = layer0_fused(ctx);
        ia.row0 = c0;
        ia.nrows = nrows;
        ia.Rpad = Rpad;
        if (!fuse0) {
            prof_begin(ctx, PC_INPUT, st);
            launch_input(L, ia, st);
            prof_end(ctx, st);
            CKL();
        }
        // forward layers
        for (int l = 0; l < ctx->depth; ++l) {
            GemmArgs g{};
            g.A = l == 0 ? ctx->d_Hin : ctx->d_Z[l - 1];
            g.B = ctx->d_W + t.dW[l];
            g.bias = ctx->d_bias + t.dB[l];
            g.out = ctx->d_Z[l];
            g.Rpad = Rpad;
            g.K = t.K[l];
            g.N = t.N[l];
            g.w0 = ctx->w0;
            const int pro = l == 0 ? ACT_NONE : act;
            prof_begin(ctx, PC_FWD, st);
            if (l == 0 && fuse0) {
                launch_layer0_fwd(L, act, ia, g.B, g.bias, g.out, g.N, amax_z(ctx, 0), st);
                CKL();
            } else if (tc_fwd[l] && (tc_mask & 1)) {
                TcGemmArgs tg{};
                tg.A = g.A;
                tg.img = ctx->tc.img + ctx->tc.img_fwd[l];
                tg.bias = g.bias;
                tg.out = g.out;
                tg.Rpad = Rpad;
                tg.K = g.K;
                tg.N = g.N;
                tg.f16 = f16_fwd[l] ? 1 : 0;
                tg.amax_in = l > 0 ? amax_z(ctx, l - 1) : amax_hin(ctx);
                tg.amax_w = amax_w(ctx, l);
                tg.amax_out = amax_z(ctx, l);
                if (launch_tc2_fwd(L, pro, tg, st)) return fail(ctx, PNX_ERR_CUDA, "tc forward launch");
                CKL();
            } else {
                launch_gemm(L, pro, EPI_BIAS, act, g, st);
                CKL();
            }
            prof_end(ctx, st);
        }
        return PNX_OK;
    };
    auto head_args = [&](int64_t c0, int nrows, int Rpad) {
        HeadArgs h{};
        h.Z = ctx->d_Z[ctx->depth - 1];
        h.Zb = ctx->d_Zb[0];
        h.zb_amax = amax_zb(ctx, ctx->depth - 1);
        h.W = ctx->d_W + t.dW[Lw - 1];
        h.b = ctx->d_bias + t.dB[Lw - 1];
        h.H = ctx->H;
        h.Rpad = Rpad;
        h.nrows = nrows;
        h.row0 = c0;
        h.bca0 = bca0; h.bca1 = bca1; h.bcb0 = bcb0; h.bcb1 = bcb1;
        h.ic0 = ic0; h.ic1 = ic1; h.int0 = int0; h.int1 = int1;
        h.bc_mode = ctx->bc;
        h.ic_t = ctx->d_ic_t;
        h.bc_t = ctx->d_bc_t;
        h.bc_vals = ctx->d_bc_vals;
        h.w_pde = (float)(2.0 * lam[0] / (double)ctx->n_int);
        h.w_ic = ctx->n_ic ? (float)(2.0 * lam[1] / (double)ctx->n_ic) : 0.0f;
        h.w_bc = ctx->n_bca ? (float)(2.0 * lam[2] / (double)ctx->n_bca) : 0.0f;
        h.pc = ctx->pc;
        h.w0 = ctx->w0;
        h.loss_part = ctx->d_loss_part;
        h.head_part = ctx->d_head_part;
        h.bad = ctx->d_bad;
        h.resid_out = ctx->capture_resid ? ctx->d_resid : nullptr;
        h.tcoord = ctx->d_coords + (int64_t)(ctx->in_dim - 1) * T;
        if (caus) {
            h.seg_M = ctx->caus_M;
            h.seg_tlo = ctx->caus_tlo;
            h.seg_span = ctx->caus_thi - ctx->caus_tlo;
            h.seg_w = ctx->d_seg_w;
            h.seg_part = ctx->d_seg_part;
        }
        if (poy) {
            h.poy0 = poy0;
            h.poy1 = poy1;
            h.poy_T = ctx->poy_T;
            h.poy_n2 = ctx->poy_grid * ctx->poy_grid;
            h.poy_g = ctx->d_poy_g;
            h.poy_part = ctx->d_poy_part;
        }
        return h;
    };
    // stats pre-pass over chunk rows [0, rows_end) + the weight kernels
    auto stats_chunk = [&](int64_t c0, int nrows, int Rpad, int rows_end) {
        HeadArgs hs = head_args(c0, nrows, Rpad);
        hs.stats = 1;
        hs.nrows = rows_end;
        launch_head(ctx->pde, act, hs, ctx->head_grid, st);
    };
    auto weights = [&]() -> int {
        if (caus) {
            k_causality_weights<<<1, 32, 0, st>>>(ctx->d_seg_part, ctx->head_grid, ctx->caus_M, ctx->d_caus_cnt,
                                                  ctx->caus_eps, lam[0], ctx->d_seg_w, ctx->d_caus_loss);
            CKL();
        }
        if (poy) {
            const double cell = (ctx->poy_box[1] - ctx->poy_box[0]) / ctx->poy_grid *
                                ((ctx->poy_box[3] - ctx->poy_box[2]) / ctx->poy_grid);
            k_poynting_weights<<<1, 32, 0, st>>>(ctx->d_poy_part, ctx->head_grid, ctx->poy_T, cell, ctx->res_eps,
                                                 ctx->res_mu, ctx->poy_w, ctx->d_poy_g, ctx->d_pen);
            CKL();
        }
        return PNX_OK;
    };
    if (caus) CK(cudaMemsetAsync(ctx->d_seg_part, 0, (size_t)ctx->head_grid * ctx->caus_M * 8, st));
    if (poy) CK(cudaMemsetAsync(ctx->d_poy_part, 0, (size_t)ctx->head_grid * 2 * ctx->poy_T * 8, st));
    if (caus && multi) {  // segment losses need every chunk before any seed
        for (int64_t c0 = 0; c0 < T; c0 += ctx->chunk_rows) {
            const int nrows = (int)std::min<int64_t>(ctx->chunk_rows, T - c0);
            const int Rpad = (int)roundup(nrows, 256);
            if (int r = forward_chunk(c0, nrows, Rpad)) return r;
            stats_chunk(c0, nrows, Rpad, nrows);
            CKL();
        }
        if (int r = weights()) return r;
    }

    for (int64_t c0 = 0; c0 < T; c0 += ctx->chunk_rows) {
        const int nrows = (int)std::min<int64_t>(ctx->chunk_rows, T - c0);
        const int Rpad = (int)roundup(nrows, 256);
        const bool fuse0 = layer0_fused(ctx);
        if (reuse) {  // the chunk's input arguments (layer-0 weight gradient, input backward)
            ia.row0 = c0;
            ia.nrows = nrows;
            ia.Rpad = Rpad;
        } else if (int r = forward_chunk(c0, nrows, Rpad)) {
            return r;
        }
        HeadArgs h = head_args(c0, nrows, Rpad);
        if (!multi && (caus || poy)) {
            stats_chunk(c0, nrows, Rpad, nrows);
            CKL();
            if (int r = weights()) return r;
        } else if (multi && !caus && poy && c0 == 0) {
            stats_chunk(c0, nrows, Rpad, (int)std::min<int64_t>(nrows, poy1));
            CKL();
            if (int r = weights()) return r;
        }
        if (ctx->bc == PNX_BC_SOFT_PERIODIC && c0 == 0) {
            HeadArgs hv = h;
            hv.values_only = 1;
            hv.vals_out = ctx->d_bc_vals;
            hv.nrows = (int)std::min<int64_t>(nrows, bcb1);
            launch_head(ctx->pde, act, hv, ctx->head_grid, st);
            CKL();
        }
        prof_begin(ctx, PC_HEAD, st);
        launch_head(ctx->pde, act, h, ctx->head_grid, st);
        prof_end(ctx, st);
        CKL();
        // reverse layers
        int cur = 0;
        for (int l = ctx->depth - 1; l >= 0; --l) {
            WgradArgs w{};
            w.A = l == 0 ? ctx->d_Hin : ctx->d_Z[l - 1];
            w.Bm = ctx->d_Zb[cur];
            w.part = ctx->d_part[l];
            w.Rpad = Rpad;
            w.nrows_valid = nrows;
            w.K = t.K[l];
            w.N = t.N[l];
            w.rows_per_split = (int)roundup((nrows + ctx->nsplit[l] - 1) / ctx->nsplit[l], WT_R);
            w.w0 = ctx->w0;
            const int pro = l == 0 ? ACT_NONE : act;
            prof_begin(ctx, PC_WGRAD, st);
            if (l == 0 && fuse0) {
                launch_layer0_wgrad(L, ia, w.Bm, t.N[0], ctx->d_part[0], kL0Blocks, st);
                CKL();
            } else if (tc_wg[l]) {
                TcWgradArgs tw{};
                tw.A = w.A;
                tw.Bm = w.Bm;
                tw.wpart = ctx->tc.wpart;
                tw.dbpart = ctx->tc.dbpart;
                tw.Rpad = Rpad;
                tw.nrows = nrows;
                tw.Kin = t.K[l];
                tw.N = t.N[l];
                tw.f16 = f16_wg[l] ? 1 : 0;
                tw.amaxA = l > 0 ? amax_z(ctx, l - 1) : amax_hin(ctx);
                tw.amaxB = amax_zb(ctx, l);
                const int ntl = std::min(tc_wgrad_groups(Rpad, t.K[l], ctx->nsm), TC_WG_MAX_GROUPS);
                const int wr = tc_wgrad_seg();
                CK(cudaMemsetAsync(ctx->tc.wpart, 0, (size_t)ntl * t.K[l] * t.N[l] * sizeof(float), st));
                if (launch_tc2_wgrad(L, pro, tw, ntl, wr, st)) return fail(ctx, PNX_ERR_CUDA, "tc wgrad launch");
                CKL();
                {
                    const int64_t len = (int64_t)t.K[l] * t.N[l] + t.N[l];
                    const unsigned gx = (unsigned)std::min<int64_t>((len / 4 + 255) / 256, 1024);
                    k_tc_wreduce1<<<dim3(gx, TC_WRED_G), 256, 0, st>>>(ctx->tc.wpart, ctx->tc.dbpart, ntl, t.K[l],
                                                                       t.N[l], ctx->tc.red);
                    CKL();
                    k_tc_wreduce2<<<(unsigned)std::min<int64_t>((len + 255) / 256, 1024), 256, 0, st>>>(
                        ctx->tc.red, len, ctx->d_part[l]);
                }
                CKL();
            } else {
                launch_wgrad(L, pro, w, ctx->nsplit[l], st);
                CKL();
            }
            prof_end(ctx, st);
            if (l > 0 || ctx->train_period) {
                GemmArgs g{};
                g.A = ctx->d_Zb[cur];
                g.B = ctx->d_Wt + t.dW[l];  // [N_l][K_l]
                g.Rpad = Rpad;
                g.K = t.N[l];
                g.N = t.K[l];
                g.w0 = ctx->w0;
                if (l > 0) {
                    g.Zlow = ctx->d_Z[l - 1];
                    g.out = ctx->d_Zb[cur ^ 1];
                    prof_begin(ctx, PC_BWD, st);
                    if (tc_bwd[l]) {
                        TcGemmArgs tg{};
                        tg.A = g.A;
                        tg.img = ctx->tc.img + ctx->tc.img_bwd[l];
                        tg.Zlow = g.Zlow;
                        tg.out = g.out;
                        tg.Rpad = Rpad;
                        tg.K = g.K;
                        tg.N = g.N;
                        tg.f16 = f16_bwd[l] ? 1 : 0;
                        tg.amax_in = amax_zb(ctx, l);
                        tg.amax_w = amax_w(ctx, l);
                        tg.amax_out = amax_zb(ctx, l - 1);
                        if (launch_tc_layer(L, 1, ACT_NONE, tg, st)) return fail(ctx, PNX_ERR_CUDA, "tc backward launch");
                        CKL();
                    } else {
                        launch_gemm(L, ACT_NONE, EPI_ACTT, act, g, st);
                        CKL();
                    }
                    prof_end(ctx, st);
                    cur ^= 1;
                } else {
                    g.out = ctx->d_Hinb;
                    launch_gemm(L, ACT_NONE, EPI_RAW, ACT_NONE, g, st);
                    CKL();
                    launch_input_bwd(L, ia, ctx->d_Hinb, ctx->d_partP, ctx->ibwd_grid, st);
                    CKL();
                }
            }
        }
    }
    // finalize: fixed-order reductions, trainable() order
    for (int l = 0; l < Lw; ++l) {
        const double* part = l < Lw - 1 ? ctx->d_part[l] : ctx->d_head_part;
        const int ns = l < Lw - 1 ? ctx->nsplit[l] : ctx->head_grid;
        const int64_t len = (int64_t)t.K[l] * t.N[l] + t.N[l];
        k_reduce_splits<<<reduce_splits_grid(len), kRsX * kRsY, 0, st>>>(part, ns, len, ctx->d_red);
        CKL();
        k_write_layer_grad<<<(unsigned)std::min<int64_t>((len + 255) / 256, 1024), 256, 0, st>>>(
            ctx->d_red, d_params, t.K[l], t.N[l], t.offW[l], t.offS[l], t.offB[l], 1.0f, d_grad);
        CKL();
        if (t.offS[l] >= 0) {
            k_write_rwf_ds<<<(unsigned)((t.N[l] + 7) / 8), 256, 0, st>>>(ctx->d_red, d_params, t.K[l], t.N[l], t.offW[l],
                                                                       t.offS[l], 1.0f, d_grad);
            CKL();
        }
    }
    {
        // 1/n per term and the period offsets live in d_losses[3..] (uploaded with the
        // rows, so the step itself enqueues kernels and memsets only: graph-capturable)
        k_write_scalar_grads<<<1, kScalarGradThreads, 0, st>>>(ctx->d_partP, ctx->ibwd_grid,
                                               reinterpret_cast<const int64_t*>(ctx->d_losses + 8), ctx->in_dim,
                                               1.0f, d_grad, ctx->d_loss_part, ctx->head_grid, ctx->d_losses + 3,
                                               d_losses ? d_losses : ctx->d_losses,
                                               caus ? ctx->d_caus_loss : nullptr);
        CKL();
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusNone) {  // a captured step is ordered by its replays' stream
        CK(cudaEventRecord(ctx->ev_done, st));
        ctx->ev_pending = true;
    }
    return PNX_OK;
}

// Host-side writes of step inputs (points, targets) must not overtake a step
// still reading them on the caller's stream (pnx_step_device is asynchronous).
int wait_last_step(pnx_ctx* ctx) {
    if (ctx->ev_pending) {
        CK(cudaEventSynchronize(ctx->ev_done));
        ctx->ev_pending = false;
    }
    return PNX_OK;
}

// name of the trainable() tensor holding flat entry i (model.cpp:64-101)
std::string param_name(const pnx_ctx* ctx, int64_t i) {
    const LayerTab& t = ctx->tab;
    for (int l = 0; l < t.n; ++l) {
        const std::string L = "layer" + std::to_string(l);
        if (i >= t.offW[l] && i < t.offW[l] + (int64_t)t.K[l] * t.N[l]) return L + (ctx->rwf ? ".V" : ".W");
        if (t.offS[l] >= 0 && i >= t.offS[l] && i < t.offS[l] + t.N[l]) return L + ".s";
        if (i >= t.offB[l] && i < t.offB[l] + t.N[l]) return L + ".b";
    }
    for (int a = 0; a < kMaxAxes; ++a)
        if (ctx->period_off[a] == i) return "periodic.P" + std::to_string(a);
    return "?";
}

}  // namespace

namespace pnx {
const double* ctx_penalty_ptr(pnx_ctx* c) { return c->n_poy > 0 && c->d_pen ? c->d_pen : nullptr; }
void set_create_error(const std::string& m) { g_create_error = m; }
}  // namespace pnx

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* pnx_create_error(void) { return g_create_error.c_str(); }

int pnx_create(const pnx_model_desc* m, const pnx_problem_desc* p, int device, pnx_ctx** out) {
    g_create_error.clear();
    if (!m || !p || !out) {
        g_create_error = "pnx_create: null argument";
        return PNX_ERR_ARG;
    }
    *out = nullptr;
    // ModelSpec::validate (model.cpp:25-33)
    if (m->in_dim <= 0 || m->hidden_dim <= 0 || m->depth <= 0 || m->out_dim <= 0) {
        g_create_error = "ModelSpec: dimensions must be positive";
        return PNX_ERR_ARG;
    }
    if (m->n_periodic_axes != 0 && m->n_periodic_axes != m->in_dim) {
        g_create_error = "ModelSpec: periodic_axes must have one entry per input axis";
        return PNX_ERR_ARG;
    }
    if (m->in_dim > kMaxAxes || m->depth + 1 > kMaxLayers) {
        g_create_error = "pnx_create: in_dim <= 4 and depth <= 15 supported";
        return PNX_ERR_ARG;
    }
    if (m->hidden_dim > 512) {
        g_create_error = "pnx_create: hidden_dim <= 512 supported";
        return PNX_ERR_ARG;
    }
    const int layout = pde_layout(p->pde);
    if (layout < 0) {
        g_create_error = "unknown pde";
        return PNX_ERR_ARG;
    }
    const bool mx = p->pde == PNX_PDE_MAXWELL_TE || p->pde == PNX_PDE_MAXWELL_TE_EH;
    const int fields = (mx || p->pde == PNX_PDE_NS_STEADY) ? 3 : 1;
    const int coords = mx ? 3 : 2;
    if (m->out_dim != fields) {  // losses.cpp:31-32
        g_create_error = "residual: model field count does not match the equation";
        return PNX_ERR_ARG;
    }
    if (m->in_dim != coords) {  // losses.cpp:29-30
        g_create_error = "residual: coordinate count mismatch";
        return PNX_ERR_ARG;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        g_create_error = "pnx_create: no CUDA device (the B200 path has no CPU fallback)";
        return PNX_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) {
        g_create_error = "pnx_create: bad device index";
        return PNX_ERR_ARG;
    }
    if (cudaSetDevice(device) != cudaSuccess) {
        g_create_error = "pnx_create: cudaSetDevice failed";
        return PNX_ERR_CUDA;
    }
    pnx_ctx* ctx = new pnx_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device);
    ctx->head_grid = kHeadBlocks * ctx->nsm;
    ctx->in_dim = m->in_dim;
    ctx->H = m->hidden_dim;
    ctx->depth = m->depth;
    ctx->F = m->out_dim;
    ctx->act = m->activation;
    ctx->w0 = (float)m->sine_w0;
    ctx->rwf = m->rwf != 0;
    ctx->rff_w = m->rff_width;
    int E = 0;
    for (int a = 0; a < m->in_dim; ++a) {
        const bool per = m->n_periodic_axes && m->periodic[a];
        ctx->periodic[a] = per;
        if (per) {
            if (!(m->period[a] > 0.0)) {
                g_create_error = "ModelSpec: periodic axis needs a positive period";
                delete ctx;
                return PNX_ERR_ARG;
            }
            ctx->period[a] = m->period[a];
        }
        E += per ? 2 : 1;
    }
    ctx->E = E;
    ctx->K0 = ctx->rff_w > 0 ? 2 * ctx->rff_w : E;
    ctx->pde = p->pde;
    ctx->bc = p->bc;
    ctx->layout = layout;
    ctx->pc.c = (float)p->advection_c;
    ctx->pc.eps = (float)p->epsilon;
    ctx->pc.mu = (float)p->mu;
    ctx->res_eps = p->epsilon;
    ctx->res_mu = p->mu;
    ctx->pc.inv_re = p->reynolds > 0 ? (float)(1.0 / p->reynolds) : 0.0f;
    switch (layout) {
        case LAY_XT: ctx->S = 3; break;
        case LAY_AC: ctx->S = 4; break;
        case LAY_MX: ctx->S = 4; break;
        case LAY_NS: ctx->S = 5; break;
    }
    ctx->Kres = fields;
    // parameter layout (model.cpp:64-101)
    LayerTab& t = ctx->tab;
    t.n = m->depth + 1;
    int64_t off = 0, dw = 0, db = 0;
    for (int l = 0; l < t.n; ++l) {
        const int K = l == 0 ? ctx->K0 : ctx->H;
        const int N = l == m->depth ? ctx->F : ctx->H;
        t.K[l] = K;
        t.N[l] = N;
        t.offW[l] = off;
        off += (int64_t)K * N;
        if (ctx->rwf) {
            t.offS[l] = off;
            off += N;
        } else {
            t.offS[l] = -1;
        }
        t.offB[l] = off;
        off += N;
        t.dW[l] = dw;
        dw += (int64_t)K * N;
        t.dB[l] = db;
        db += N;
    }
    for (int a = 0; a < m->in_dim; ++a) {
        if (ctx->periodic[a] && m->period_trainable && m->period_trainable[a]) {
            ctx->period_off[a] = off++;
            ctx->train_period = true;
        }
    }
    ctx->P = off;
    ctx->wsize = dw;
    ctx->bsize = db;
    int rc = PNX_OK;
    cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if ((rc = dalloc(ctx, &ctx->d_W, dw)) || (rc = dalloc(ctx, &ctx->d_Wt, dw)) ||
        (rc = dalloc(ctx, &ctx->d_bias, db)) || (rc = dalloc(ctx, &ctx->d_params, ctx->P)) ||
        (rc = dalloc(ctx, &ctx->d_grad, ctx->P)) || (rc = dalloc(ctx, &ctx->d_losses, 16)) ||
        (rc = dalloc(ctx, &ctx->d_head_part, (size_t)ctx->head_grid * (ctx->H * ctx->F + ctx->F))) ||
        (rc = dalloc(ctx, &ctx->d_loss_part, (size_t)ctx->head_grid * 3)) ||
        (rc = dalloc(ctx, &ctx->d_partP, (size_t)ctx->ibwd_grid * kMaxAxes)) ||
        (rc = dalloc(ctx, &ctx->d_bad, 8)) || (rc = dalloc(ctx, &ctx->d_amax, kAmaxLen)) ||
        (rc = (cudaMemset(ctx->d_bad, 0x7f, 8 * sizeof(int)) == cudaSuccess ? PNX_OK : PNX_ERR_CUDA)) ||
        (rc = (cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming) == cudaSuccess ? PNX_OK
                                                                                                : PNX_ERR_CUDA))) {
        g_create_error = ctx->err;
        pnx_destroy(ctx);
        return rc;
    }
    int64_t redmax = 0;
    for (int l = 0; l < t.n; ++l) redmax = std::max<int64_t>(redmax, (int64_t)t.K[l] * t.N[l] + t.N[l]);
    if ((rc = dalloc(ctx, &ctx->d_red, redmax))) {
        g_create_error = ctx->err;
        pnx_destroy(ctx);
        return rc;
    }
    if (ctx->rff_w > 0) {
        if (!m->rff_B) {
            g_create_error = "pnx_create: rff_B required when rff_width > 0";
            pnx_destroy(ctx);
            return PNX_ERR_ARG;
        }
        const size_t nB = (size_t)E * ctx->rff_w;
        if ((rc = dalloc(ctx, &ctx->d_rffB, nB)) ||
            cudaMemcpy(ctx->d_rffB, m->rff_B, nB * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
            g_create_error = "pnx_create: rff_B upload failed";
            pnx_destroy(ctx);
            return PNX_ERR_CUDA;
        }
    }
    *out = ctx;
    return PNX_OK;
}

void pnx_destroy(pnx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaFree(ctx->d_coords);
    cudaFree(ctx->d_ic_t);
    cudaFree(ctx->d_bc_t);
    cudaFree(ctx->d_rffB);
    cudaFree(ctx->d_W);
    cudaFree(ctx->d_Wt);
    cudaFree(ctx->d_bias);
    cudaFree(ctx->d_params);
    cudaFree(ctx->d_grad);
    cudaFree(ctx->d_losses);
    cudaFree(ctx->d_Hin);
    cudaFree(ctx->d_Hinb);
    for (float* z : ctx->d_Z) cudaFree(z);
    cudaFree(ctx->d_Zb[0]);
    cudaFree(ctx->d_Zb[1]);
    for (double* p : ctx->d_part) cudaFree(p);
    cudaFree(ctx->d_head_part);
    cudaFree(ctx->d_loss_part);
    cudaFree(ctx->d_partP);
    cudaFree(ctx->d_red);
    cudaFree(ctx->d_bc_vals);
    cudaFree(ctx->d_caus_cnt);
    cudaFree(ctx->d_seg_part);
    cudaFree(ctx->d_caus_loss);
    cudaFree(ctx->d_seg_w);
    cudaFree(ctx->d_poy_part);
    cudaFree(ctx->d_poy_g);
    cudaFree(ctx->d_pen);
    cudaFree(ctx->d_bad);
    cudaFree(ctx->d_amax);
    cudaFree(ctx->d_resid);
    cudaFree(ctx->d_sn_slot);
    tc_workspace_free(ctx->tc);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    if (ctx->g_exec) cudaGraphExecDestroy(ctx->g_exec);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* pnx_last_error(const pnx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pnx_param_count(const pnx_ctx* ctx, int64_t* n) {
    if (!ctx || !n) return PNX_ERR_ARG;
    *n = ctx->P;
    return PNX_OK;
}

int pnx_set_points(pnx_ctx* ctx, const double* coords, int64_t n, int32_t n_axes) {
    if (!ctx) return PNX_ERR_ARG;
    if (n_axes != ctx->in_dim) return fail(ctx, PNX_ERR_ARG, "residual: coordinate count mismatch");
    if (n <= 0 || !coords) return fail(ctx, PNX_ERR_ARG, "residual_loss: empty point set");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->rows_dirty && n == ctx->n_int && ctx->d_coords) {
        ctx->int_on_device = false;
        // same row layout (e.g. resampled points, trainer.cpp:421-434): copy the
        // caller's axis-major buffer straight into the interior segment on device
        const int64_t off = ctx->int_off_prev;
        if (int r = wait_last_step(ctx)) return r;  // the previous step may still read d_coords
        for (int a = 0; a < n_axes; ++a)
            CK(cudaMemcpyAsync(ctx->d_coords + a * ctx->ld + off, coords + a * n, (size_t)n * 8,
                               cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->h_int_stale = true;
        return causality_counts(ctx, coords + (int64_t)(n_axes - 1) * n, n);
    }
    ++ctx->state_ver;  // new row layout (the same-size path above only rewrites device memory)
    ctx->h_int.assign(coords, coords + n * n_axes);
    ctx->h_int_stale = false;
    ctx->int_on_device = false;
    ctx->n_int = n;
    ctx->rows_dirty = true;
    if ((int64_t)n * ctx->Kres > ctx->resid_cap) {
        if (int r = dalloc(ctx, &ctx->d_resid, (size_t)n * ctx->Kres)) return r;
        ctx->resid_cap = (int64_t)n * ctx->Kres;
    }
    return PNX_OK;
}

int pnx_sample_points(pnx_ctx* ctx, int32_t mode, const double* bounds, const int64_t* dims, int64_t n_total,
                      uint64_t seed, int64_t row_lo, int64_t row_hi) {
    if (!ctx || !bounds) return PNX_ERR_ARG;
    ++ctx->state_ver;
    const int d = ctx->in_dim;
    SampleArgs a{};
    a.mode = mode;
    a.d = d;
    a.seed = seed;
    int64_t total = 1;
    for (int k = 0; k < d; ++k) {
        a.lo[k] = bounds[2 * k];
        a.hi[k] = bounds[2 * k + 1];
        if (mode != SAMPLE_LHS) {
            if (!dims || dims[k] <= 0) return fail(ctx, PNX_ERR_ARG, "sample_uniform: zero points on an axis");
            a.dims[k] = dims[k];
            total *= dims[k];
        }
    }
    if (mode == SAMPLE_LHS) {
        if (n_total <= 0) return fail(ctx, PNX_ERR_ARG, "sample_lhs: n must be positive");
        total = n_total;
    } else if (mode != SAMPLE_UNIFORM && mode != SAMPLE_LHS_PER_AXIS) {
        return fail(ctx, PNX_ERR_ARG, "pnx_sample_points: unknown design");
    }
    if (row_lo < 0 || row_hi > total || row_hi <= row_lo)
        return fail(ctx, PNX_ERR_ARG, "residual_loss: empty point set");
    a.n = total;
    a.row0 = row_lo;
    a.nrows = row_hi - row_lo;
    CK(cudaSetDevice(ctx->device));
    ctx->samp = a;
    if (!ctx->rows_dirty && a.nrows == ctx->n_int && ctx->d_coords) {
        // same row layout (resampling, trainer.cpp:421-434): generate in place
        if (int r = wait_last_step(ctx)) return r;
        ctx->int_on_device = true;
        ctx->h_int_stale = false;
        return generate_interior(ctx);
    }
    ctx->h_int.clear();
    ctx->h_int_stale = false;
    ctx->int_on_device = true;
    ctx->n_int = a.nrows;
    ctx->rows_dirty = true;  // laid out (and generated) by the next step
    if (a.nrows * ctx->Kres > ctx->resid_cap) {
        if (int r = dalloc(ctx, &ctx->d_resid, (size_t)a.nrows * ctx->Kres)) return r;
        ctx->resid_cap = a.nrows * ctx->Kres;
    }
    return PNX_OK;
}

int pnx_set_causality(pnx_ctx* ctx, int32_t segments, double epsilon, double t_lo, double t_hi) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    CK(cudaSetDevice(ctx->device));
    if (segments <= 0) {
        ctx->caus_M = 0;
        return PNX_OK;
    }
    if (segments > kStatMax) return fail(ctx, PNX_ERR_ARG, "causality: at most 64 segments");
    if (!(t_hi > t_lo)) return fail(ctx, PNX_ERR_ARG, "causality: empty time interval");
    ctx->caus_M = segments;
    ctx->caus_eps = epsilon;
    ctx->caus_tlo = t_lo;
    ctx->caus_thi = t_hi;
    if (int r = dalloc(ctx, &ctx->d_caus_cnt, (size_t)segments)) return r;
    if (int r = dalloc(ctx, &ctx->d_seg_part, (size_t)ctx->head_grid * segments)) return r;
    if (int r = dalloc(ctx, &ctx->d_caus_loss, 1)) return r;
    if (int r = dalloc(ctx, &ctx->d_seg_w, (size_t)segments)) return r;
    CK(cudaMemset(ctx->d_caus_cnt, 0, (size_t)segments * 8));
    if (ctx->n_int > 0) {  // counts of the current shard
        if (ctx->int_on_device) {
            if (!ctx->rows_dirty && ctx->d_coords) {
                if (int r = wait_last_step(ctx)) return r;
                if (int r = generate_interior(ctx)) return r;  // regenerates and recounts
            }
        } else if (ctx->h_int_stale || ctx->rows_dirty) {
            ctx->rows_dirty = true;  // recounted by the next upload
        } else {
            if (int r = causality_counts(ctx, ctx->h_int.data() + (size_t)(ctx->in_dim - 1) * ctx->n_int, ctx->n_int))
                return r;
        }
    }
    return PNX_OK;
}

int pnx_set_poynting(pnx_ctx* ctx, double weight, int32_t grid, int32_t time_samples, const double box[6]) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    CK(cudaSetDevice(ctx->device));
    if (weight == 0.0 || ctx->pde != PNX_PDE_MAXWELL_TE) {  // trainer.cpp:240: maxwell_te only
        if (ctx->n_poy) ctx->rows_dirty = true;
        ctx->poy_w = 0.0;
        ctx->n_poy = 0;
        ctx->h_poy.clear();
        return PNX_OK;
    }
    if (time_samples < 2) return fail(ctx, PNX_ERR_ARG, "poynting_penalty: need at least 2 time samples");
    if (time_samples > kStatMax || grid <= 0 || !box) return fail(ctx, PNX_ERR_ARG, "poynting_penalty: bad grid");
    ctx->poy_w = weight;
    if (grid == ctx->poy_grid && time_samples == ctx->poy_T && ctx->n_poy > 0 &&
        std::equal(box, box + 6, ctx->poy_box))
        return PNX_OK;  // same nodes: only the weight changed
    ctx->poy_grid = grid;
    ctx->poy_T = time_samples;
    std::copy(box, box + 6, ctx->poy_box);
    // midpoint nodes per time sample (losses.cpp:196-205), time = linspace (sampling.cpp:10-20)
    const int64_t n2 = (int64_t)grid * grid, np = n2 * time_samples;
    const double hx = (box[1] - box[0]) / grid, hy = (box[3] - box[2]) / grid;
    const double ht = (box[5] - box[4]) / (double)(time_samples - 1);
    ctx->h_poy.assign((size_t)(3 * np), 0.0);
    for (int j = 0; j < time_samples; ++j) {
        const double tv = j + 1 == time_samples ? box[5] : box[4] + (double)j * ht;
        for (int64_t i = 0; i < grid; ++i)
            for (int64_t k = 0; k < grid; ++k) {
                const int64_t r = j * n2 + i * grid + k;
                ctx->h_poy[(size_t)r] = box[0] + ((double)i + 0.5) * hx;
                ctx->h_poy[(size_t)(np + r)] = box[2] + ((double)k + 0.5) * hy;
                ctx->h_poy[(size_t)(2 * np + r)] = tv;
            }
    }
    ctx->n_poy = np;
    ctx->rows_dirty = true;
    if (int r = dalloc(ctx, &ctx->d_poy_part, (size_t)ctx->head_grid * 2 * time_samples)) return r;
    if (int r = dalloc(ctx, &ctx->d_poy_g, (size_t)3 * time_samples)) return r;
    if (int r = dalloc(ctx, &ctx->d_pen, 1)) return r;
    CK(cudaMemset(ctx->d_pen, 0, 8));
    return PNX_OK;
}

int pnx_last_penalty(pnx_ctx* ctx, double* pen) {
    if (!ctx || !pen) return PNX_ERR_ARG;
    *pen = 0.0;
    if (ctx->n_poy == 0 || !ctx->d_pen) return PNX_OK;
    CK(cudaSetDevice(ctx->device));
    if (int r = wait_last_step(ctx)) return r;
    CK(cudaMemcpy(pen, ctx->d_pen, 8, cudaMemcpyDeviceToHost));
    return PNX_OK;
}

int pnx_set_ic(pnx_ctx* ctx, const double* coords, const double* targets, int64_t n) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    if (n < 0 || (n > 0 && (!coords || !targets))) return fail(ctx, PNX_ERR_ARG, "ic_loss: empty point set");
    ctx->h_ic.assign(coords, coords + n * ctx->in_dim);
    ctx->h_ic_t.resize((size_t)(n * ctx->F));
    for (int64_t i = 0; i < n * ctx->F; ++i) ctx->h_ic_t[(size_t)i] = (float)targets[i];
    ctx->n_ic = n;
    ctx->rows_dirty = true;
    return PNX_OK;
}

int pnx_set_bc(pnx_ctx* ctx, const double* a, const double* b, const double* targets, int64_t n) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    if (ctx->bc == PNX_BC_HARD) {
        if (n != 0) return fail(ctx, PNX_ERR_ARG, "pnx_set_bc: problem has hard (architectural) BC");
        return PNX_OK;
    }
    if (n <= 0 || !a) return fail(ctx, PNX_ERR_ARG, "bc_loss: empty point set");
    ctx->h_bca.assign(a, a + n * ctx->in_dim);
    ctx->n_bca = n;
    if (ctx->bc == PNX_BC_SOFT_PERIODIC) {
        if (!b) return fail(ctx, PNX_ERR_ARG, "bc_loss: boundary traces must pair up");
        ctx->h_bcb.assign(b, b + n * ctx->in_dim);
        ctx->n_bcb = n;
        ctx->h_bc_t.clear();
    } else {
        if (!targets) return fail(ctx, PNX_ERR_ARG, "loss: field/target count mismatch");
        ctx->h_bcb.clear();
        ctx->n_bcb = 0;
        ctx->h_bc_t.resize((size_t)(n * ctx->F));
        for (int64_t i = 0; i < n * ctx->F; ++i) ctx->h_bc_t[(size_t)i] = (float)targets[i];
    }
    ctx->rows_dirty = true;
    return PNX_OK;
}

int pnx_set_engine(pnx_ctx* ctx, int engine) {
    if (!ctx || engine < 0 || engine > 3) return PNX_ERR_ARG;
    ++ctx->state_ver;
    ctx->engine = engine;
    return PNX_OK;
}

int pnx_set_chunk_rows(pnx_ctx* ctx, int64_t rows) {
    if (!ctx || rows < 0) return PNX_ERR_ARG;
    ++ctx->state_ver;
    ctx->chunk_override = rows;
    ctx->rows_dirty = true;
    return PNX_OK;
}

int pnx_profile(pnx_ctx* ctx, int on) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    ctx->prof = on != 0;
    prof_collect(ctx);
    for (int i = 0; i < 8; ++i) {
        ctx->prof_ms[i] = 0.0;
        ctx->prof_n[i] = 0;
    }
    return PNX_OK;
}

int pnx_profile_read(pnx_ctx* ctx, double* ms, int64_t* counts, int n) {
    if (!ctx || !ms || !counts || n <= 0) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    prof_collect(ctx);
    for (int i = 0; i < n && i < 8; ++i) {
        ms[i] = ctx->prof_ms[i];
        counts[i] = ctx->prof_n[i];
    }
    return PNX_OK;
}

int pnx_last_launch_count(const pnx_ctx* ctx, int64_t* n) {
    if (!ctx || !n) return PNX_ERR_ARG;
    *n = ctx->launches;
    return PNX_OK;
}

int pnx_step_device(pnx_ctx* ctx, const float* d_params, const double lambdas[3], float* d_grad,
                    double* d_losses, void* stream) {
    if (!ctx || !d_params || !d_grad || !lambdas) return PNX_ERR_ARG;
    ++ctx->state_ver;
    CK(cudaSetDevice(ctx->device));
    return run_step(ctx, d_params, lambdas, d_grad, d_losses, reinterpret_cast<cudaStream_t>(stream));
}

// pnx_step's device step through the context's CUDA graph (PNX_STEP_GRAPH=0: eager)
static int step_graphed(pnx_ctx* ctx, const double lam[3]) {
    static const bool off = getenv("PNX_STEP_GRAPH") && getenv("PNX_STEP_GRAPH")[0] == '0';
    const bool graphable = !off && !ctx->reuse_fwd && !ctx->no_penalty && !ctx->capture_resid && !ctx->prof;
    auto same = [&](const double* a) { return a[0] == lam[0] && a[1] == lam[1] && a[2] == lam[2]; };
    if (graphable && ctx->g_exec && ctx->g_ver == ctx->state_ver && same(ctx->g_lam)) {
        CK(cudaGraphLaunch(ctx->g_exec, ctx->stream));
    } else if (graphable && ctx->g_warm_ver == ctx->state_ver && same(ctx->g_warm_lam)) {
        if (ctx->g_exec) cudaGraphExecDestroy(ctx->g_exec);
        ctx->g_exec = nullptr;
        ctx->g_ver = 0;
        cudaGraph_t gr = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        const int r = run_step(ctx, ctx->d_params, lam, ctx->d_grad, ctx->d_losses, ctx->stream);
        const cudaError_t e = cudaStreamEndCapture(ctx->stream, &gr);
        if (r != PNX_OK) {
            if (gr) cudaGraphDestroy(gr);
            return r;
        }
        CK(e);
        const cudaError_t ei = cudaGraphInstantiate(&ctx->g_exec, gr, 0);
        cudaGraphDestroy(gr);
        CK(ei);
        ctx->g_ver = ctx->state_ver;
        for (int k = 0; k < 3; ++k) ctx->g_lam[k] = lam[k];
        CK(cudaGraphLaunch(ctx->g_exec, ctx->stream));
    } else {
        if (int r = run_step(ctx, ctx->d_params, lam, ctx->d_grad, ctx->d_losses, ctx->stream)) return r;
        ctx->g_warm_ver = ctx->state_ver;
        for (int k = 0; k < 3; ++k) ctx->g_warm_lam[k] = lam[k];
        return PNX_OK;
    }
    // a replayed step is ordered for later host writes like an eager one
    CK(cudaEventRecord(ctx->ev_done, ctx->stream));
    ctx->ev_pending = true;
    return PNX_OK;
}

static int report_bad(pnx_ctx* ctx, const int* bad);

int pnx_check(pnx_ctx* ctx) {
    if (!ctx) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    if (int r = wait_last_step(ctx)) return r;
    int bad[5];
    CK(cudaDeviceSynchronize());  // Adam may run on another stream than the step
    CK(cudaMemcpy(bad, ctx->d_bad, sizeof(bad), cudaMemcpyDeviceToHost));
    if (int r = guard_check(ctx)) return r;
    return report_bad(ctx, bad);
}

// the sticky flags as read back: PNX_OK, or reset them and raise the first one
static int report_bad(pnx_ctx* ctx, const int* bad) {
    bool any = false;
    for (int k = 0; k < 5; ++k) any |= bad[k] != kBadNone;
    if (!any) return PNX_OK;
    CK(cudaMemset(ctx->d_bad, 0x7f, 8 * sizeof(int)));  // sticky until read
    for (int k = 0; k < ctx->Kres; ++k)
        if (bad[k] != kBadNone)
            return fail(ctx, PNX_ERR_NONFINITE,
                        "residual_loss: non-finite residual at point index " + std::to_string(bad[k]));
    if (bad[3] != kBadNone)
        return fail(ctx, PNX_ERR_NONFINITE,
                    "adam: non-finite gradient for parameter " + param_name(ctx, bad[3]) + " at step " +
                        (bad[4] != kBadNone ? std::to_string(bad[4]) : std::string("?")));
    return PNX_OK;
}

int pnx_step(pnx_ctx* ctx, const double* params, const double lambdas[3], double* grad_out,
             double losses_out[3]) {
    if (!ctx || !params || !lambdas) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    const int64_t P = ctx->P;
    if (ctx->stage_cap < 2 * P) {  // pinned: the copies are DMA at link speed, not staged by the driver
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        ctx->h_stage = nullptr;
        ctx->stage_cap = 0;
        CK(cudaMallocHost(&ctx->h_stage, (size_t)(2 * P) * 4 + 64));
        ctx->stage_cap = 2 * P;
    }
    // pinned layout: [params f32 P][grad f32 P][losses f64 x3][flags i32 x5] (2P floats keep 8 B alignment)
    float* p32 = ctx->h_stage;
    float* g32 = ctx->h_stage + P;
    double* hl = reinterpret_cast<double*>(ctx->h_stage + 2 * P);
    int* hbad = reinterpret_cast<int*>(hl + 3);
    if (int r = wait_last_step(ctx)) return r;  // an earlier step may still read the staging buffer
    host_par_for(P, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) p32[i] = (float)params[i];
    });
    CK(cudaMemcpyAsync(ctx->d_params, p32, (size_t)P * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (int r = step_graphed(ctx, lambdas)) return r;
    // gradient, losses and the sticky non-finite flags (written by this step's
    // kernels on ctx->stream) in one pinned read-back, one synchronisation
    CK(cudaMemcpyAsync(g32, ctx->d_grad, (size_t)P * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(hl, ctx->d_losses, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(hbad, ctx->d_bad, 5 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (int r = guard_check(ctx)) return r;
    if (int r = report_bad(ctx, hbad)) return r;
    const double losses[3] = {hl[0], hl[1], hl[2]};
    for (int t = 0; t < 3; ++t)
        if (!std::isfinite(losses[t])) return fail(ctx, PNX_ERR_NONFINITE, "non-finite loss in worker step");
    if (grad_out) {
        std::vector<int64_t> first_bad(8, INT64_MAX);  // first non-finite entry per thread range
        std::atomic<int> slot{0};
        host_par_for(P, [&](int64_t lo, int64_t hi) {
            const int me = slot.fetch_add(1);
            for (int64_t i = lo; i < hi; ++i) {
                if (!std::isfinite(g32[i])) {
                    first_bad[me] = i;
                    return;
                }
                grad_out[i] = (double)g32[i];
            }
        });
        const int64_t bad = *std::min_element(first_bad.begin(), first_bad.end());
        if (bad != INT64_MAX) return fail(ctx, PNX_ERR_NONFINITE, "non-finite gradient entry " + std::to_string(bad));
    }
    if (losses_out)
        for (int t = 0; t < 3; ++t) losses_out[t] = losses[t];
    return PNX_OK;
}

int pnx_step_terms(pnx_ctx* ctx, const double* params, double* grad_terms_out, double losses_out[3]) {
    if (!ctx || !params || !grad_terms_out) return PNX_ERR_ARG;
    ctx->no_penalty = true;
    int r = PNX_OK;
    static const bool no_reuse = getenv("PNX_TERMS_NO_REUSE") != nullptr;  // A/B and tests
    for (int k = 0; k < 3 && r == PNX_OK; ++k) {
        const double lam[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
        ctx->reuse_fwd = k > 0 && !no_reuse;
        r = pnx_step(ctx, params, lam, grad_terms_out + (int64_t)k * ctx->P, k == 0 ? losses_out : nullptr);
    }
    ctx->reuse_fwd = false;
    ctx->no_penalty = false;
    return r;
}

int pnx_step_terms_device(pnx_ctx* ctx, const float* d_params, float* d_grads, double* d_losses, void* stream) {
    if (!ctx || !d_params || !d_grads) return PNX_ERR_ARG;
    ++ctx->state_ver;
    CK(cudaSetDevice(ctx->device));
    ctx->no_penalty = true;
    int r = PNX_OK;
    static const bool no_reuse = getenv("PNX_TERMS_NO_REUSE") != nullptr;  // A/B and tests
    for (int k = 0; k < 3 && r == PNX_OK; ++k) {
        const double lam[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
        ctx->reuse_fwd = k > 0 && !no_reuse;
        r = run_step(ctx, d_params, lam, d_grads + (int64_t)k * ctx->P, k == 0 ? d_losses : nullptr,
                     reinterpret_cast<cudaStream_t>(stream));
    }
    ctx->reuse_fwd = false;
    ctx->no_penalty = false;
    return r;
}

int pnx_adam_step_device_state(pnx_ctx* ctx, float* d_params, const float* d_grad, float* d_m, float* d_v,
                               int64_t n, double* d_state, double lr0, double gamma, double beta1, double beta2,
                               double eps, double grad_scale, void* stream) {
    if (!ctx || !d_params || !d_grad || !d_m || !d_v || !d_state || n <= 0) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_any_nonfinite<<<grid, 256, 0, st>>>(d_grad, n, ctx->d_bad + 3);
    CKL();
    k_adam_state<<<grid, 256, 0, st>>>(d_params, d_grad, d_m, d_v, n, d_state, lr0, gamma, beta1, beta2,
                                       (float)eps, (float)grad_scale, ctx->d_bad + 3);
    CKL();
    k_adam_tick<<<1, 1, 0, st>>>(d_state, ctx->d_bad + 3);
    CKL();
    return PNX_OK;
}

int pnx_adam_step_device(pnx_ctx* ctx, float* d_params, const float* d_grad, float* d_m, float* d_v,
                         int64_t n, double lr, double beta1, double beta2, double eps, int64_t t,
                         double grad_scale, void* stream) {
    if (!ctx || !d_params || !d_grad || !d_m || !d_v || n <= 0 || t <= 0) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    const float bc1 = (float)(1.0 - std::pow(beta1, (double)t));
    const float bc2 = (float)(1.0 - std::pow(beta2, (double)t));
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    k_any_nonfinite<<<grid, 256, 0, st>>>(d_grad, n, ctx->d_bad + 3);
    CKL();
    k_adam<<<grid, 256, 0, st>>>(d_params, d_grad, d_m, d_v, n, (float)lr, (float)beta1, (float)beta2, (float)eps,
                                 bc1, bc2, (float)grad_scale, ctx->d_bad + 3, (int)t);
    CKL();
    return PNX_OK;
}

// Diagnostics (residual_components, losses.hpp:51-53): interior residuals of
// the last pnx_step, component-major [K][n_int] float64.
int pnx_capture_residuals(pnx_ctx* ctx, int on) {
    if (!ctx) return PNX_ERR_ARG;
    ++ctx->state_ver;
    ctx->capture_resid = on != 0;
    return PNX_OK;
}

int pnx_copy_points(pnx_ctx* ctx, double* out) {
    if (!ctx || !out) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    if (ctx->rows_dirty)
        if (int r = upload_rows(ctx)) return r;
    if (int r = wait_last_step(ctx)) return r;
    for (int a = 0; a < ctx->in_dim; ++a)
        CK(cudaMemcpy(out + a * ctx->n_int, ctx->d_coords + a * ctx->ld + ctx->int_off_prev, (size_t)ctx->n_int * 8,
                      cudaMemcpyDeviceToHost));
    return PNX_OK;
}

int pnx_copy_residuals(pnx_ctx* ctx, double* out) {
    if (!ctx || !out || !ctx->d_resid) return PNX_ERR_ARG;
    CK(cudaSetDevice(ctx->device));
    if (int r = wait_last_step(ctx)) return r;
    std::vector<float> r((size_t)(ctx->n_int * ctx->Kres));
    CK(cudaMemcpy(r.data(), ctx->d_resid, r.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    return PNX_OK;
}

}  // extern "C"
