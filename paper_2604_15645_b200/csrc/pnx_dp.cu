// pnx_dp.cu -- data-parallel group over the local GPUs (C ABI, include/pnx.h).
//
// Replaces the reference's in-process data parallelism: train() spawns one
// std::thread per worker per epoch and joins them (trainer.cpp:441-460), then
// average_grads sums the worker gradients in rank order and scales by 1/W
// (trainer.cpp:264-281), and one Adam update is copied to every replica
// (trainer.cpp:626-638). Here:
//   * rank r is a worker context (pnx_ctx) on devices[r]; the ranks of one
//     device are its local replicas (several ranks may share a GPU);
//   * one persistent host thread per device enqueues that device's work;
//   * per step and device: every local rank's device step writes its packed
//     [grad (P) | l_pde, l_ic, l_bc, pen] (float32) and the packs are summed on
//     the device in rank order; ONE ncclAllReduce (sum, float32, in place) over
//     the devices' communicators (ncclCommInitAll) joins them; the device Adam
//     applies the 1/R average to that device's parameter replica -- the
//     replicas stay bit-identical because every device applies the same update
//     to the same bits (checked by pnx_dp_get_params + param_hash, on_sync);
//   * optionally the whole per-device step (steps + sums + all-reduce + Adam) is
//     captured once in a CUDA graph and replayed while the loss weights stay.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pnx.h"
#include "launch.h"

namespace {

__global__ void k_dp_pack_losses(const double* __restrict__ l, const double* __restrict__ pen,
                                 float* __restrict__ dst) {
    if (threadIdx.x < 3) dst[threadIdx.x] = (float)l[threadIdx.x];
    if (threadIdx.x == 3) dst[3] = pen ? (float)*pen : 0.0f;
}
__global__ void k_dp_add(float* __restrict__ a, const float* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] += b[i];
}
__global__ void k_dp_zero_state(double* s) {
    s[0] = 0.0;
    s[1] = 0.0;
}

struct Dev {
    int device = 0;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    std::vector<int> ranks;            // local ranks, rank order
    float *d_params = nullptr, *d_m = nullptr, *d_v = nullptr;
    float* d_pack = nullptr;           // [P + 4] sum of the local ranks, then the all-reduce
    std::vector<float*> d_extra;       // packs of local ranks 1..
    float* d_terms = nullptr;          // [3P + 4] per-term gradients (balancing epochs)
    std::vector<float*> d_terms_extra;
    double* d_losses = nullptr;        // 3 per local rank
    double* d_state = nullptr;         // Adam (steps, epoch)
    cudaGraphExec_t gexec = nullptr;
    double glam[3] = {0, 0, 0};
};

}  // namespace

struct pnx_dp {
    int R = 0, D = 0, in_dim = 0;
    int64_t P = 0;
    std::vector<pnx_ctx*> ctx;  // per rank
    std::vector<int> rank_dev;  // rank -> index into dev
    std::vector<Dev> dev;
    double lr = 1e-3, gamma = 1.0, b1 = 0.9, b2 = 0.999, eps = 1e-8;
    bool graph = false;
    bool warm = false;  // a step ran eagerly since the last input change (uploads happen outside capture)
    std::string err;
    // one host thread per device
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    std::function<int(int)> job;
    uint64_t gen = 0;
    int pending = 0;
    bool quit = false;
    std::vector<int> rc;
    std::vector<std::string> msg;
};

namespace {

int dp_fail(pnx_dp* dp, int code, const std::string& m) {
    if (dp) dp->err = m;
    return code;
}

#define DPCK(call)                                                                                 \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            msg = std::string(#call ": ") + cudaGetErrorString(e_);                                \
            return PNX_ERR_CUDA;                                                                   \
        }                                                                                          \
    } while (0)
#define DPNC(call)                                                                                 \
    do {                                                                                           \
        ncclResult_t n_ = (call);                                                                  \
        if (n_ != ncclSuccess) {                                                                   \
            msg = std::string(#call ": ") + ncclGetErrorString(n_);                                \
            return PNX_ERR_CUDA;                                                                   \
        }                                                                                          \
    } while (0)

void dp_thread(pnx_dp* dp, int d) {
    cudaSetDevice(dp->dev[(size_t)d].device);
    uint64_t seen = 0;
    for (;;) {
        std::function<int(int)> job;
        {
            std::unique_lock<std::mutex> lk(dp->mu);
            dp->cv.wait(lk, [&] { return dp->quit || dp->gen != seen; });
            if (dp->quit) return;
            seen = dp->gen;
            job = dp->job;
        }
        const int r = job(d);
        {
            std::lock_guard<std::mutex> lk(dp->mu);
            dp->rc[(size_t)d] = r;
            if (--dp->pending == 0) dp->cv_done.notify_all();
        }
    }
}

// Run job(d) on every device's thread; first failure (device order) wins.
int run_all(pnx_dp* dp, std::function<int(int, std::string&)> f) {
    for (auto& m : dp->msg) m.clear();
    {
        std::unique_lock<std::mutex> lk(dp->mu);
        dp->job = [dp, f](int d) { return f(d, dp->msg[(size_t)d]); };
        dp->pending = dp->D;
        ++dp->gen;
        dp->cv.notify_all();
        dp->cv_done.wait(lk, [&] { return dp->pending == 0; });
    }
    for (int d = 0; d < dp->D; ++d)
        if (dp->rc[(size_t)d] != PNX_OK) return dp_fail(dp, dp->rc[(size_t)d], dp->msg[(size_t)d]);
    return PNX_OK;
}

int ctx_call(pnx_ctx* c, int r, std::string& msg) {
    if (r != PNX_OK) msg = pnx_last_error(c);
    return r;
}

// One device's share of a step: local ranks' steps summed in rank order into
// d_pack, the all-reduce, and (update) the Adam step on the device replica.
int enqueue_step(pnx_dp* dp, Dev& v, const double lam[3], bool update, std::string& msg) {
    const int64_t n = dp->P + 4;
    for (size_t i = 0; i < v.ranks.size(); ++i) {
        pnx_ctx* c = dp->ctx[(size_t)v.ranks[i]];
        float* pk = i == 0 ? v.d_pack : v.d_extra[i - 1];
        if (int r = ctx_call(c, pnx_step_device(c, v.d_params, lam, pk, v.d_losses + 3 * i, v.stream), msg)) return r;
        k_dp_pack_losses<<<1, 32, 0, v.stream>>>(v.d_losses + 3 * i, pnx::ctx_penalty_ptr(c), pk + dp->P);
        DPCK(cudaGetLastError());
        if (i > 0) {
            k_dp_add<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, v.stream>>>(v.d_pack, pk, n);
            DPCK(cudaGetLastError());
        }
    }
    nvtxRangePushA("pnx_dp ncclAllReduce [grad | losses]");
    const ncclResult_t nr = ncclAllReduce(v.d_pack, v.d_pack, (size_t)n, ncclFloat, ncclSum, v.comm, v.stream);
    nvtxRangePop();
    DPNC(nr);
    if (update) {
        pnx_ctx* c = dp->ctx[(size_t)v.ranks[0]];
        if (int r = ctx_call(c, pnx_adam_step_device_state(c, v.d_params, v.d_pack, v.d_m, v.d_v, dp->P, v.d_state,
                                                          dp->lr, dp->gamma, dp->b1, dp->b2, dp->eps,
                                                          1.0 / (double)dp->R, v.stream),
                             msg))
            return r;
    }
    return PNX_OK;
}

// host copies of the averaged losses (and gradient) from device 0's pack
int read_pack(pnx_dp* dp, const float* d_pack, int64_t len, double* losses_out, double* grad_out) {
    Dev& v = dp->dev[0];
    std::string msg;
    DPCK(cudaSetDevice(v.device));
    DPCK(cudaStreamSynchronize(v.stream));
    std::vector<float> h((size_t)(grad_out ? len + 4 : 4));
    if (grad_out) {
        DPCK(cudaMemcpy(h.data(), d_pack, (size_t)(len + 4) * 4, cudaMemcpyDeviceToHost));
    } else {
        DPCK(cudaMemcpy(h.data(), d_pack + len, 16, cudaMemcpyDeviceToHost));
    }
    const double inv = 1.0 / (double)dp->R;
    const float* l = grad_out ? h.data() + len : h.data();
    if (losses_out)
        for (int k = 0; k < 4; ++k) losses_out[k] = (double)l[k] * inv;
    if (grad_out)
        for (int64_t i = 0; i < len; ++i) grad_out[i] = (double)h[(size_t)i] * inv;
    return PNX_OK;
}

void invalidate_graphs(pnx_dp* dp) {
    dp->warm = false;
    for (auto& v : dp->dev)
        if (v.gexec) {
            cudaSetDevice(v.device);
            cudaGraphExecDestroy(v.gexec);
            v.gexec = nullptr;
        }
}

template <class T>
int dev_alloc(T** p, size_t n, std::string& msg) {
    DPCK(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)));
    DPCK(cudaMemset(*p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return PNX_OK;
}

}  // namespace

extern "C" {

int pnx_device_count(int* n) {
    if (!n) return PNX_ERR_ARG;
    *n = 0;
    return cudaGetDeviceCount(n) == cudaSuccess ? PNX_OK : PNX_ERR_CUDA;
}

int pnx_dp_create(const pnx_model_desc* m, const pnx_problem_desc* p, const int* devices, int n_ranks,
                  pnx_dp** out) {
    if (!m || !p || !devices || n_ranks <= 0 || !out) return PNX_ERR_ARG;
    *out = nullptr;
    auto* dp = new pnx_dp();
    dp->R = n_ranks;
    dp->in_dim = m->in_dim;
    std::string msg;
    // devices in first-use order; ranks of one device are its local replicas
    for (int r = 0; r < n_ranks; ++r) {
        int d = -1;
        for (int k = 0; k < (int)dp->dev.size(); ++k)
            if (dp->dev[(size_t)k].device == devices[r]) d = k;
        if (d < 0) {
            d = (int)dp->dev.size();
            dp->dev.emplace_back();
            dp->dev.back().device = devices[r];
        }
        dp->rank_dev.push_back(d);
        dp->dev[(size_t)d].ranks.push_back(r);
        pnx_ctx* c = nullptr;
        if (int rc = pnx_create(m, p, devices[r], &c)) {
            dp->ctx.push_back(nullptr);
            pnx_dp_destroy(dp);
            return rc;
        }
        dp->ctx.push_back(c);
    }
    dp->D = (int)dp->dev.size();
    pnx_param_count(dp->ctx[0], &dp->P);
    std::vector<int> devlist;
    for (auto& v : dp->dev) devlist.push_back(v.device);
    std::vector<ncclComm_t> comms((size_t)dp->D);
    int rc = PNX_OK;
    if (ncclCommInitAll(comms.data(), dp->D, devlist.data()) != ncclSuccess) {
        rc = PNX_ERR_CUDA;
        msg = "pnx_dp_create: ncclCommInitAll failed";
    }
    for (int d = 0; d < dp->D && rc == PNX_OK; ++d) {
        Dev& v = dp->dev[(size_t)d];
        v.comm = comms[(size_t)d];
        if (cudaSetDevice(v.device) != cudaSuccess ||
            cudaStreamCreateWithFlags(&v.stream, cudaStreamNonBlocking) != cudaSuccess) {
            rc = PNX_ERR_CUDA;
            msg = "pnx_dp_create: stream";
            break;
        }
        const size_t P = (size_t)dp->P, L = v.ranks.size();
        if ((rc = dev_alloc(&v.d_params, P, msg)) || (rc = dev_alloc(&v.d_m, P, msg)) ||
            (rc = dev_alloc(&v.d_v, P, msg)) || (rc = dev_alloc(&v.d_pack, P + 4, msg)) ||
            (rc = dev_alloc(&v.d_losses, 3 * L, msg)) || (rc = dev_alloc(&v.d_state, 2, msg)))
            break;
        v.d_extra.assign(L - 1, nullptr);
        for (auto& e : v.d_extra)
            if ((rc = dev_alloc(&e, P + 4, msg))) break;
    }
    if (rc != PNX_OK) {
        pnx::set_create_error(msg);
        pnx_dp_destroy(dp);
        return rc;
    }
    dp->rc.assign((size_t)dp->D, PNX_OK);
    dp->msg.assign((size_t)dp->D, std::string());
    try {  // no exception may cross the C ABI
        for (int d = 0; d < dp->D; ++d) dp->th.emplace_back(dp_thread, dp, d);
    } catch (...) {
        pnx::set_create_error("pnx_dp_create: cannot start the per-device host threads");
        pnx_dp_destroy(dp);  // joins the threads that did start
        return PNX_ERR_CUDA;
    }
    *out = dp;
    return PNX_OK;
}

void pnx_dp_destroy(pnx_dp* dp) {
    if (!dp) return;
    {
        std::lock_guard<std::mutex> lk(dp->mu);
        dp->quit = true;
        dp->cv.notify_all();
    }
    for (auto& t : dp->th) t.join();
    for (auto& v : dp->dev) {
        cudaSetDevice(v.device);
        if (v.stream) cudaStreamSynchronize(v.stream);
        if (v.gexec) cudaGraphExecDestroy(v.gexec);
        if (v.comm) ncclCommDestroy(v.comm);
        cudaFree(v.d_params);
        cudaFree(v.d_m);
        cudaFree(v.d_v);
        cudaFree(v.d_pack);
        for (float* e : v.d_extra) cudaFree(e);
        cudaFree(v.d_terms);
        for (float* e : v.d_terms_extra) cudaFree(e);
        cudaFree(v.d_losses);
        cudaFree(v.d_state);
        if (v.stream) cudaStreamDestroy(v.stream);
    }
    for (pnx_ctx* c : dp->ctx)
        if (c) pnx_destroy(c);
    delete dp;
}

const char* pnx_dp_last_error(const pnx_dp* dp) { return dp ? dp->err.c_str() : "null group"; }

int pnx_dp_size(const pnx_dp* dp, int* n_ranks, int* n_devices) {
    if (!dp) return PNX_ERR_ARG;
    if (n_ranks) *n_ranks = dp->R;
    if (n_devices) *n_devices = dp->D;
    return PNX_OK;
}

int pnx_dp_rank_ctx(pnx_dp* dp, int rank, pnx_ctx** ctx) {
    if (!dp || !ctx || rank < 0 || rank >= dp->R) return PNX_ERR_ARG;
    invalidate_graphs(dp);  // the caller may reconfigure the rank (causality, Poynting, engine)
    *ctx = dp->ctx[(size_t)rank];
    return PNX_OK;
}

int pnx_dp_set_points(pnx_dp* dp, const double* coords, int64_t n, int32_t n_axes) {
    if (!dp || !coords || n_axes <= 0) return PNX_ERR_ARG;
    const int64_t base = n / dp->R;
    if (base == 0) return dp_fail(dp, PNX_ERR_ARG, "data parallel: fewer interior points than workers");
    invalidate_graphs(dp);
    std::vector<double> shard;
    for (int r = 0; r < dp->R; ++r) {  // shard_interior: contiguous, last takes the remainder
        const int64_t lo = r * base, hi = r + 1 == dp->R ? n : lo + base;
        shard.resize((size_t)((hi - lo) * n_axes));
        for (int a = 0; a < n_axes; ++a)
            std::memcpy(shard.data() + (size_t)(a * (hi - lo)), coords + a * n + lo, (size_t)(hi - lo) * 8);
        pnx_ctx* c = dp->ctx[(size_t)r];
        if (int rc = pnx_set_points(c, shard.data(), hi - lo, n_axes)) return dp_fail(dp, rc, pnx_last_error(c));
    }
    return PNX_OK;
}

int pnx_dp_sample_points(pnx_dp* dp, int32_t mode, const double* bounds, const int64_t* dims, int64_t n_total,
                         uint64_t seed) {
    if (!dp || !bounds) return PNX_ERR_ARG;
    int64_t total = n_total;
    if (mode != 1) {  // grid designs: the product of the axis counts
        if (!dims) return PNX_ERR_ARG;
        total = 1;
        for (int a = 0; a < dp->in_dim; ++a) total *= dims[a] > 0 ? dims[a] : 0;
    }
    const int64_t base = total / dp->R;
    if (base == 0) return dp_fail(dp, PNX_ERR_ARG, "data parallel: fewer interior points than workers");
    invalidate_graphs(dp);
    for (int r = 0; r < dp->R; ++r) {  // shard_interior: contiguous, last takes the remainder
        const int64_t lo = r * base, hi = r + 1 == dp->R ? total : lo + base;
        pnx_ctx* c = dp->ctx[(size_t)r];
        if (int rc = pnx_sample_points(c, mode, bounds, dims, n_total, seed, lo, hi))
            return dp_fail(dp, rc, pnx_last_error(c));
    }
    return PNX_OK;
}

int pnx_dp_set_ic(pnx_dp* dp, const double* coords, const double* targets, int64_t n) {
    if (!dp) return PNX_ERR_ARG;
    invalidate_graphs(dp);
    for (pnx_ctx* c : dp->ctx)
        if (int rc = pnx_set_ic(c, coords, targets, n)) return dp_fail(dp, rc, pnx_last_error(c));
    return PNX_OK;
}

int pnx_dp_set_bc(pnx_dp* dp, const double* a, const double* b, const double* targets, int64_t n) {
    if (!dp) return PNX_ERR_ARG;
    invalidate_graphs(dp);
    for (pnx_ctx* c : dp->ctx)
        if (int rc = pnx_set_bc(c, a, b, targets, n)) return dp_fail(dp, rc, pnx_last_error(c));
    return PNX_OK;
}

int pnx_dp_set_params(pnx_dp* dp, const double* params) {
    if (!dp || !params) return PNX_ERR_ARG;
    std::vector<float> h((size_t)dp->P);
    for (int64_t i = 0; i < dp->P; ++i) h[(size_t)i] = (float)params[i];
    return run_all(dp, [&](int d, std::string& msg) -> int {
        Dev& v = dp->dev[(size_t)d];
        DPCK(cudaMemcpyAsync(v.d_params, h.data(), h.size() * 4, cudaMemcpyHostToDevice, v.stream));
        DPCK(cudaMemsetAsync(v.d_m, 0, h.size() * 4, v.stream));
        DPCK(cudaMemsetAsync(v.d_v, 0, h.size() * 4, v.stream));
        k_dp_zero_state<<<1, 1, 0, v.stream>>>(v.d_state);
        DPCK(cudaGetLastError());
        DPCK(cudaStreamSynchronize(v.stream));
        return PNX_OK;
    });
}

int pnx_dp_get_params(pnx_dp* dp, int rank, double* params) {
    if (!dp || !params || rank < 0 || rank >= dp->R) return PNX_ERR_ARG;
    Dev& v = dp->dev[(size_t)dp->rank_dev[(size_t)rank]];
    std::string msg;
    std::vector<float> h((size_t)dp->P);
    auto body = [&]() -> int {
        DPCK(cudaSetDevice(v.device));
        DPCK(cudaStreamSynchronize(v.stream));
        DPCK(cudaMemcpy(h.data(), v.d_params, h.size() * 4, cudaMemcpyDeviceToHost));
        return PNX_OK;
    };
    if (int rc = body()) return dp_fail(dp, rc, msg);
    for (int64_t i = 0; i < dp->P; ++i) params[i] = (double)h[(size_t)i];
    return PNX_OK;
}

int pnx_dp_set_optimizer(pnx_dp* dp, double lr, double gamma, double beta1, double beta2, double eps) {
    if (!dp || !(lr > 0.0)) return PNX_ERR_ARG;
    invalidate_graphs(dp);
    dp->lr = lr;
    dp->gamma = gamma;
    dp->b1 = beta1;
    dp->b2 = beta2;
    dp->eps = eps;
    return PNX_OK;
}

int pnx_dp_set_graph(pnx_dp* dp, int on) {
    if (!dp) return PNX_ERR_ARG;
    invalidate_graphs(dp);
    dp->graph = on != 0;
    return PNX_OK;
}

int pnx_dp_step(pnx_dp* dp, const double lambdas[3], int update, double* losses_out, double* grad_out) {
    if (!dp || !lambdas) return PNX_ERR_ARG;
    const bool use_graph = dp->graph && update && dp->warm;
    int rc = run_all(dp, [&](int d, std::string& msg) -> int {
        Dev& v = dp->dev[(size_t)d];
        if (!use_graph) return enqueue_step(dp, v, lambdas, update != 0, msg);
        if (v.gexec && !std::equal(lambdas, lambdas + 3, v.glam)) {
            DPCK(cudaGraphExecDestroy(v.gexec));
            v.gexec = nullptr;
        }
        if (!v.gexec) {  // capture this device's step once (steps + sums + all-reduce + Adam)
            cudaGraph_t g = nullptr;
            DPCK(cudaStreamBeginCapture(v.stream, cudaStreamCaptureModeThreadLocal));
            const int r = enqueue_step(dp, v, lambdas, true, msg);
            const cudaError_t e = cudaStreamEndCapture(v.stream, &g);
            if (r != PNX_OK) return r;
            DPCK(e);
            DPCK(cudaGraphInstantiate(&v.gexec, g, 0));
            cudaGraphDestroy(g);
            std::copy(lambdas, lambdas + 3, v.glam);
        }
        DPCK(cudaGraphLaunch(v.gexec, v.stream));
        return PNX_OK;
    });
    if (rc != PNX_OK) return rc;
    dp->warm = true;
    if (losses_out || grad_out) {
        if ((rc = read_pack(dp, dp->dev[0].d_pack, dp->P, losses_out, grad_out))) return rc;
        return pnx_dp_check(dp);
    }
    return PNX_OK;
}

int pnx_dp_step_terms(pnx_dp* dp, double* grad_terms_out, double* losses_out) {
    if (!dp || !grad_terms_out) return PNX_ERR_ARG;
    const int64_t P = dp->P, n = 3 * P + 4;
    int rc = run_all(dp, [&](int d, std::string& msg) -> int {
        Dev& v = dp->dev[(size_t)d];
        if (!v.d_terms) {
            if (int r = dev_alloc(&v.d_terms, (size_t)n, msg)) return r;
            v.d_terms_extra.assign(v.ranks.size() - 1, nullptr);
            for (auto& e : v.d_terms_extra)
                if (int r = dev_alloc(&e, (size_t)n, msg)) return r;
        }
        for (size_t i = 0; i < v.ranks.size(); ++i) {
            pnx_ctx* c = dp->ctx[(size_t)v.ranks[i]];
            float* pk = i == 0 ? v.d_terms : v.d_terms_extra[i - 1];
            if (int r = ctx_call(c, pnx_step_terms_device(c, v.d_params, pk, v.d_losses + 3 * i, v.stream), msg))
                return r;
            k_dp_pack_losses<<<1, 32, 0, v.stream>>>(v.d_losses + 3 * i, nullptr, pk + 3 * P);
            DPCK(cudaGetLastError());
            if (i > 0) {
                k_dp_add<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, v.stream>>>(v.d_terms, pk, n);
                DPCK(cudaGetLastError());
            }
        }
        DPNC(ncclAllReduce(v.d_terms, v.d_terms, (size_t)n, ncclFloat, ncclSum, v.comm, v.stream));
        return PNX_OK;
    });
    if (rc != PNX_OK) return rc;
    double l4[4];
    if ((rc = read_pack(dp, dp->dev[0].d_terms, 3 * P, l4, grad_terms_out))) return rc;
    if (losses_out) std::copy(l4, l4 + 3, losses_out);
    return pnx_dp_check(dp);
}

int pnx_dp_apply_gradient(pnx_dp* dp, const double* grad) {
    if (!dp || !grad) return PNX_ERR_ARG;
    std::vector<float> h((size_t)dp->P);
    for (int64_t i = 0; i < dp->P; ++i) h[(size_t)i] = (float)grad[i];
    return run_all(dp, [&](int d, std::string& msg) -> int {
        Dev& v = dp->dev[(size_t)d];
        DPCK(cudaMemcpyAsync(v.d_pack, h.data(), h.size() * 4, cudaMemcpyHostToDevice, v.stream));
        pnx_ctx* c = dp->ctx[(size_t)v.ranks[0]];
        if (int r = ctx_call(c, pnx_adam_step_device_state(c, v.d_params, v.d_pack, v.d_m, v.d_v, dp->P, v.d_state,
                                                          dp->lr, dp->gamma, dp->b1, dp->b2, dp->eps, 1.0, v.stream),
                             msg))
            return r;
        DPCK(cudaStreamSynchronize(v.stream));  // h is released on return
        return PNX_OK;
    });
}

int pnx_dp_check(pnx_dp* dp) {
    if (!dp) return PNX_ERR_ARG;
    return run_all(dp, [&](int d, std::string& msg) -> int {
        Dev& v = dp->dev[(size_t)d];
        DPCK(cudaStreamSynchronize(v.stream));
        for (int r : v.ranks)
            if (int rc = ctx_call(dp->ctx[(size_t)r], pnx_check(dp->ctx[(size_t)r]), msg)) return rc;
        return PNX_OK;
    });
}

}  // extern "C"
