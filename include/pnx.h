/*
 * pnx.h -- C ABI of the B200 PINN train-step hot path (libpnx.so).
 *
 * Drop-in boundary for the reference pinnlab core (/root/reference/proj/core).
 * The reference has no FFI; its seam is the per-worker step
 *   run_worker_epoch(const WorkerTask&) -> WorkerOutput   (trainer.cpp:189-262)
 * and the public one-step contract
 *   data_parallel_gradient(Model&, const TrainingProblem&,
 *                          const TrainConfig&, int W)     (trainer.hpp:118-119)
 * Each entry point below names the reference interface it replaces. Arrays
 * crossing the ABI are plain pointers + sizes; floating-point data at the host
 * boundary is float64 like the reference's Tensor (tensor.hpp:19-22); the
 * device computes in float32 (FP32 FMA / 3xTF32 tensor-core contractions).
 *
 * Errors: every call returns PNX_OK (0) or a negative code; pnx_last_error()
 * returns the message, which uses the reference's TensorError text where one
 * exists (e.g. "residual_loss: non-finite residual at point index 17",
 * losses.cpp:86-90; "data parallel: fewer interior points than workers",
 * trainer.cpp:147). No exceptions cross the ABI. A context is single-threaded
 * (like Graph, graph.hpp:69-70) and bound to one CUDA device.
 */
#ifndef PNX_H_
#define PNX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PNX_OK 0
#define PNX_ERR_ARG -1       /* invalid argument / shape (TensorError) */
#define PNX_ERR_CUDA -2      /* CUDA runtime failure / no device */
#define PNX_ERR_NONFINITE -3 /* non-finite residual, loss or gradient */
#define PNX_ERR_STATE -4     /* call order (e.g. step before set_points) */

typedef struct pnx_ctx pnx_ctx;

/* Activation (model.hpp:12). */
enum { PNX_ACT_TANH = 0, PNX_ACT_SINE = 1, PNX_ACT_SWISH = 2 };
/* PdeId (losses.hpp:14) + the ns_steady extension and the
 * TE-mode naming of Maxwell with fields (Ex, Ey, Hz) (BASELINE configs[3];
 * eps Ex_t = Hz_y, eps Ey_t = -Hz_x, mu Hz_t = Ex_y - Ey_x; extension: the
 * reference's maxwell_te is the (Ez, Hx, Hy) system, losses.cpp:57-72). */
enum { PNX_PDE_ADVECTION = 0, PNX_PDE_ALLEN_CAHN = 1, PNX_PDE_BURGERS = 2,
       PNX_PDE_MAXWELL_TE = 3, PNX_PDE_NS_STEADY = 4, PNX_PDE_MAXWELL_TE_EH = 5 };
/* TrainingProblem::Bc (trainer.hpp:23-27). */
enum { PNX_BC_HARD = 0, PNX_BC_SOFT_PERIODIC = 1, PNX_BC_DIRICHLET_ZERO = 2 };
/* Contraction engine for the hidden layers. */
/* TC3XF16: the tensor-core engine with 3xFP16 operands (hi/lo fp16 pairs scaled
 * by powers of two from recorded absmax bounds: the same 22-bit operand
 * precision as 3xTF32 at twice the tensor rate) where the kernels support it. */
enum { PNX_ENGINE_AUTO = 0, PNX_ENGINE_FFMA = 1, PNX_ENGINE_TC3XTF32 = 2, PNX_ENGINE_TC3XF16 = 3 };

/* ModelSpec (model.hpp:41-57). rff_B is the frozen RFF matrix Model::rff_matrix()
 * [embedded_width x rff_width] row-major (model.cpp:58-62); NULL when rff_width==0.
 * periodic/period/period_trainable have n_periodic_axes entries (0 or in_dim)
 * mirroring ModelSpec::periodic_axes (AxisPeriodic, model.hpp:32-36). */
typedef struct {
    int32_t in_dim, hidden_dim, depth, out_dim;
    int32_t activation;
    double sine_w0;
    int32_t n_periodic_axes;
    const int32_t* periodic;
    const double* period;
    const int32_t* period_trainable;
    int32_t rff_width;
    const double* rff_B;
    int32_t rwf; /* 1: layers are (V, s) pairs, W = V * exp(s) (model.cpp:117-126) */
} pnx_model_desc;

/* ResidualSpec (losses.hpp:22-30) + TrainingProblem::bc. */
typedef struct {
    int32_t pde;
    double advection_c, epsilon, mu, reynolds;
    int32_t bc;
} pnx_problem_desc;

/* Create a worker context on CUDA device `device`. Replaces the per-worker
 * Graph + Model::bind of run_worker_epoch (trainer.cpp:205-207). */
int pnx_create(const pnx_model_desc* model, const pnx_problem_desc* problem, int device,
               pnx_ctx** out);
void pnx_destroy(pnx_ctx* ctx);
const char* pnx_last_error(const pnx_ctx* ctx);
/* Message of the last failure of pnx_create (no context exists then). */
const char* pnx_create_error(void);

/* Model::trainable_count() (model.cpp:104-108); the flat layout is
 * flatten_params (trainer.cpp:290-298): trainable() order, row-major. */
int pnx_param_count(const pnx_ctx* ctx, int64_t* n);

/* Interior collocation shard (WorkerTask::interior, trainer.cpp:192), axis-major
 * float64 [n_axes][n] (Points::coords, losses.hpp:39-43; space first, time last).
 * The caller's buffer is copied before the call returns (the copy waits for the
 * last enqueued step that reads the points); pinned buffers are copied by DMA. */
int pnx_set_points(pnx_ctx* ctx, const double* coords, int64_t n, int32_t n_axes);
/* Interior points generated on the device instead (sampling.cpp:10-103): design
 * mode 0 = uniform tensor grid of linspace axes, last axis fastest
 * (sample_uniform; bit-exact), 1 = joint Latin hypercube of n_total points
 * (sample_lhs), 2 = per-axis jittered LHS (sample_lhs_per_axis); bounds =
 * {lo0, hi0, lo1, hi1, ...} per axis (Domain::bounds), dims per axis (modes 0/2).
 * This worker's shard is rows [row_lo, row_hi) of the global design (no host
 * copy, no upload). Randomness is counter-based on (seed, axis, index), not the
 * reference's mt19937_64 stream; same designs. Resampling (trainer.cpp:421-434)
 * with seed + epoch regenerates in place. */
int pnx_sample_points(pnx_ctx* ctx, int32_t mode, const double* bounds, const int64_t* dims, int64_t n_total,
                      uint64_t seed, int64_t row_lo, int64_t row_hi);
/* Replicated IC set + per-field targets [out_dim][n] (CollocationData::ic_points /
 * ic_targets, trainer.hpp:140-146; losses.cpp:113-119). */
int pnx_set_ic(pnx_ctx* ctx, const double* coords, const double* targets, int64_t n);
/* Replicated BC set (trainer.cpp:98-125). soft_periodic: a and b paired traces
 * (losses.cpp:121-135), targets NULL. dirichlet_zero: a = stacked traces,
 * b NULL, targets [out_dim][n] (losses.cpp:137-144). */
int pnx_set_bc(pnx_ctx* ctx, const double* a, const double* b, const double* targets, int64_t n);

/* One worker step: losses + gradient of total = lam_pde L_pde + lam_ic L_ic
 * (+ lam_bc L_bc) (trainer.cpp:234-253) for the current shard. params/grad_out
 * are flat float64 in trainable() order; losses_out = {pde, ic, bc}
 * (TermLosses, trainer.cpp:179-181). Host buffers; synchronous. */
int pnx_step(pnx_ctx* ctx, const double* params, const double lambdas[3], double* grad_out,
             double losses_out[3]);

/* Adam with the step count and epoch kept on the device (d_state[0] = steps
 * taken, d_state[1] = epoch; both advanced by the call): lr = lr0 * gamma^epoch
 * (ExponentialLr::at, optim.cpp:71-73) and the bias corrections are formed on
 * the device, so pnx_step_device + all-reduce + this call can be captured once
 * in a CUDA graph and replayed every epoch. */
int pnx_adam_step_device_state(pnx_ctx* ctx, float* d_params, const float* d_grad, float* d_m, float* d_v,
                               int64_t n, double* d_state, double lr0, double gamma, double beta1, double beta2,
                               double eps, double grad_scale, void* stream);

/* Per-term gradients of l_pde, l_ic, l_bc alone (run_worker_epoch with
 * want_term_grads, trainer.cpp:256-260): three reverse passes with unit
 * weights and the Poynting penalty excluded; grad_terms_out holds 3 x
 * param_count doubles (pde | ic | bc). Used on loss-balancing epochs
 * (trainer.cpp:462-506). */
int pnx_step_terms(pnx_ctx* ctx, const double* params, double* grad_terms_out, double losses_out[3]);
int pnx_step_terms_device(pnx_ctx* ctx, const float* d_params, float* d_grads, double* d_losses, void* stream);

/* Temporal causality (CausalityConfig, trainer.hpp:51-55): this worker's
 * interior points are bucketed by their last coordinate over [t_lo, t_hi]
 * into `segments` (split_time_segments, trainer.cpp:156-177); pnx_step then
 * minimises l_pde = (1/M) sum_i omega_i L_i with omega from the segment losses
 * (causality_weights / weighted_pde_loss, losses.cpp:163-185; omega is a
 * constant of the step). segments <= 0 disables (the default). */
int pnx_set_causality(pnx_ctx* ctx, int32_t segments, double epsilon, double t_lo, double t_hi);

/* Poynting energy penalty (PoyntingConfig, trainer.hpp:57-61; poynting_penalty,
 * losses.cpp:187-223): maxwell_te only; weight 0 disables (the default).
 * box = {x_lo, x_hi, y_lo, y_hi, t_lo, t_hi}; grid^2 midpoint nodes at each of
 * time_samples = linspace(t_lo, t_hi) instants are evaluated on every worker
 * (replicated like the IC set) and weight * penalty joins the total loss. */
int pnx_set_poynting(pnx_ctx* ctx, double weight, int32_t grid, int32_t time_samples, const double box[6]);
/* Penalty value (unweighted) of the last step; synchronizes the ctx stream. */
int pnx_last_penalty(pnx_ctx* ctx, double* pen);

/* Device-resident variant (no host copies): d_params/d_grad are float32 device
 * pointers of param_count entries, d_losses (may be NULL) receives 3 doubles;
 * work is enqueued on `stream` (a cudaStream_t, 0 = legacy default). The
 * non-finite check is deferred: call pnx_check(ctx) after synchronizing. */
int pnx_step_device(pnx_ctx* ctx, const float* d_params, const double lambdas[3], float* d_grad,
                    double* d_losses, void* stream);
/* Synchronizes the device and reports the sticky non-finite flags (residual
 * point index, Adam gradient entry and step); with the environment variable
 * PNX_GUARD=1 set at load time it also verifies the 512-byte guard tail of
 * every context buffer ("guard: write past the end ..."), a debug stand-in for
 * a memory checker. */
int pnx_check(pnx_ctx* ctx);

/* Device Adam (optim.cpp:7-41) with ExponentialLr lr = base*gamma^epoch
 * (optim.cpp:71-73) and an optional 1/W gradient scale (average_grads,
 * trainer.cpp:278-280), fused in one kernel: p -= lr*mhat/(sqrt(vhat)+eps).
 * t is the step count AFTER increment (first step t=1). */
int pnx_adam_step_device(pnx_ctx* ctx, float* d_params, const float* d_grad, float* d_m, float* d_v,
                         int64_t n, double lr, double beta1, double beta2, double eps, int64_t t,
                         double grad_scale, void* stream);

/* Engine selection and chunking (rows per pass through the layer stack). */
int pnx_set_engine(pnx_ctx* ctx, int engine);
int pnx_set_chunk_rows(pnx_ctx* ctx, int64_t rows);
/* Number of kernels the last step launched (for bench evidence). */
int pnx_last_launch_count(const pnx_ctx* ctx, int64_t* n);

/* Kernel-class timing with CUDA events recorded on the launching stream around
 * every launch of a class (0 input, 1 forward GEMM, 2 head, 3 reverse GEMM,
 * 4 weight-gradient GEMM, 5 finalize, 6 the single-kernel step of a narrow
 * network). pnx_profile(ctx, 1) resets and enables;
 * pnx_profile_read synchronizes and returns accumulated ms and launch counts. */
int pnx_profile(pnx_ctx* ctx, int on);
int pnx_profile_read(pnx_ctx* ctx, double* ms, int64_t* counts, int n);

/* Diagnostics mirroring residual_components (losses.hpp:51-53): when capture
 * is on, pnx_step records the interior residuals, copied out component-major
 * [K][n_interior] as float64. */
int pnx_capture_residuals(pnx_ctx* ctx, int on);
int pnx_copy_residuals(pnx_ctx* ctx, double* out);
/* The interior points the next step uses, axis-major float64 [n_axes][n]
 * (e.g. a device design from pnx_sample_points). */
int pnx_copy_points(pnx_ctx* ctx, double* out);

/* ---- data-parallel group over the local GPUs (libpnx links NCCL) -------------
 * Replaces train()'s per-epoch worker threads (trainer.cpp:441-460), the
 * rank-ordered average_grads (trainer.cpp:264-281) and the replica update
 * (trainer.cpp:626-638): rank r is a worker context on devices[r] (ranks of one
 * device are its local replicas), one persistent host thread per device, and
 * per step ONE ncclAllReduce (sum, float32, in place) of the packed
 * [grad (P) | l_pde, l_ic, l_bc, pen] over one communicator per device
 * (ncclCommInitAll), then the device Adam applies the 1/R average to every
 * device's parameter replica. Interior points are sharded contiguously, the
 * last rank taking the remainder (shard_interior, trainer.cpp:143-154); IC/BC
 * sets are replicated on every rank (trainer.cpp:225-232). */
typedef struct pnx_dp pnx_dp;
int pnx_device_count(int* n);
int pnx_dp_create(const pnx_model_desc* model, const pnx_problem_desc* problem, const int* devices, int n_ranks,
                  pnx_dp** out);
void pnx_dp_destroy(pnx_dp* dp);
const char* pnx_dp_last_error(const pnx_dp* dp);
int pnx_dp_size(const pnx_dp* dp, int* n_ranks, int* n_devices);
/* The worker context of one rank (engine, chunking, causality, Poynting). */
int pnx_dp_rank_ctx(pnx_dp* dp, int rank, pnx_ctx** ctx);
/* Global interior set, axis-major float64 [n_axes][n]; sharded over the ranks. */
int pnx_dp_set_points(pnx_dp* dp, const double* coords, int64_t n, int32_t n_axes);
/* The global interior as a device design (pnx_sample_points), each rank generating its shard. */
int pnx_dp_sample_points(pnx_dp* dp, int32_t mode, const double* bounds, const int64_t* dims, int64_t n_total,
                         uint64_t seed);
int pnx_dp_set_ic(pnx_dp* dp, const double* coords, const double* targets, int64_t n);
int pnx_dp_set_bc(pnx_dp* dp, const double* a, const double* b, const double* targets, int64_t n);
/* Parameters of every replica (flat trainable() order); resets Adam's moments and step. */
int pnx_dp_set_params(pnx_dp* dp, const double* params);
/* Host copy of the replica that `rank` trains (for param_hash / on_sync, trainer.cpp:540-544). */
int pnx_dp_get_params(pnx_dp* dp, int rank, double* params);
/* AdamConfig + ExponentialLr (optim.hpp:21-50); defaults lr 1e-3, gamma 1, 0.9, 0.999, 1e-8. */
int pnx_dp_set_optimizer(pnx_dp* dp, double lr, double gamma, double beta1, double beta2, double eps);
/* Capture each device's step (worker steps + sums + all-reduce + Adam) in a CUDA
 * graph and replay it while the loss weights stay the same. */
int pnx_dp_set_graph(pnx_dp* dp, int on);
/* One synchronized step with loss weights lambdas: update != 0 applies Adam.
 * losses_out (4: pde, ic, bc, penalty; means over ranks) and grad_out (P, the
 * averaged gradient) are optional host buffers; with both NULL the call only
 * enqueues (no host synchronization). Non-finite residuals / gradients raise
 * PNX_ERR_NONFINITE with the reference's text at the next synchronizing call. */
int pnx_dp_step(pnx_dp* dp, const double lambdas[3], int update, double* losses_out, double* grad_out);
/* Per-term gradients averaged over ranks (balancing epochs, trainer.cpp:256-260,
 * 462-506): grad_terms_out holds 3 x P (pde | ic | bc), losses_out 3. */
int pnx_dp_step_terms(pnx_dp* dp, double* grad_terms_out, double* losses_out);
/* Adam step of every replica with a host gradient (the balanced lambda-weighted sum). */
int pnx_dp_apply_gradient(pnx_dp* dp, const double* grad);
/* Synchronize and raise any non-finite flag of any rank. */
int pnx_dp_check(pnx_dp* dp);

#ifdef __cplusplus
}
#endif

#endif /* PNX_H_ */
