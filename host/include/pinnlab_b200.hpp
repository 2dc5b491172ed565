// pinnlab_b200.hpp -- C++ host API mirroring the reference pinnlab core
// (/root/reference/proj/core/include/pinnlab) for the train-step path, with the
// per-worker step executed by libpnx (include/pnx.h) on B200s.
//
// Same names, argument meaning and error behaviour as the reference:
//   ModelSpec / AxisPeriodic / RFFSpec / RWFSpec      model.hpp:14-57
//   Model (init draws, trainable() order)             model.cpp:52-102
//   ResidualSpec / PdeId                              losses.hpp:14-30
//   Domain, linspace, sample_uniform                  sampling.hpp:13-36
//   TrainingProblem, CollocationConfig, TrainConfig   trainer.hpp:17-86
//   build_collocation (uniform / LHS modes)           trainer.cpp:47-128
//   data_parallel_gradient                            trainer.hpp:118-119
//   train (Adam phase: balancing, causality, Poynting) trainer.cpp:332-555
//   param_hash                                        trainer.cpp:22-35
// Errors are thrown as pinnlab_b200::TensorError with the reference's text.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace pinnlab_b200 {

class TensorError : public std::runtime_error {
public:
    explicit TensorError(const std::string& what) : std::runtime_error(what) {}
};

enum class Activation { tanh, sine, swish };

struct RFFSpec {
    std::size_t width = 64;
    double sigma = 10.0;
    double mean = 0.0;
};
struct RWFSpec {
    double mean = 1.0;
    double stddev = 0.1;
};
struct AxisPeriodic {
    bool periodic = false;
    double period = 0.0;
    bool trainable = false;
};

struct ModelSpec {
    std::size_t in_dim = 2;
    std::size_t hidden_dim = 64;
    std::size_t depth = 3;
    std::size_t out_dim = 1;
    Activation activation = Activation::tanh;
    double sine_w0 = 1.0;
    std::vector<AxisPeriodic> periodic_axes;
    std::optional<RFFSpec> rff;
    std::optional<RWFSpec> rwf;

    std::size_t embedded_width() const;
    std::size_t first_layer_width() const;
    void validate() const;
};

// Row-major float64 tensor of rank 0..2 (tensor.hpp:19-109, reduced to storage).
struct Tensor {
    std::vector<std::size_t> shape;
    std::vector<double> data;
    std::size_t size() const { return data.size(); }
};

struct NamedTensor {
    std::string name;
    Tensor value;
};

class Model {
public:
    Model(ModelSpec spec, std::uint64_t seed);
    const ModelSpec& spec() const { return spec_; }
    std::vector<NamedTensor>& trainable() { return params_; }
    const std::vector<NamedTensor>& trainable() const { return params_; }
    const Tensor& rff_matrix() const { return rff_B_; }
    std::size_t trainable_count() const;

private:
    ModelSpec spec_;
    std::vector<NamedTensor> params_;
    Tensor rff_B_;
};

// + extensions: ns_steady and maxwell_te_eh, the TE system with
// fields (Ex, Ey, Hz) (the reference's maxwell_te is the (Ez, Hx, Hy) system)
enum class PdeId { advection, allen_cahn, burgers, maxwell_te, ns_steady, maxwell_te_eh };

struct ResidualSpec {
    PdeId id = PdeId::advection;
    double advection_c = 1.0;
    double epsilon = 1.0;
    double mu = 1.0;
    double reynolds = 100.0;  // ns_steady extension

    std::size_t field_count() const {
        return (id == PdeId::maxwell_te || id == PdeId::maxwell_te_eh || id == PdeId::ns_steady) ? 3 : 1;
    }
    std::size_t coord_count() const { return (id == PdeId::maxwell_te || id == PdeId::maxwell_te_eh) ? 3 : 2; }
};

struct Points {
    std::vector<std::vector<double>> coords;  // one column per axis
    std::size_t count() const { return coords.empty() ? 0 : coords[0].size(); }
};

struct Domain {
    std::vector<std::array<double, 2>> bounds;
    std::size_t dim() const { return bounds.size(); }
};

std::vector<double> linspace(double lo, double hi, std::size_t n);
Points sample_uniform(const Domain& dom, std::span<const std::size_t> dims);
// Latin hypercube designs with the reference's mt19937_64 stream (sampling.cpp:55-103)
Points sample_lhs(const Domain& dom, std::size_t n, std::uint64_t seed);
Points sample_lhs_per_axis(const Domain& dom, std::span<const std::size_t> dims, std::uint64_t seed);

struct TrainingProblem {
    ResidualSpec residual;
    Domain domain;
    std::function<std::vector<double>(std::span<const double>)> initial;
    enum class Bc { hard, soft_periodic, dirichlet_zero };
    Bc bc = Bc::hard;
};

struct CollocationConfig {  // trainer.hpp:31-43
    enum class Mode { uniform, lhs, lhs_per_axis };
    Mode mode = Mode::uniform;
    std::vector<std::size_t> dims;  // per-axis counts (uniform / per-axis LHS)
    std::size_t n = 0;              // point count for joint LHS
    std::size_t n_ic = 128;
    std::size_t n_bc = 64;
    int resample_every = 0;         // LHS modes: fresh interior every k epochs (seed + epoch)
};

struct CollocationData {
    Points interior;
    Points ic_points;
    std::vector<std::vector<double>> ic_targets;  // one column per field
    Points bc_a, bc_b;
    std::vector<std::vector<double>> bc_targets;
};
CollocationData build_collocation(const TrainingProblem& prob, const CollocationConfig& cc, std::uint64_t seed);

struct AdamConfig {
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
};

struct BalancingConfig {  // trainer.hpp:45-49
    bool enabled = true;
    double alpha = 0.9;
    int update_period = 100;
};
struct CausalityConfig {  // trainer.hpp:51-55
    bool enabled = false;
    int segments = 10;
    double epsilon = 1.0;
};
struct PoyntingConfig {  // trainer.hpp:57-61
    double weight = 0.0;
    std::size_t grid = 32;
    std::size_t time_samples = 4;
};

struct SwitchPolicy {  // optim.hpp:54-62
    enum class Trigger { none, epoch_threshold, loss_plateau };
    Trigger trigger = Trigger::none;
    long epoch_threshold = 0;
    int plateau_window = 0;
    double plateau_rel_improvement = 0.0;
    bool should_switch(long epoch, std::span<const double> loss_history) const;
};
struct LbfgsConfig {  // lbfgs.hpp:10-17
    int history = 50;
    double c1 = 1e-4;
    double c2 = 0.9;
    int max_line_search = 25;
    double grad_tol = 1e-10;
    double curvature_floor = 1e-10;
};

struct TrainConfig {
    long epochs = 1000;
    std::uint64_t seed = 0;
    int workers = 1;
    AdamConfig adam;
    double scheduler_gamma = 1.0;
    CollocationConfig collocation;
    BalancingConfig balancing;
    CausalityConfig causality;
    PoyntingConfig poynting;
    SwitchPolicy switch_policy;
    long lbfgs_max_iters = 0;  // quasi-Newton refinement budget after the switch
    LbfgsConfig lbfgs;
    std::array<double, 3> lambdas{1.0, 1.0, 1.0};  // initial loss weights
    int device = 0;  // first CUDA device
    int gpus = 0;    // GPUs used (0: every visible device from `device` on); worker w runs on
                     // device + w % gpus -- workers sharing a GPU are summed on it, GPUs join in
                     // one NCCL all-reduce per step (pnx_dp, include/pnx.h)
    std::function<void(long epoch, std::span<const std::uint64_t>)> on_sync;
};

struct MetricsRecord {
    long epoch = 0;
    double l_pde = 0.0, l_ic = 0.0, l_bc = 0.0;
    double lambda_pde = 1.0, lambda_ic = 1.0, lambda_bc = 1.0;
    double lr = 0.0;
};
struct TrainResult {
    std::vector<MetricsRecord> metrics;
    long epochs_run = 0;
    bool switched_to_lbfgs = false;
    bool aborted = false;
    std::string abort_reason;
};

// One data-parallel gradient evaluation (shard, per-worker step, rank-ordered
// average), returned aligned with Model::trainable().
std::vector<Tensor> data_parallel_gradient(Model& model, const TrainingProblem& prob, const TrainConfig& cfg,
                                           int workers);

// Adam training loop (loss balancing, causality weights, Poynting penalty as
// configured): the W worker replicas live on the GPUs (pnx_dp: device steps,
// one NCCL all-reduce and the device Adam per epoch, CUDA-graph replays);
// on_sync receives one param_hash per replica, read from that replica's device.
TrainResult train(Model& model, const TrainingProblem& prob, const TrainConfig& cfg);

std::uint64_t param_hash(const std::vector<NamedTensor>& params);

// One Adam update in place (optim.cpp:7-41): t is the 1-based step count, lr
// already scheduled (optim.cpp:71-73).
void adam_update(double* p, double* m, double* v, const double* g, std::size_t n, double lr,
                 const AdamConfig& a, std::int64_t t);

}  // namespace pinnlab_b200

// C ABI of the host Adam, for callers that drive pnx_step with host buffers
// from another language (bench.py's end-to-end leg). Returns 0.
extern "C" int pinnlab_adam_step(double* p, double* m, double* v, const double* g, std::int64_t n,
                                 double lr, double beta1, double beta2, double eps, std::int64_t t);
