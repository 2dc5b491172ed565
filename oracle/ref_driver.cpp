// oracle/_ref driver: runs the UNMODIFIED reference pinnlab core (compiled from
// /root/reference/proj/core/src by oracle/Makefile against the Eigen-API shim)
// on a JSON job and dumps little-endian float64 results. TEST INFRASTRUCTURE
// ONLY -- used to generate tests/golden fixtures, to pin oracle/pinn_oracle.py,
// and as the CPU baseline (`bench.py --impl reference`). Never linked into the
// product library.
//
// Modes
//   step      one data-parallel gradient evaluation. The gradient comes from the
//             reference's own `data_parallel_gradient` (trainer.hpp:118,
//             trainer.cpp:649-678); per-shard losses are recomputed with the same
//             public calls run_worker_epoch makes (trainer.cpp:200-262:
//             residual_loss, ic_loss, bc_*; losses.cpp:77-144). Per-point residual
//             components come from residual_components (losses.cpp:26-75).
//   train     the reference `train()` loop (trainer.cpp:332-624); dumps the metrics
//             stream (trainer.cpp:517-538), final params and on_sync hashes.
//
// Usage: pinnlab_ref_driver <job.json>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <numbers>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "pinnlab/checkpoint.hpp"
#include "pinnlab/losses.hpp"
#include "pinnlab/model.hpp"
#include "pinnlab/trainer.hpp"

using namespace pinnlab;
using nlohmann::json;

namespace {

void write_f64(const std::string& path, const std::vector<double>& v) {
    std::ofstream os(path, std::ios::binary);
    os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

std::vector<double> read_f64(const std::string& path) {
    std::ifstream is(path, std::ios::binary | std::ios::ate);
    if (!is) throw std::runtime_error("cannot open " + path);
    std::streamsize n = is.tellg();
    is.seekg(0);
    std::vector<double> v(static_cast<std::size_t>(n / 8));
    is.read(reinterpret_cast<char*>(v.data()), n);
    return v;
}

std::vector<double> flat_params(const std::vector<NamedTensor>& ps) {
    std::vector<double> v;
    for (const auto& p : ps) v.insert(v.end(), p.value.data(), p.value.data() + p.value.size());
    return v;
}

std::vector<double> flat_tensors(const std::vector<Tensor>& ts) {
    std::vector<double> v;
    for (const auto& t : ts) v.insert(v.end(), t.data(), t.data() + t.size());
    return v;
}

std::vector<double> flat_points(const Points& p) {
    // axis-major: all of axis 0, then axis 1, ...
    std::vector<double> v;
    for (const auto& c : p.coords) v.insert(v.end(), c.data(), c.data() + c.size());
    return v;
}

std::function<std::vector<double>(std::span<const double>)> initial_fn(const std::string& name,
                                                                       std::size_t fields) {
    if (name == "sin_pi_x")
        return [](std::span<const double> x) { return std::vector<double>{std::sin(std::numbers::pi * x[0])}; };
    if (name == "sin_x")
        return [](std::span<const double> x) { return std::vector<double>{std::sin(x[0])}; };
    if (name == "gauss25")
        return [](std::span<const double> x) {
            double r2 = x[0] * x[0] + (x.size() > 1 ? x[1] * x[1] : 0.0);
            return std::vector<double>{std::exp(-25.0 * r2), 0.0, 0.0};
        };
    if (name == "zero")
        return [fields](std::span<const double>) { return std::vector<double>(fields, 0.0); };
    throw std::runtime_error("unknown initial function " + name);
}

TrainingProblem make_problem(const json& j) {
    TrainingProblem p;
    const json& pde = j.at("pde");
    p.residual.id = pde_from_name(pde.at("id").get<std::string>());
    p.residual.advection_c = pde.value("advection_c", 1.0);
    p.residual.epsilon = pde.value("epsilon", 1.0);
    p.residual.mu = pde.value("mu", 1.0);
    for (const auto& b : j.at("domain")) p.domain.bounds.push_back({b[0].get<double>(), b[1].get<double>()});
    p.initial = initial_fn(j.value("initial", std::string("zero")), p.residual.field_count());
    std::string bc = j.value("bc", std::string("hard"));
    if (bc == "hard") p.bc = TrainingProblem::Bc::hard;
    else if (bc == "soft_periodic") p.bc = TrainingProblem::Bc::soft_periodic;
    else if (bc == "dirichlet_zero") p.bc = TrainingProblem::Bc::dirichlet_zero;
    else throw std::runtime_error("unknown bc " + bc);
    return p;
}

CollocationConfig make_colloc(const json& j) {
    CollocationConfig c;
    std::string mode = j.value("mode", std::string("uniform"));
    if (mode == "uniform") c.mode = CollocationConfig::Mode::uniform;
    else if (mode == "lhs") c.mode = CollocationConfig::Mode::lhs;
    else if (mode == "lhs_per_axis") c.mode = CollocationConfig::Mode::lhs_per_axis;
    if (j.contains("dims")) c.dims = j.at("dims").get<std::vector<std::size_t>>();
    c.n = j.value("n", std::size_t{0});
    c.n_ic = j.value("n_ic", std::size_t{128});
    c.n_bc = j.value("n_bc", std::size_t{64});
    c.resample_every = j.value("resample_every", 0);
    return c;
}

void set_params(Model& m, const std::vector<double>& flat) {
    std::size_t at = 0;
    for (auto& p : m.trainable())
        for (std::size_t k = 0; k < p.value.size(); ++k) p.value[k] = flat.at(at++);
    if (at != flat.size()) throw std::runtime_error("params_in length mismatch");
}

// The non-causal body of run_worker_epoch (trainer.cpp:200-262) through public
// calls, returning the term losses; gradients come from data_parallel_gradient.
std::array<double, 3> worker_losses(const Model& model, const TrainingProblem& prob,
                                    const Points& shard, const CollocationData& shared) {
    Graph g;
    Model::Binding binding = model.bind(g);
    FieldFn f = model_fields(model, binding);
    double pde = g.value(residual_loss(g, f, shard, prob.residual)).item();
    double ic = g.value(ic_loss(g, f, shared.ic_points, shared.ic_targets)).item();
    double bc = 0.0;
    if (prob.bc == TrainingProblem::Bc::soft_periodic)
        bc = g.value(bc_periodic_loss(g, f, shared.bc_a, shared.bc_b)).item();
    else if (prob.bc == TrainingProblem::Bc::dirichlet_zero)
        bc = g.value(bc_dirichlet_loss(g, f, shared.bc_a, shared.bc_targets)).item();
    return {pde, ic, bc};
}

// poynting_penalty (losses.cpp:187-223) value as run_worker_epoch adds it
// (trainer.cpp:240-247): time samples = linspace over the last axis.
double worker_penalty(const Model& model, const TrainingProblem& prob, const TrainConfig& cfg) {
    Graph g;
    Model::Binding binding = model.bind(g);
    FieldFn f = model_fields(model, binding);
    auto ts = linspace(prob.domain.bounds.back()[0], prob.domain.bounds.back()[1], cfg.poynting.time_samples);
    Value pen = poynting_penalty(g, f, ts, prob.domain.bounds[0], prob.domain.bounds[1], cfg.poynting.grid,
                                 prob.residual.epsilon, prob.residual.mu);
    return g.value(pen).item();
}

std::vector<double> residual_values(const Model& model, const TrainingProblem& prob,
                                    const Points& pts) {
    Graph g;
    Model::Binding binding = model.bind(g);
    FieldFn f = model_fields(model, binding);
    std::vector<Value> leaves;
    for (const Tensor& c : pts.coords) leaves.push_back(g.leaf(c));
    std::vector<Value> rs = residual_components(g, f, leaves, prob.residual);
    std::vector<double> out;  // component-major
    for (Value r : rs) {
        const Tensor& t = g.value(r);
        out.insert(out.end(), t.data(), t.data() + t.size());
    }
    return out;
}

std::vector<double> model_outputs(const Model& model, const Points& pts) {
    Graph g;
    std::vector<Value> leaves;
    for (const Tensor& c : pts.coords) leaves.push_back(g.leaf(c));
    const Tensor& t = g.value(model.forward(g, leaves));
    return std::vector<double>(t.data(), t.data() + t.size());  // [N, out] row-major
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: " << argv[0] << " job.json\n";
        return 2;
    }
    try {
        std::ifstream js(argv[1]);
        json job = json::parse(js);
        const std::string out = job.at("out").get<std::string>();
        const std::string mode = job.value("mode", std::string("step"));

        ModelSpec spec = model_spec_from_json(job.at("model").dump());
        std::uint64_t seed = job.value("seed", std::uint64_t{0});
        Model model(spec, seed);
        if (job.contains("params_in")) set_params(model, read_f64(job.at("params_in").get<std::string>()));
        TrainingProblem prob = make_problem(job);

        TrainConfig cfg;
        cfg.seed = job.value("colloc_seed", std::uint64_t{0});
        cfg.collocation = make_colloc(job.at("collocation"));
        cfg.workers = job.value("workers", 1);
        if (job.contains("poynting")) {  // PoyntingConfig (trainer.hpp:57-61)
            const json& pj = job.at("poynting");
            cfg.poynting.weight = pj.value("weight", 0.0);
            cfg.poynting.grid = pj.value("grid", std::size_t{32});
            cfg.poynting.time_samples = pj.value("time_samples", std::size_t{4});
        }
        if (job.contains("causality")) {  // CausalityConfig (trainer.hpp:51-55)
            const json& cj = job.at("causality");
            cfg.causality.enabled = cj.value("enabled", true);
            cfg.causality.segments = cj.value("segments", 10);
            cfg.causality.epsilon = cj.value("epsilon", 1.0);
        }

        json meta;
        json pnames = json::array();
        for (const auto& p : model.trainable()) pnames.push_back({{"name", p.name}, {"shape", p.value.shape()}});
        meta["params"] = pnames;
        meta["rff_shape"] = model.rff_matrix().shape();
        write_f64(out + "/params.bin", flat_params(model.trainable()));
        if (spec.rff)
            write_f64(out + "/rff_B.bin", std::vector<double>(model.rff_matrix().data(),
                                                              model.rff_matrix().data() + model.rff_matrix().size()));

        CollocationData data = build_collocation(prob, cfg.collocation, cfg.seed);
        write_f64(out + "/interior.bin", flat_points(data.interior));
        write_f64(out + "/ic_points.bin", flat_points(data.ic_points));
        write_f64(out + "/ic_targets.bin", flat_tensors(data.ic_targets));
        write_f64(out + "/bc_a.bin", flat_points(data.bc_a));
        write_f64(out + "/bc_b.bin", flat_points(data.bc_b));
        write_f64(out + "/bc_targets.bin", flat_tensors(data.bc_targets));
        meta["n_interior"] = data.interior.count();
        meta["n_ic"] = data.ic_points.count();
        meta["n_bc_a"] = data.bc_a.count();
        meta["n_bc_b"] = data.bc_b.count();

        if (mode == "step") {
            const int W = cfg.workers;
            // Same contiguous sharding as shard_interior (trainer.cpp:143-154).
            std::size_t n = data.interior.count(), base = n / static_cast<std::size_t>(W);
            json wl = json::array();
            for (int w = 0; w < W; ++w) {
                std::size_t from = static_cast<std::size_t>(w) * base;
                std::size_t to = (w + 1 == W) ? n : from + base;
                Points shard;
                for (const Tensor& c : data.interior.coords) {
                    Tensor col({to - from, 1});
                    for (std::size_t i = from; i < to; ++i) col[i - from] = c[i];
                    shard.coords.push_back(std::move(col));
                }
                auto l = worker_losses(model, prob, shard, data);
                wl.push_back({{"pde", l[0]}, {"ic", l[1]}, {"bc", l[2]}, {"from", from}, {"to", to}});
            }
            meta["worker_losses"] = wl;
            if (cfg.poynting.weight > 0.0 && prob.residual.id == PdeId::maxwell_te)
                meta["penalty"] = worker_penalty(model, prob, cfg);
            auto t0 = std::chrono::steady_clock::now();
            std::vector<Tensor> grads = data_parallel_gradient(model, prob, cfg, W);
            meta["grad_seconds"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            write_f64(out + "/grad.bin", flat_tensors(grads));
            if (job.value("dump_residuals", true)) {
                write_f64(out + "/residuals.bin", residual_values(model, prob, data.interior));
                write_f64(out + "/outputs.bin", model_outputs(model, data.interior));
            }
        } else if (mode == "train") {
            const json& t = job.at("train");
            cfg.epochs = t.value("epochs", 10L);
            cfg.adam.lr = t.value("lr", 1e-3);
            cfg.scheduler_gamma = t.value("gamma", 1.0);
            cfg.balancing.enabled = t.value("balancing", false);
            cfg.balancing.update_period = t.value("update_period", 100);
            cfg.balancing.alpha = t.value("alpha", 0.9);
            cfg.poynting.weight = t.value("poynting_weight", cfg.poynting.weight);
            if (t.contains("switch")) {  // SwitchPolicy (optim.hpp:54-62) + L-BFGS phase (trainer.cpp:549-617)
                const json& sw = t.at("switch");
                const std::string trig = sw.value("trigger", std::string("none"));
                cfg.switch_policy.trigger = trig == "epoch" ? SwitchPolicy::Trigger::epoch_threshold
                                            : trig == "plateau" ? SwitchPolicy::Trigger::loss_plateau
                                                                : SwitchPolicy::Trigger::none;
                cfg.switch_policy.epoch_threshold = sw.value("epoch_threshold", 0L);
                cfg.switch_policy.plateau_window = sw.value("plateau_window", 0);
                cfg.switch_policy.plateau_rel_improvement = sw.value("plateau_rel_improvement", 0.0);
                cfg.lbfgs_max_iters = t.value("lbfgs_max_iters", 0L);
                if (t.contains("lbfgs")) {
                    const json& lj = t.at("lbfgs");
                    cfg.lbfgs.history = lj.value("history", cfg.lbfgs.history);
                    cfg.lbfgs.c1 = lj.value("c1", cfg.lbfgs.c1);
                    cfg.lbfgs.c2 = lj.value("c2", cfg.lbfgs.c2);
                    cfg.lbfgs.max_line_search = lj.value("max_line_search", cfg.lbfgs.max_line_search);
                    cfg.lbfgs.grad_tol = lj.value("grad_tol", cfg.lbfgs.grad_tol);
                    cfg.lbfgs.curvature_floor = lj.value("curvature_floor", cfg.lbfgs.curvature_floor);
                }
            }
            cfg.save_every = t.value("save_every", 0L);
            cfg.run_dir = t.value("run_dir", std::string());        // train() writes final.ckpt there
            cfg.resume_from = t.value("resume_from", std::string());  // PLABCK01 checkpoint to resume
            json hashes = json::array();
            cfg.on_sync = [&hashes](long epoch, std::span<const std::uint64_t> hs) {
                json row = json::array();
                for (auto h : hs) row.push_back(std::to_string(h));
                hashes.push_back({{"epoch", epoch}, {"hashes", row}});
            };
            TrainResult r = train(model, prob, cfg);
            json ms = json::array();
            for (const auto& m : r.metrics)
                ms.push_back({m.epoch, m.l_pde, m.l_ic, m.l_bc, m.lambda_pde, m.lambda_ic, m.lambda_bc, m.lr, m.wall_s});
            meta["metrics"] = ms;
            meta["aborted"] = r.aborted;
            meta["switched_to_lbfgs"] = r.switched_to_lbfgs;
            meta["epochs_run"] = r.epochs_run;
            meta["abort_reason"] = r.abort_reason;
            meta["hashes"] = hashes;
            write_f64(out + "/final_params.bin", flat_params(model.trainable()));
        } else if (mode == "ckpt_info") {
            // Checkpoint::load (checkpoint.cpp:142-170) of job["ckpt"]: header + payload
            Checkpoint ck = Checkpoint::load(job.at("ckpt").get<std::string>());
            json tl = json::array();
            std::vector<double> all;
            for (const auto& t : ck.tensors) {
                tl.push_back({{"name", t.name}, {"shape", t.value.shape()}});
                all.insert(all.end(), t.value.data(), t.value.data() + t.value.size());
            }
            meta["ckpt_tensors"] = tl;
            meta["ckpt_scalars"] = ck.scalars;
            meta["ckpt_seed"] = ck.seed;
            meta["ckpt_model"] = json::parse(model_spec_to_json(ck.spec));
            write_f64(out + "/ckpt_data.bin", all);
            Model m2 = ck.restore_model();  // throws on a missing / misshapen trainable tensor
            write_f64(out + "/restored_params.bin", flat_params(m2.trainable()));
        } else {
            throw std::runtime_error("unknown mode " + mode);
        }
        std::ofstream(out + "/meta.json") << meta.dump(1) << "\n";
    } catch (const std::exception& e) {
        std::cerr << "pinnlab_ref_driver: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
