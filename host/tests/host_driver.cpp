// host_driver.cpp -- exercises the C++ host API (pinnlab_b200) the way a
// reference user would: Model(spec, seed), build_collocation, and
// data_parallel_gradient / train on the GPU. Driven by tests/test_host_cpp.py.
//
//   host_driver cpu   job.txt outdir   -> params.bin rffB.bin interior.bin hash.txt
//   host_driver grad  job.txt outdir   -> grad.bin               (needs a GPU)
//   host_driver train job.txt outdir   -> metrics.bin final.bin  (needs a GPU)
//
// job.txt: one "key v1 v2 ..." per line (written by the test from a fixture).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <numbers>
#include <sstream>
#include <string>
#include <vector>

#include "pinnlab_b200.hpp"

using namespace pinnlab_b200;

namespace {

std::map<std::string, std::vector<std::string>> read_job(const std::string& path) {
    std::map<std::string, std::vector<std::string>> kv;
    std::ifstream is(path);
    std::string line;
    while (std::getline(is, line)) {
        std::istringstream ss(line);
        std::string key, v;
        ss >> key;
        while (ss >> v) kv[key].push_back(v);
    }
    return kv;
}

void write_f64(const std::string& path, const std::vector<double>& v) {
    std::ofstream os(path, std::ios::binary);
    os.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::cerr << "usage: host_driver cpu|grad|train job.txt outdir\n";
        return 2;
    }
    try {
        const std::string mode = argv[1], out = argv[3];
        auto kv = read_job(argv[2]);
        auto num = [&](const std::string& k, double d) { return kv.count(k) ? std::stod(kv[k][0]) : d; };
        ModelSpec s;
        s.in_dim = static_cast<std::size_t>(num("in_dim", 2));
        s.hidden_dim = static_cast<std::size_t>(num("hidden_dim", 64));
        s.depth = static_cast<std::size_t>(num("depth", 3));
        s.out_dim = static_cast<std::size_t>(num("out_dim", 1));
        const std::string act = kv["activation"].empty() ? "tanh" : kv["activation"][0];
        s.activation = act == "sine" ? Activation::sine : (act == "swish" ? Activation::swish : Activation::tanh);
        s.sine_w0 = num("sine_w0", 1.0);
        if (kv.count("periodic"))
            for (std::size_t a = 0; a < kv["periodic"].size() / 3; ++a)
                s.periodic_axes.push_back({kv["periodic"][3 * a] == "1", std::stod(kv["periodic"][3 * a + 1]),
                                           kv["periodic"][3 * a + 2] == "1"});
        if (kv.count("rff")) s.rff = RFFSpec{std::stoul(kv["rff"][0]), std::stod(kv["rff"][1]), std::stod(kv["rff"][2])};
        if (kv.count("rwf")) s.rwf = RWFSpec{std::stod(kv["rwf"][0]), std::stod(kv["rwf"][1])};
        Model model(s, static_cast<std::uint64_t>(num("seed", 0)));

        TrainingProblem prob;
        const std::string pde = kv["pde"][0];
        prob.residual.id = pde == "burgers" ? PdeId::burgers
                           : pde == "maxwell_te" ? PdeId::maxwell_te
                           : pde == "allen_cahn" ? PdeId::allen_cahn
                                                 : PdeId::advection;
        prob.residual.advection_c = num("advection_c", 1.0);
        prob.residual.epsilon = num("epsilon", 1.0);
        prob.residual.mu = num("mu", 1.0);
        for (std::size_t a = 0; a < kv["domain"].size() / 2; ++a)
            prob.domain.bounds.push_back({std::stod(kv["domain"][2 * a]), std::stod(kv["domain"][2 * a + 1])});
        const std::string init = kv["initial"][0];
        const std::size_t fields = prob.residual.field_count();
        prob.initial = [init, fields](std::span<const double> x) {
            std::vector<double> v(fields, 0.0);
            if (init == "sin_pi_x") v[0] = std::sin(std::numbers::pi * x[0]);
            else if (init == "sin_x") v[0] = std::sin(x[0]);
            else if (init == "gauss25") v[0] = std::exp(-25.0 * (x[0] * x[0] + (x.size() > 1 ? x[1] * x[1] : 0.0)));
            return v;
        };
        const std::string bc = kv["bc"][0];
        prob.bc = bc == "dirichlet_zero" ? TrainingProblem::Bc::dirichlet_zero
                  : bc == "soft_periodic" ? TrainingProblem::Bc::soft_periodic
                                          : TrainingProblem::Bc::hard;
        TrainConfig cfg;
        for (const auto& d : kv["dims"]) cfg.collocation.dims.push_back(std::stoul(d));
        if (kv.count("colloc_mode")) {
            const std::string cm = kv["colloc_mode"][0];
            cfg.collocation.mode = cm == "lhs" ? CollocationConfig::Mode::lhs
                                   : cm == "lhs_per_axis" ? CollocationConfig::Mode::lhs_per_axis
                                                          : CollocationConfig::Mode::uniform;
        }
        cfg.collocation.n = static_cast<std::size_t>(num("colloc_n", 0));
        cfg.collocation.resample_every = static_cast<int>(num("resample_every", 0));
        cfg.seed = static_cast<std::uint64_t>(num("colloc_seed", 0));
        cfg.collocation.n_ic = static_cast<std::size_t>(num("n_ic", 128));
        cfg.collocation.n_bc = static_cast<std::size_t>(num("n_bc", 64));
        const int workers = static_cast<int>(num("workers", 1));
        cfg.balancing.enabled = num("balancing", 0) != 0.0;
        cfg.balancing.alpha = num("alpha", 0.9);
        cfg.balancing.update_period = static_cast<int>(num("update_period", 100));
        cfg.causality.enabled = num("causality_segments", 0) > 0;
        cfg.causality.segments = static_cast<int>(num("causality_segments", 10));
        cfg.causality.epsilon = num("causality_epsilon", 1.0);
        cfg.poynting.weight = num("poynting_weight", 0.0);
        cfg.poynting.grid = static_cast<std::size_t>(num("poynting_grid", 32));
        cfg.poynting.time_samples = static_cast<std::size_t>(num("poynting_time_samples", 4));
        if (num("switch_epoch", -1) >= 0) {
            cfg.switch_policy.trigger = SwitchPolicy::Trigger::epoch_threshold;
            cfg.switch_policy.epoch_threshold = static_cast<long>(num("switch_epoch", 0));
        }
        cfg.lbfgs_max_iters = static_cast<long>(num("lbfgs_max_iters", 0));
        cfg.lbfgs.history = static_cast<int>(num("lbfgs_history", 50));

        if (mode == "cpu") {
            std::vector<double> p;
            for (const auto& t : model.trainable()) p.insert(p.end(), t.value.data.begin(), t.value.data.end());
            write_f64(out + "/params.bin", p);
            write_f64(out + "/rffB.bin", model.rff_matrix().data);
            CollocationData data = build_collocation(prob, cfg.collocation, cfg.seed);
            std::vector<double> pts;
            for (const auto& c : data.interior.coords) pts.insert(pts.end(), c.begin(), c.end());
            write_f64(out + "/interior.bin", pts);
            std::ofstream(out + "/hash.txt") << param_hash(model.trainable()) << "\n";
        } else if (mode == "grad") {
            std::vector<Tensor> g = data_parallel_gradient(model, prob, cfg, workers);
            std::vector<double> flat;
            for (const auto& t : g) flat.insert(flat.end(), t.data.begin(), t.data.end());
            write_f64(out + "/grad.bin", flat);
        } else if (mode == "train") {
            cfg.workers = workers;
            cfg.epochs = static_cast<long>(num("epochs", 10));
            cfg.adam.lr = num("lr", 1e-3);
            cfg.scheduler_gamma = num("gamma", 1.0);
            cfg.gpus = static_cast<int>(num("gpus", 0));
            std::vector<std::vector<std::uint64_t>> sync;  // per epoch: one hash per replica
            cfg.on_sync = [&sync](long, std::span<const std::uint64_t> h) { sync.emplace_back(h.begin(), h.end()); };
            TrainResult r = train(model, prob, cfg);
            if (r.aborted) throw TensorError(r.abort_reason);
            std::vector<double> m;
            for (const auto& rec : r.metrics) {
                for (double x : {rec.l_pde, rec.l_ic, rec.l_bc, rec.lambda_pde, rec.lambda_ic, rec.lambda_bc})
                    m.push_back(x);
            }
            write_f64(out + "/metrics.bin", m);
            std::vector<double> p;
            for (const auto& t : model.trainable()) p.insert(p.end(), t.value.data.begin(), t.value.data.end());
            write_f64(out + "/final.bin", p);
            std::ofstream os(out + "/hash.txt");  // one line per epoch, one hash per replica
            for (const auto& row : sync) {
                for (auto h : row) os << h << " ";
                os << "\n";
            }
        } else {
            throw TensorError("unknown mode " + mode);
        }
    } catch (const std::exception& e) {
        std::cerr << "host_driver: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
