// pinnlab_b200.cpp -- C++ host mirror of the reference pinnlab API over libpnx.
// See host/include/pinnlab_b200.hpp for the reference file:line map.
#include "pinnlab_b200.hpp"

#include <deque>
#include <algorithm>
#include <numeric>

#include <cmath>
#include <memory>
#include <numbers>
#include <random>
#include <thread>

#include "../../include/pnx.h"

namespace pinnlab_b200 {

// ---------------------------------------------------------------------------
// ModelSpec / Model (model.cpp:14-108)
// ---------------------------------------------------------------------------

std::size_t ModelSpec::embedded_width() const {
    if (periodic_axes.empty()) return in_dim;
    std::size_t w = 0;
    for (const auto& ax : periodic_axes) w += ax.periodic ? 2 : 1;
    return w;
}

std::size_t ModelSpec::first_layer_width() const { return rff ? 2 * rff->width : embedded_width(); }

void ModelSpec::validate() const {
    if (in_dim == 0 || hidden_dim == 0 || depth == 0 || out_dim == 0)
        throw TensorError("ModelSpec: dimensions must be positive");
    if (!periodic_axes.empty() && periodic_axes.size() != in_dim)
        throw TensorError("ModelSpec: periodic_axes must have one entry per input axis");
    for (const auto& ax : periodic_axes)
        if (ax.periodic && !(ax.period > 0.0)) throw TensorError("ModelSpec: periodic axis needs a positive period");
    if (rff && rff->width == 0) throw TensorError("ModelSpec: rff width must be positive");
}

namespace {

// Same engine and distributions as the reference Rng (rng.hpp:10-27): one
// fresh std::normal_distribution per draw, so libstdc++ reproduces its values.
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    double normal(double mean, double stddev) { return std::normal_distribution<double>(mean, stddev)(engine_); }

private:
    std::mt19937_64 engine_;
};

}  // namespace

Model::Model(ModelSpec spec, std::uint64_t seed) : spec_(std::move(spec)) {
    spec_.validate();
    Rng rng(seed);
    if (spec_.rff) {  // frozen RFF frequencies drawn first (model.cpp:58-62)
        rff_B_.shape = {spec_.embedded_width(), spec_.rff->width};
        rff_B_.data.resize(spec_.embedded_width() * spec_.rff->width);
        for (auto& v : rff_B_.data) v = rng.normal(spec_.rff->mean, spec_.rff->sigma);
    }
    auto make_layer = [&](std::size_t in, std::size_t out, std::size_t index) {
        const double xavier = std::sqrt(2.0 / static_cast<double>(in + out));
        Tensor W{{in, out}, std::vector<double>(in * out)};
        for (auto& v : W.data) v = rng.normal(0.0, xavier);
        const std::string base = "layer" + std::to_string(index) + ".";
        if (spec_.rwf) {
            params_.push_back({base + "V", std::move(W)});
            Tensor s{{1, out}, std::vector<double>(out)};
            for (auto& v : s.data) v = rng.normal(spec_.rwf->mean, spec_.rwf->stddev);
            params_.push_back({base + "s", std::move(s)});
        } else {
            params_.push_back({base + "W", std::move(W)});
        }
        params_.push_back({base + "b", Tensor{{1, out}, std::vector<double>(out, 0.0)}});
    };
    std::size_t in = spec_.first_layer_width();
    for (std::size_t l = 0; l < spec_.depth; ++l) {
        make_layer(in, spec_.hidden_dim, l);
        in = spec_.hidden_dim;
    }
    make_layer(in, spec_.out_dim, spec_.depth);
    for (std::size_t a = 0; a < spec_.periodic_axes.size(); ++a) {
        const auto& ax = spec_.periodic_axes[a];
        if (ax.periodic && ax.trainable)
            params_.push_back({"periodic.P" + std::to_string(a), Tensor{{}, std::vector<double>{ax.period}}});
    }
}

std::size_t Model::trainable_count() const {
    std::size_t n = 0;
    for (const auto& p : params_) n += p.value.size();
    return n;
}

// ---------------------------------------------------------------------------
// sampling (sampling.cpp:10-54) and collocation (trainer.cpp:47-128)
// ---------------------------------------------------------------------------

std::vector<double> linspace(double lo, double hi, std::size_t n) {
    std::vector<double> v(n);
    if (n == 1) {
        v[0] = lo;
        return v;
    }
    const double h = (hi - lo) / static_cast<double>(n - 1);
    for (std::size_t i = 0; i < n; ++i) v[i] = lo + static_cast<double>(i) * h;
    v[n - 1] = hi;
    return v;
}

Points sample_uniform(const Domain& dom, std::span<const std::size_t> dims) {
    if (dims.size() != dom.dim()) throw TensorError("sample_uniform: dims/domain mismatch");
    std::size_t total = 1;
    std::vector<std::vector<double>> axes(dom.dim());
    for (std::size_t a = 0; a < dom.dim(); ++a) {
        if (dims[a] == 0) throw TensorError("sample_uniform: zero points on an axis");
        axes[a] = linspace(dom.bounds[a][0], dom.bounds[a][1], dims[a]);
        total *= dims[a];
    }
    Points pts;
    pts.coords.assign(dom.dim(), std::vector<double>(total));
    for (std::size_t idx = 0; idx < total; ++idx) {  // last axis fastest
        std::size_t rem = idx;
        for (std::size_t a = dom.dim(); a-- > 0;) {
            pts.coords[a][idx] = axes[a][rem % dims[a]];
            rem /= dims[a];
        }
    }
    return pts;
}

Points sample_lhs(const Domain& dom, std::size_t n, std::uint64_t seed) {
    if (n == 0) throw TensorError("sample_lhs: n must be positive");
    std::mt19937_64 eng(seed);
    Points pts;
    pts.coords.assign(dom.dim(), std::vector<double>(n));
    std::vector<std::size_t> perm(n);
    for (std::size_t a = 0; a < dom.dim(); ++a) {
        std::iota(perm.begin(), perm.end(), 0);
        std::shuffle(perm.begin(), perm.end(), eng);
        const double lo = dom.bounds[a][0], hi = dom.bounds[a][1];
        const double h = (hi - lo) / static_cast<double>(n);
        for (std::size_t i = 0; i < n; ++i) {
            const double jitter = std::uniform_real_distribution<double>(0.0, 1.0)(eng);
            pts.coords[a][i] = lo + (static_cast<double>(perm[i]) + jitter) * h;
        }
    }
    return pts;
}

Points sample_lhs_per_axis(const Domain& dom, std::span<const std::size_t> dims, std::uint64_t seed) {
    if (dims.size() != dom.dim()) throw TensorError("sample_lhs_per_axis: dims/domain mismatch");
    std::mt19937_64 eng(seed);
    std::vector<std::vector<double>> axes(dom.dim());
    std::size_t total = 1;
    for (std::size_t a = 0; a < dom.dim(); ++a) {
        const double lo = dom.bounds[a][0], hi = dom.bounds[a][1];
        const std::size_t n = dims[a];
        if (n == 0) throw TensorError("sample_lhs_per_axis: zero points on an axis");
        const double h = (hi - lo) / static_cast<double>(n);
        axes[a].resize(n);
        for (std::size_t i = 0; i < n; ++i)
            axes[a][i] = lo + (static_cast<double>(i) + std::uniform_real_distribution<double>(0.0, 1.0)(eng)) * h;
        total *= n;
    }
    Points pts;
    pts.coords.assign(dom.dim(), std::vector<double>(total));
    for (std::size_t idx = 0; idx < total; ++idx) {  // last axis fastest
        std::size_t rem = idx;
        for (std::size_t a = dom.dim(); a-- > 0;) {
            const std::size_t k = rem % dims[a];
            rem /= dims[a];
            pts.coords[a][idx] = axes[a][k];
        }
    }
    return pts;
}

CollocationData build_collocation(const TrainingProblem& prob, const CollocationConfig& cc, std::uint64_t seed) {
    const Domain& dom = prob.domain;
    const std::size_t d = dom.dim();
    if (d < 2) throw TensorError("build_collocation: need at least one spatial axis plus time");
    CollocationData data;
    switch (cc.mode) {
        case CollocationConfig::Mode::uniform: data.interior = sample_uniform(dom, cc.dims); break;
        case CollocationConfig::Mode::lhs: data.interior = sample_lhs(dom, cc.n, seed); break;
        case CollocationConfig::Mode::lhs_per_axis: data.interior = sample_lhs_per_axis(dom, cc.dims, seed); break;
    }
    const std::size_t spatial = d - 1;
    Points ic;
    if (spatial == 1) {
        ic.coords.push_back(linspace(dom.bounds[0][0], dom.bounds[0][1], cc.n_ic));
    } else {
        const auto per_axis = static_cast<std::size_t>(
            std::ceil(std::pow(static_cast<double>(cc.n_ic), 1.0 / static_cast<double>(spatial))));
        Domain sdom{std::vector<std::array<double, 2>>(dom.bounds.begin(), dom.bounds.end() - 1)};
        std::vector<std::size_t> dims(spatial, per_axis);
        ic = sample_uniform(sdom, dims);
    }
    const std::size_t n_ic = ic.coords[0].size();
    ic.coords.push_back(std::vector<double>(n_ic, 0.0));  // t = 0
    data.ic_points = std::move(ic);
    const std::size_t fields = prob.residual.field_count();
    data.ic_targets.assign(fields, std::vector<double>(n_ic));
    std::vector<double> xbuf(spatial);
    for (std::size_t i = 0; i < n_ic; ++i) {
        for (std::size_t a = 0; a < spatial; ++a) xbuf[a] = data.ic_points.coords[a][i];
        std::vector<double> vals = prob.initial(xbuf);
        if (vals.size() != fields) throw TensorError("build_collocation: initial() field count mismatch");
        for (std::size_t f = 0; f < fields; ++f) data.ic_targets[f][i] = vals[f];
    }
    if (prob.bc != TrainingProblem::Bc::hard) {
        const auto ts = linspace(dom.bounds[d - 1][0], dom.bounds[d - 1][1], cc.n_bc);
        auto trace = [&](double xval) {
            Points p;
            p.coords.push_back(std::vector<double>(cc.n_bc, xval));
            for (std::size_t a = 1; a < spatial; ++a)
                p.coords.push_back(std::vector<double>(cc.n_bc, 0.5 * (dom.bounds[a][0] + dom.bounds[a][1])));
            p.coords.push_back(ts);
            return p;
        };
        data.bc_a = trace(dom.bounds[0][0]);
        data.bc_b = trace(dom.bounds[0][1]);
        if (prob.bc == TrainingProblem::Bc::dirichlet_zero) {
            Points both;
            for (std::size_t a = 0; a < d; ++a) {
                std::vector<double> col(2 * cc.n_bc);
                for (std::size_t i = 0; i < cc.n_bc; ++i) {
                    col[i] = data.bc_a.coords[a][i];
                    col[cc.n_bc + i] = data.bc_b.coords[a][i];
                }
                both.coords.push_back(std::move(col));
            }
            data.bc_a = std::move(both);
            data.bc_b = Points{};
            data.bc_targets.assign(fields, std::vector<double>(2 * cc.n_bc, 0.0));
        }
    }
    return data;
}

std::uint64_t param_hash(const std::vector<NamedTensor>& params) {
    std::uint64_t h = 1469598103934665603ULL;
    auto mix = [&h](const unsigned char* p, std::size_t n) {
        for (std::size_t i = 0; i < n; ++i) {
            h ^= p[i];
            h *= 1099511628211ULL;
        }
    };
    for (const auto& p : params) {
        mix(reinterpret_cast<const unsigned char*>(p.name.data()), p.name.size());
        mix(reinterpret_cast<const unsigned char*>(p.value.data.data()), p.value.data.size() * 8);
    }
    return h;
}

// ---------------------------------------------------------------------------
// worker contexts over the C ABI
// ---------------------------------------------------------------------------

namespace {

struct Ctx {
    pnx_ctx* ctx = nullptr;
    ~Ctx() {
        if (ctx) pnx_destroy(ctx);
    }
    void check(int rc) const {
        if (rc != PNX_OK) throw TensorError(pnx_last_error(ctx));
    }
};

int pde_code(PdeId id) {
    switch (id) {
        case PdeId::advection: return PNX_PDE_ADVECTION;
        case PdeId::allen_cahn: return PNX_PDE_ALLEN_CAHN;
        case PdeId::burgers: return PNX_PDE_BURGERS;
        case PdeId::maxwell_te: return PNX_PDE_MAXWELL_TE;
        case PdeId::ns_steady: return PNX_PDE_NS_STEADY;
        case PdeId::maxwell_te_eh: return PNX_PDE_MAXWELL_TE_EH;
    }
    return -1;
}

std::vector<double> axis_major(const Points& p) {
    std::vector<double> v;
    for (const auto& c : p.coords) v.insert(v.end(), c.begin(), c.end());
    return v;
}

std::vector<double> field_major(const std::vector<std::vector<double>>& t) {
    std::vector<double> v;
    for (const auto& c : t) v.insert(v.end(), c.begin(), c.end());
    return v;
}

// pnx_model_desc / pnx_problem_desc of a Model + TrainingProblem (the arrays
// they point into live in the Descs object)
struct Descs {
    std::vector<int32_t> per, tr;
    std::vector<double> period;
    pnx_model_desc md{};
    pnx_problem_desc pd{};
    Descs(const Model& m, const TrainingProblem& prob) {
        const ModelSpec& s = m.spec();
        for (const auto& ax : s.periodic_axes) {
            per.push_back(ax.periodic ? 1 : 0);
            period.push_back(ax.period);
            tr.push_back(ax.trainable ? 1 : 0);
        }
        md = pnx_model_desc{static_cast<int32_t>(s.in_dim), static_cast<int32_t>(s.hidden_dim),
                            static_cast<int32_t>(s.depth), static_cast<int32_t>(s.out_dim),
                            static_cast<int32_t>(s.activation), s.sine_w0, static_cast<int32_t>(per.size()),
                            per.data(), period.data(), tr.data(), s.rff ? static_cast<int32_t>(s.rff->width) : 0,
                            s.rff ? m.rff_matrix().data.data() : nullptr, s.rwf ? 1 : 0};
        pd = pnx_problem_desc{pde_code(prob.residual.id), prob.residual.advection_c, prob.residual.epsilon,
                              prob.residual.mu, prob.residual.reynolds, static_cast<int32_t>(prob.bc)};
    }
};

// causality / Poynting options of one worker context (trainer.cpp:240-247, 361-367)
void configure_objective(pnx_ctx* c, const TrainingProblem& prob, const TrainConfig& cfg) {
    auto check = [c](int rc) {
        if (rc != PNX_OK) throw TensorError(pnx_last_error(c));
    };
    const auto& dom = prob.domain.bounds;
    if (cfg.causality.enabled)  // segments over the last axis
        check(pnx_set_causality(c, cfg.causality.segments, cfg.causality.epsilon, dom.back()[0], dom.back()[1]));
    if (cfg.poynting.weight > 0.0 && prob.residual.id == PdeId::maxwell_te) {
        const double box[6] = {dom[0][0], dom[0][1], dom[1][0], dom[1][1], dom.back()[0], dom.back()[1]};
        check(pnx_set_poynting(c, cfg.poynting.weight, static_cast<int32_t>(cfg.poynting.grid),
                               static_cast<int32_t>(cfg.poynting.time_samples), box));
    }
}

// Single worker context over a point set (the full-batch L-BFGS objective,
// trainer.cpp:564-585).
std::unique_ptr<Ctx> make_worker(const Model& m, const TrainingProblem& prob, const Points& shard,
                                 const CollocationData& data, const TrainConfig& cfg) {
    Descs d(m, prob);
    auto w = std::make_unique<Ctx>();
    if (pnx_create(&d.md, &d.pd, cfg.device, &w->ctx) != PNX_OK) throw TensorError(pnx_create_error());
    auto pts = axis_major(shard);
    w->check(pnx_set_points(w->ctx, pts.data(), static_cast<int64_t>(shard.count()),
                            static_cast<int32_t>(shard.coords.size())));
    auto ic = axis_major(data.ic_points);
    auto ict = field_major(data.ic_targets);
    w->check(pnx_set_ic(w->ctx, ic.data(), ict.data(), static_cast<int64_t>(data.ic_points.count())));
    if (prob.bc != TrainingProblem::Bc::hard) {
        auto a = axis_major(data.bc_a), b = axis_major(data.bc_b);
        auto t = field_major(data.bc_targets);
        w->check(pnx_set_bc(w->ctx, a.data(), b.empty() ? nullptr : b.data(), t.empty() ? nullptr : t.data(),
                            static_cast<int64_t>(data.bc_a.count())));
    }
    configure_objective(w->ctx, prob, cfg);
    return w;
}

// The data-parallel group (pnx_dp): W ranks, worker w on GPU
// cfg.device + w % gpus, one NCCL all-reduce per step, device Adam replicas.
struct Group {
    pnx_dp* dp = nullptr;
    ~Group() {
        if (dp) pnx_dp_destroy(dp);
    }
    void check(int rc) const {
        if (rc != PNX_OK) throw TensorError(pnx_dp_last_error(dp));
    }
};

std::unique_ptr<Group> make_group(const Model& m, const TrainingProblem& prob, const CollocationData& data,
                                  const TrainConfig& cfg, int W) {
    int ndev = 0;
    if (pnx_device_count(&ndev) != PNX_OK || ndev <= cfg.device)
        throw TensorError("pnx: no CUDA device (the B200 path has no CPU fallback)");
    const int gpus = cfg.gpus > 0 ? std::min(cfg.gpus, ndev - cfg.device) : ndev - cfg.device;
    std::vector<int> devices;
    for (int w = 0; w < W; ++w) devices.push_back(cfg.device + w % gpus);
    Descs d(m, prob);
    auto g = std::make_unique<Group>();
    if (pnx_dp_create(&d.md, &d.pd, devices.data(), W, &g->dp) != PNX_OK) throw TensorError(pnx_create_error());
    if (data.interior.count() < static_cast<std::size_t>(W))
        throw TensorError("data parallel: fewer interior points than workers");
    auto pts = axis_major(data.interior);
    g->check(pnx_dp_set_points(g->dp, pts.data(), static_cast<int64_t>(data.interior.count()),
                               static_cast<int32_t>(data.interior.coords.size())));
    auto ic = axis_major(data.ic_points);
    auto ict = field_major(data.ic_targets);
    g->check(pnx_dp_set_ic(g->dp, ic.data(), ict.data(), static_cast<int64_t>(data.ic_points.count())));
    if (prob.bc != TrainingProblem::Bc::hard) {
        auto a = axis_major(data.bc_a), b = axis_major(data.bc_b);
        auto t = field_major(data.bc_targets);
        g->check(pnx_dp_set_bc(g->dp, a.data(), b.empty() ? nullptr : b.data(), t.empty() ? nullptr : t.data(),
                               static_cast<int64_t>(data.bc_a.count())));
    }
    for (int w = 0; w < W; ++w) {
        pnx_ctx* c = nullptr;
        g->check(pnx_dp_rank_ctx(g->dp, w, &c));
        configure_objective(c, prob, cfg);
    }
    return g;
}

std::vector<double> flatten(const std::vector<NamedTensor>& ps) {
    std::vector<double> v;
    for (const auto& p : ps) v.insert(v.end(), p.value.data.begin(), p.value.data.end());
    return v;
}

double dot(const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

// Limited-memory BFGS with a strong-Wolfe line search (lbfgs.cpp:22-155).
class Lbfgs {
public:
    explicit Lbfgs(LbfgsConfig c) : cfg_(c) {}
    struct Result {
        double loss = 0.0;
        bool converged = false, line_search_failed = false;
    };
    using Fn = std::function<double(const std::vector<double>&, std::vector<double>&)>;

    std::vector<double> apply_inverse_hessian(const std::vector<double>& v) const {
        std::vector<double> q = v;
        std::vector<double> alpha(pairs_.size());
        for (std::size_t i = pairs_.size(); i-- > 0;) {
            alpha[i] = pairs_[i].rho * dot(pairs_[i].s, q);
            for (std::size_t k = 0; k < q.size(); ++k) q[k] -= alpha[i] * pairs_[i].y[k];
        }
        if (!pairs_.empty()) {
            const double sc = dot(pairs_.back().s, pairs_.back().y) / dot(pairs_.back().y, pairs_.back().y);
            for (auto& x : q) x *= sc;
        }
        for (std::size_t i = 0; i < pairs_.size(); ++i) {
            const double beta = pairs_[i].rho * dot(pairs_[i].y, q);
            for (std::size_t k = 0; k < q.size(); ++k) q[k] += (alpha[i] - beta) * pairs_[i].s[k];
        }
        return q;
    }

    Result step(std::vector<double>& x, const Fn& fn) {
        Result res;
        std::vector<double> g(x.size());
        double f0;
        if (have_grad_) {
            g = last_grad_;
            f0 = last_loss_;
        } else {
            f0 = fn(x, g);
        }
        res.loss = f0;
        const double gn = std::sqrt(dot(g, g));
        if (gn < cfg_.grad_tol) {
            res.converged = true;
            return res;
        }
        std::vector<double> p = apply_inverse_hessian(g);
        for (auto& v : p) v = -v;
        double dphi0 = dot(g, p);
        if (dphi0 >= 0.0) {
            for (std::size_t k = 0; k < p.size(); ++k) p[k] = -g[k];
            dphi0 = dot(g, p);
            pairs_.clear();
        }
        int evals = 0;
        std::vector<double> gt(x.size()), xt(x.size());
        auto phi = [&](double a, double& d) {
            for (std::size_t k = 0; k < x.size(); ++k) xt[k] = x[k] + a * p[k];
            const double f = fn(xt, gt);
            ++evals;
            d = dot(gt, p);
            return f;
        };
        const double c1 = cfg_.c1, c2 = cfg_.c2;
        double accepted = -1.0, f_acc = 0.0;
        double a_prev = 0.0, f_prev = f0, d_prev = dphi0;
        double a = pairs_.empty() ? std::min(1.0, 1.0 / std::max(gn, 1e-12)) : 1.0;
        double lo = -1.0, hi = -1.0, f_lo = 0.0, d_lo = 0.0, f_hi = 0.0;
        bool zooming = false;
        while (evals < cfg_.max_line_search) {
            if (!zooming) {
                double d;
                const double f = phi(a, d);
                if (f > f0 + c1 * a * dphi0 || (evals > 1 && f >= f_prev)) {
                    lo = a_prev; f_lo = f_prev; d_lo = d_prev; hi = a; f_hi = f; zooming = true;
                    continue;
                }
                if (std::abs(d) <= -c2 * dphi0) { accepted = a; f_acc = f; break; }
                if (d >= 0.0) {
                    lo = a; f_lo = f; d_lo = d; hi = a_prev; f_hi = f_prev; zooming = true;
                    continue;
                }
                a_prev = a; f_prev = f; d_prev = d;
                a *= 2.0;
            } else {
                const double dd = hi - lo, denom = f_hi - f_lo - d_lo * dd;
                double trial = std::abs(denom) < 1e-300 ? 0.5 * (lo + hi) : lo - 0.5 * d_lo * dd * dd / denom;
                const double span = std::abs(hi - lo);
                if (!(trial >= std::min(lo, hi) + 0.1 * span && trial <= std::max(lo, hi) - 0.1 * span))
                    trial = 0.5 * (lo + hi);
                double d;
                const double f = phi(trial, d);
                if (f > f0 + c1 * trial * dphi0 || f >= f_lo) {
                    hi = trial; f_hi = f;
                } else {
                    if (std::abs(d) <= -c2 * dphi0) { accepted = trial; f_acc = f; break; }
                    if (d * (hi - lo) >= 0.0) { hi = lo; f_hi = f_lo; }
                    lo = trial; f_lo = f; d_lo = d;
                }
                if (span < 1e-16 * std::max(1.0, std::abs(lo))) break;
            }
        }
        if (accepted < 0.0) {
            pairs_.clear();
            have_grad_ = false;
            res.line_search_failed = true;
            return res;
        }
        Pair pr;
        pr.s.resize(x.size());
        pr.y.resize(x.size());
        for (std::size_t k = 0; k < x.size(); ++k) {
            const double xn = x[k] + accepted * p[k];
            pr.s[k] = xn - x[k];
            pr.y[k] = gt[k] - g[k];
            x[k] = xn;
        }
        const double sy = dot(pr.s, pr.y);
        if (sy > cfg_.curvature_floor) {
            pr.rho = 1.0 / sy;
            pairs_.push_back(std::move(pr));
            while (pairs_.size() > static_cast<std::size_t>(cfg_.history)) pairs_.pop_front();
        }
        last_grad_ = gt;
        last_loss_ = f_acc;
        have_grad_ = true;
        res.loss = f_acc;
        return res;
    }

private:
    struct Pair {
        std::vector<double> s, y;
        double rho = 0.0;
    };
    LbfgsConfig cfg_;
    std::deque<Pair> pairs_;
    std::vector<double> last_grad_;
    double last_loss_ = 0.0;
    bool have_grad_ = false;
};


}  // namespace

bool SwitchPolicy::should_switch(long epoch, std::span<const double> h) const {  // optim.cpp:75-95
    switch (trigger) {
        case Trigger::none: return false;
        case Trigger::epoch_threshold: return epoch >= epoch_threshold;
        case Trigger::loss_plateau: {
            if (h.empty()) throw TensorError("switch policy: plateau trigger needs loss history");
            if (plateau_window <= 0 || h.size() < static_cast<std::size_t>(plateau_window) + 1) return false;
            const double past = h[h.size() - 1 - static_cast<std::size_t>(plateau_window)], now = h.back();
            if (past <= 0.0) return true;
            return (past - now) / past < plateau_rel_improvement;
        }
    }
    return false;
}

std::vector<Tensor> data_parallel_gradient(Model& model, const TrainingProblem& prob, const TrainConfig& cfg,
                                           int workers) {
    const int W = std::max(1, workers);
    CollocationData data = build_collocation(prob, cfg.collocation, cfg.seed);
    auto grp = make_group(model, prob, data, cfg, W);
    std::vector<double> p = flatten(model.trainable());
    grp->check(pnx_dp_set_params(grp->dp, p.data()));
    std::vector<double> g(p.size());
    double losses[4];
    const double lam[3] = {1.0, 1.0, 1.0};
    grp->check(pnx_dp_step(grp->dp, lam, 0, losses, g.data()));  // no update: the averaged gradient
    std::vector<Tensor> out;
    std::size_t at = 0;
    for (const auto& prm : model.trainable()) {
        Tensor t{prm.value.shape, std::vector<double>(g.begin() + static_cast<std::ptrdiff_t>(at),
                                                      g.begin() + static_cast<std::ptrdiff_t>(at + prm.value.size()))};
        at += prm.value.size();
        out.push_back(std::move(t));
    }
    return out;
}

TrainResult train(Model& model, const TrainingProblem& prob, const TrainConfig& cfg) {
    TrainResult result;
    const int W = std::max(1, cfg.workers);
    CollocationData data = build_collocation(prob, cfg.collocation, cfg.seed);
    // W worker replicas on the GPUs, one NCCL all-reduce + device Adam per epoch
    // (trainer.cpp:441-460, 264-281, 626-638)
    auto grp = make_group(model, prob, data, cfg, W);
    std::vector<double> p = flatten(model.trainable());
    grp->check(pnx_dp_set_params(grp->dp, p.data()));
    const AdamConfig& ad = cfg.adam;
    grp->check(pnx_dp_set_optimizer(grp->dp, ad.lr, cfg.scheduler_gamma, ad.beta1, ad.beta2, ad.eps));
    grp->check(pnx_dp_set_graph(grp->dp, 1));  // one CUDA graph per device and loss weighting
    std::array<double, 3> lam = cfg.lambdas;   // LossState (losses.hpp:70-78)
    const bool has_bc = prob.bc != TrainingProblem::Bc::hard;
    const bool pen_on = cfg.poynting.weight > 0.0 && prob.residual.id == PdeId::maxwell_te;
    const std::size_t P = p.size();
    std::vector<double> loss_history, terms(3 * P), g(P), replica(P);
    bool switched = false;
    long next_epoch = 0;
    auto sync_model = [&](int rank) {  // the replica a rank trains -> Model::trainable()
        grp->check(pnx_dp_get_params(grp->dp, rank, p.data()));
        std::size_t at = 0;
        for (auto& prm : model.trainable())
            for (auto& x : prm.value.data) x = p[at++];
    };
    for (long epoch = 0; epoch < cfg.epochs; ++epoch) {
        double losses[4] = {0, 0, 0, 0};
        try {
            // optional interior resampling (trainer.cpp:421-434): fresh LHS set with seed + epoch
            if (cfg.collocation.resample_every > 0 && epoch > 0 && epoch % cfg.collocation.resample_every == 0 &&
                cfg.collocation.mode != CollocationConfig::Mode::uniform) {
                CollocationData rd =
                    build_collocation(prob, cfg.collocation, cfg.seed + static_cast<std::uint64_t>(epoch));
                data.interior = std::move(rd.interior);
                auto pts = axis_major(data.interior);
                grp->check(pnx_dp_set_points(grp->dp, pts.data(), static_cast<int64_t>(data.interior.count()),
                                             static_cast<int32_t>(data.interior.coords.size())));
            }
            const bool balance_now = cfg.balancing.enabled && cfg.balancing.update_period > 0 &&
                                     epoch % cfg.balancing.update_period == 0;
            if (!balance_now) {
                grp->check(pnx_dp_step(grp->dp, lam.data(), 1, losses, nullptr));
            } else {  // trainer.cpp:462-506: per-term gradients (one all-reduce), new lambdas
                grp->check(pnx_dp_step_terms(grp->dp, terms.data(), losses));
                auto norm = [&](int k) {
                    double s2 = 0.0;
                    for (std::size_t i = 0; i < P; ++i) s2 += terms[k * P + i] * terms[k * P + i];
                    return std::sqrt(s2);
                };
                std::array<double, 3> norms{norm(0), norm(1), has_bc ? norm(2) : 0.0};
                const double a = cfg.balancing.alpha;
                const std::array<double, 3> old = lam;
                const double tot = norms[0] + norms[1] + (has_bc ? norms[2] : 0.0);
                for (int k = 0; k < (has_bc ? 3 : 2); ++k)
                    lam[static_cast<std::size_t>(k)] = a * lam[static_cast<std::size_t>(k)] +
                                                       (1.0 - a) * (tot / std::max(norms[static_cast<std::size_t>(k)], 1e-9));
                if (pen_on) {  // total gradient under the previous weights (trainer.cpp:491-498)
                    double l4[4];
                    grp->check(pnx_dp_step(grp->dp, old.data(), 1, l4, nullptr));
                } else {
                    for (std::size_t i = 0; i < P; ++i) {
                        double s2 = lam[0] * terms[i] + lam[1] * terms[P + i];
                        if (has_bc) s2 += lam[2] * terms[2 * P + i];
                        g[i] = s2;
                    }
                    grp->check(pnx_dp_apply_gradient(grp->dp, g.data()));
                    grp->check(pnx_dp_check(grp->dp));  // Adam's non-finite check (optim.cpp:16-22)
                }
            }
        } catch (const std::exception& e) {  // TensorError with the reference's text
            result.aborted = true;
            result.abort_reason = e.what();
            break;
        }
        const double lr = ad.lr * std::pow(cfg.scheduler_gamma, static_cast<double>(epoch));  // optim.cpp:71-73
        result.metrics.push_back({epoch, losses[0], losses[1], losses[2], lam[0], lam[1], lam[2], lr});
        loss_history.push_back(lam[0] * losses[0] + lam[1] * losses[1] + lam[2] * losses[2]);
        if (cfg.on_sync) {  // one hash per replica, each from its own device copy (trainer.cpp:540-544)
            std::vector<std::uint64_t> hashes;
            std::vector<NamedTensor> view = model.trainable();
            for (int w = 0; w < W; ++w) {
                grp->check(pnx_dp_get_params(grp->dp, w, replica.data()));
                std::size_t at = 0;
                for (auto& prm : view)
                    for (auto& x : prm.value.data) x = replica[at++];
                hashes.push_back(param_hash(view));
            }
            cfg.on_sync(epoch, hashes);
        }
        ++result.epochs_run;
        if (cfg.lbfgs_max_iters > 0 && cfg.switch_policy.should_switch(epoch, loss_history)) {
            switched = true;
            next_epoch = epoch + 1;
            break;
        }
    }
    sync_model(0);
    if (switched && !result.aborted) {  // quasi-Newton refinement, full batch (trainer.cpp:558-617)
        result.switched_to_lbfgs = true;
        auto full = make_worker(model, prob, data.interior, data, cfg);
        std::array<double, 3> last{};
        double pen = 0.0;
        auto objective = [&](const std::vector<double>& v, std::vector<double>& grad) {
            full->check(pnx_step(full->ctx, v.data(), lam.data(), grad.data(), last.data()));
            double f = lam[0] * last[0] + lam[1] * last[1] + lam[2] * last[2];
            if (pen_on) {
                full->check(pnx_last_penalty(full->ctx, &pen));
                f += cfg.poynting.weight * pen;
            }
            return f;
        };
        Lbfgs lb(cfg.lbfgs);
        for (long it = 0; it < cfg.lbfgs_max_iters; ++it) {
            Lbfgs::Result r;
            try {
                r = lb.step(p, objective);
            } catch (const std::exception& e) {
                result.aborted = true;
                result.abort_reason = e.what();
                break;
            }
            std::size_t at = 0;
            for (auto& prm : model.trainable())
                for (auto& x : prm.value.data) x = p[at++];
            result.metrics.push_back({next_epoch + it, last[0], last[1], last[2], lam[0], lam[1], lam[2], 0.0});
            ++result.epochs_run;
            if (r.converged) break;
            if (r.line_search_failed) {
                result.abort_reason = "line search failed; quasi-Newton phase stopped";
                break;
            }
        }
    }
    return result;
}

namespace {

// one Adam pass over [lo, hi) (optim.cpp:7-41, the same expression order)
void adam_range(double* __restrict p, double* __restrict m, double* __restrict v, const double* __restrict g,
                std::size_t lo, std::size_t hi, double lr, double b1, double b2, double eps, double bc1,
                double bc2) {
    for (std::size_t k = lo; k < hi; ++k) {
        m[k] = b1 * m[k] + (1.0 - b1) * g[k];
        v[k] = b2 * v[k] + (1.0 - b2) * g[k] * g[k];
        p[k] -= lr * (m[k] / bc1) / (std::sqrt(v[k] / bc2) + eps);
    }
}

}  // namespace

void adam_update(double* p, double* m, double* v, const double* g, std::size_t n, double lr,
                 const AdamConfig& a, std::int64_t t) {
    const double bc1 = 1.0 - std::pow(a.beta1, static_cast<double>(t));
    const double bc2 = 1.0 - std::pow(a.beta2, static_cast<double>(t));
    // elementwise and divide/sqrt-bound: large vectors split over host threads
    // (each element is computed exactly as in the serial loop)
    const std::size_t kMinPerThread = 16384;
    std::size_t nt = std::min<std::size_t>(std::max(1u, std::thread::hardware_concurrency()), 8);
    nt = std::max<std::size_t>(1, std::min(nt, n / kMinPerThread));
    if (nt <= 1) {
        adam_range(p, m, v, g, 0, n, lr, a.beta1, a.beta2, a.eps, bc1, bc2);
        return;
    }
    std::vector<std::thread> pool;
    const std::size_t per = (n + nt - 1) / nt;
    auto range = [&](std::size_t i) {
        const std::size_t lo = std::min(n, i * per), hi = std::min(n, lo + per);
        adam_range(p, m, v, g, lo, hi, lr, a.beta1, a.beta2, a.eps, bc1, bc2);
    };
    std::size_t started = 1;
    try {  // pinnlab_adam_step is a C entry point: ranges without a thread run here
        pool.reserve(nt - 1);
        for (; started < nt; ++started) pool.emplace_back(range, started);
    } catch (...) {
    }
    range(0);
    for (std::size_t i = started; i < nt; ++i) range(i);
    for (auto& th : pool) th.join();
}

}  // namespace pinnlab_b200

extern "C" int pinnlab_adam_step(double* p, double* m, double* v, const double* g, std::int64_t n,
                                 double lr, double beta1, double beta2, double eps, std::int64_t t) {
    pinnlab_b200::AdamConfig a;
    a.lr = lr;
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.eps = eps;
    pinnlab_b200::adam_update(p, m, v, g, static_cast<std::size_t>(n), lr, a, t);
    return 0;
}

