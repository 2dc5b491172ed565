// pnx_worker_epoch.hpp -- the reference-side binding of libpnx (include/pnx.h)
// into the pinnlab core: the body of run_worker_epoch (trainer.cpp:200-262)
// replaced by the B200 worker step.
//
// A maintainer edits trainer.cpp's run_worker_epoch to this body. To prove the
// binding compiles and runs against the UNMODIFIED reference without copying it,
// integration/Makefile force-includes this header ahead of the reference's own
// trainer.cpp: every call site of run_worker_epoch there (the epoch loop
// trainer.cpp:443/451, the L-BFGS objective :580, data_parallel_gradient
// :667/673) passes a non-const WorkerTask lvalue, for which the constrained
// overload below is a better match than the reference's
// run_worker_epoch(const WorkerTask&) (a less cv-qualified reference binding,
// [over.ics.rank]). The reference's Graph body stays compiled but is never
// called; its return type names WorkerOutput for this template.
//
// Per worker replica (task.model, one per worker, trainer.cpp:358-367) one pnx
// context lives on GPU (k % device count), k counting contexts in creation
// order. Points are uploaded when the worker's shard changes (resampling,
// trainer.cpp:421-434); causality and the Poynting penalty are configured once
// per context from TrainConfig (trainer.cpp:209-247). Errors come back as the
// reference's TensorError with the reference's text.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "pinnlab/losses.hpp"
#include "pinnlab/model.hpp"
#include "pinnlab/trainer.hpp"
#include "pnx.h"

namespace pinnlab {
namespace pnx_binding {

struct Slot {
    pnx_ctx* ctx = nullptr;
    std::vector<double> probe;  // cheap fingerprint of the uploaded shard
};

inline std::mutex& slots_mutex() {
    static std::mutex m;
    return m;
}
inline std::map<const void*, Slot>& slots() {
    static std::map<const void*, Slot> s;
    return s;
}

inline void check(pnx_ctx* c, int rc) {
    if (rc != PNX_OK) throw TensorError(c ? pnx_last_error(c) : pnx_create_error());
}

inline std::vector<double> axis_major(const Points& p) {
    std::vector<double> v;
    for (const Tensor& c : p.coords) v.insert(v.end(), c.data(), c.data() + c.size());
    return v;
}
inline std::vector<double> columns(const std::vector<Tensor>& t) {
    std::vector<double> v;
    for (const Tensor& c : t) v.insert(v.end(), c.data(), c.data() + c.size());
    return v;
}
// size + 17 evenly spaced coordinates per axis: changes when a shard is resampled
inline std::vector<double> fingerprint(const Points& p) {
    std::vector<double> f{static_cast<double>(p.count())};
    for (const Tensor& c : p.coords)
        for (std::size_t k = 0; k <= 16 && c.size() > 0; ++k) f.push_back(c[(c.size() - 1) * k / 16]);
    return f;
}

inline pnx_ctx* create(const Model& m, const TrainingProblem& prob, const CollocationData& shared,
                       const TrainConfig& cfg) {
    static std::atomic<int> created{0};
    int ndev = 0;
    check(nullptr, pnx_device_count(&ndev) == PNX_OK && ndev > 0 ? PNX_OK : PNX_ERR_CUDA);
    const ModelSpec& s = m.spec();
    std::vector<int32_t> per, tr;
    std::vector<double> period;
    for (const auto& ax : s.periodic_axes) {
        per.push_back(ax.periodic ? 1 : 0);
        period.push_back(ax.period);
        tr.push_back(ax.trainable ? 1 : 0);
    }
    pnx_model_desc md{static_cast<int32_t>(s.in_dim), static_cast<int32_t>(s.hidden_dim),
                      static_cast<int32_t>(s.depth), static_cast<int32_t>(s.out_dim),
                      static_cast<int32_t>(s.activation), s.sine_w0, static_cast<int32_t>(per.size()),
                      per.data(), period.data(), tr.data(), s.rff ? static_cast<int32_t>(s.rff->width) : 0,
                      s.rff ? m.rff_matrix().data() : nullptr, s.rwf ? 1 : 0};
    pnx_problem_desc pd{static_cast<int32_t>(prob.residual.id), prob.residual.advection_c, prob.residual.epsilon,
                        prob.residual.mu, 0.0, static_cast<int32_t>(prob.bc)};
    pnx_ctx* ctx = nullptr;
    check(nullptr, pnx_create(&md, &pd, created++ % ndev, &ctx));
    auto ic = axis_major(shared.ic_points);
    auto ict = columns(shared.ic_targets);
    check(ctx, pnx_set_ic(ctx, ic.data(), ict.data(), static_cast<int64_t>(shared.ic_points.count())));
    if (prob.bc != TrainingProblem::Bc::hard) {
        auto a = axis_major(shared.bc_a), b = axis_major(shared.bc_b);
        auto t = columns(shared.bc_targets);
        check(ctx, pnx_set_bc(ctx, a.data(), b.empty() ? nullptr : b.data(), t.empty() ? nullptr : t.data(),
                              static_cast<int64_t>(shared.bc_a.count())));
    }
    const auto& dom = prob.domain.bounds;
    if (cfg.causality.enabled)  // the shard is bucketed by its last coordinate inside the context
        check(ctx, pnx_set_causality(ctx, cfg.causality.segments, cfg.causality.epsilon, dom.back()[0],
                                     dom.back()[1]));
    if (cfg.poynting.weight > 0.0 && prob.residual.id == PdeId::maxwell_te) {
        const double box[6] = {dom[0][0], dom[0][1], dom[1][0], dom[1][1], dom.back()[0], dom.back()[1]};
        check(ctx, pnx_set_poynting(ctx, cfg.poynting.weight, static_cast<int32_t>(cfg.poynting.grid),
                                    static_cast<int32_t>(cfg.poynting.time_samples), box));
    }
    return ctx;
}

inline std::vector<Tensor> unflatten(const std::vector<NamedTensor>& like, const double* flat) {
    std::vector<Tensor> out;
    for (const auto& p : like) {
        Tensor g(p.value.shape());
        std::memcpy(g.data(), flat, g.size() * sizeof(double));
        flat += g.size();
        out.push_back(std::move(g));
    }
    return out;
}

}  // namespace pnx_binding

// run_worker_epoch(const WorkerTask&) -> WorkerOutput on the B200 path.
template <class Task>
    requires(!std::is_const_v<Task>)
auto run_worker_epoch(Task& task) {
    using Out = decltype(run_worker_epoch(std::as_const(task)));  // WorkerOutput (trainer.cpp:183-187)
    const Model& model = *task.model;
    const TrainConfig& cfg = *task.cfg;
    pnx_ctx* ctx = nullptr;
    bool upload = false;
    {
        std::lock_guard<std::mutex> lk(pnx_binding::slots_mutex());
        pnx_binding::Slot& s = pnx_binding::slots()[task.model];
        if (!s.ctx) s.ctx = pnx_binding::create(model, *task.prob, *task.shared, cfg);
        auto fp = pnx_binding::fingerprint(*task.interior);
        upload = fp != s.probe;
        if (upload) s.probe = std::move(fp);
        ctx = s.ctx;
    }
    if (upload) {
        auto pts = pnx_binding::axis_major(*task.interior);
        pnx_binding::check(ctx, pnx_set_points(ctx, pts.data(), static_cast<int64_t>(task.interior->count()),
                                               static_cast<int32_t>(task.interior->coords.size())));
    }
    std::vector<double> params;
    for (const auto& p : model.trainable()) params.insert(params.end(), p.value.data(), p.value.data() + p.value.size());
    std::vector<double> grad(params.size());
    double losses[3];
    pnx_binding::check(ctx, pnx_step(ctx, params.data(), task.lambdas.data(), grad.data(), losses));
    Out out;
    if (cfg.poynting.weight > 0.0 && task.prob->residual.id == PdeId::maxwell_te)
        pnx_binding::check(ctx, pnx_last_penalty(ctx, &out.losses.pen));
    out.losses.pde = losses[0];
    out.losses.ic = losses[1];
    out.losses.bc = task.prob->bc != TrainingProblem::Bc::hard ? losses[2] : 0.0;
    out.total_grad = pnx_binding::unflatten(model.trainable(), grad.data());
    if (task.want_term_grads) {  // balancing epochs: gradients of l_pde, l_ic, l_bc alone (trainer.cpp:256-260)
        std::vector<double> g3(3 * params.size());
        pnx_binding::check(ctx, pnx_step_terms(ctx, params.data(), g3.data(), nullptr));
        for (int k = 0; k < 3; ++k)
            if (k < 2 || task.prob->bc != TrainingProblem::Bc::hard)
                out.term_grads[k] = pnx_binding::unflatten(model.trainable(), g3.data() + k * params.size());
    }
    return out;
}

}  // namespace pinnlab
