"""Adam -> L-BFGS refinement (trainer.cpp:549-617) over the device step.

SwitchPolicy (optim.hpp:54-62, optim.cpp:75-95) decides when the Adam phase
ends; Lbfgs (lbfgs.hpp / lbfgs.cpp:22-155) is limited-memory BFGS with a
strong-Wolfe line search (bracketing, then quadratic zoom) and the two-loop
recursion seeded with s.y / y.y. The parameter, gradient and (s, y) history
vectors stay on the GPU in float64; every objective evaluation is one
pnx_step_device of a worker holding the whole interior (the reference's
full-batch task), f = sum_k lambda_k l_k (+ w_pen * penalty).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

__all__ = ["LbfgsConfig", "SwitchPolicy", "Lbfgs", "lbfgs_refine"]


@dataclass
class LbfgsConfig:
    """lbfgs.hpp:10-17."""
    history: int = 50
    c1: float = 1e-4
    c2: float = 0.9
    max_line_search: int = 25
    grad_tol: float = 1e-10
    curvature_floor: float = 1e-10


@dataclass
class SwitchPolicy:
    """trigger: 'none' | 'epoch' (epoch >= epoch_threshold) | 'plateau' (relative
    improvement over plateau_window epochs below plateau_rel_improvement)."""
    trigger: str = "none"
    epoch_threshold: int = 0
    plateau_window: int = 0
    plateau_rel_improvement: float = 0.0

    def should_switch(self, epoch: int, loss_history: List[float]) -> bool:
        if self.trigger == "epoch":
            return epoch >= self.epoch_threshold
        if self.trigger == "plateau":
            if not loss_history:
                from .pinn import TensorError
                raise TensorError("switch policy: plateau trigger needs loss history")
            if self.plateau_window <= 0 or len(loss_history) < self.plateau_window + 1:
                return False
            past, now = loss_history[-1 - self.plateau_window], loss_history[-1]
            if past <= 0.0:
                return True
            return (past - now) / past < self.plateau_rel_improvement
        return False


class Lbfgs:
    """One quasi-Newton iteration per step(); x is a float64 device tensor updated in place."""

    def __init__(self, cfg: LbfgsConfig = LbfgsConfig()):
        self.cfg = cfg
        self.pairs: List[Tuple[object, object, float]] = []
        self.have_grad = False
        self.last_grad = None
        self.last_loss = 0.0

    def apply_inverse_hessian(self, v):
        q = v.clone()
        alpha = [0.0] * len(self.pairs)
        for i in reversed(range(len(self.pairs))):
            s, y, rho = self.pairs[i]
            alpha[i] = rho * float(s.dot(q))
            q.add_(y, alpha=-alpha[i])
        if self.pairs:
            s, y, _ = self.pairs[-1]
            q.mul_(float(s.dot(y)) / float(y.dot(y)))
        for i, (s, y, rho) in enumerate(self.pairs):
            beta = rho * float(y.dot(q))
            q.add_(s, alpha=alpha[i] - beta)
        return q

    def step(self, x, fn: Callable):
        c = self.cfg
        if self.have_grad:
            g, f0 = self.last_grad, self.last_loss
        else:
            f0, g = fn(x)
        gn = float(g.norm())
        res = {"loss": f0, "grad_norm": gn, "converged": False, "line_search_failed": False}
        if gn < c.grad_tol:
            res["converged"] = True
            return res
        p = -self.apply_inverse_hessian(g)
        dphi0 = float(g.dot(p))
        if dphi0 >= 0.0:  # not a descent direction: steepest descent, history cleared
            p = -g
            dphi0 = float(g.dot(p))
            self.pairs.clear()
        evals = 0
        gt = [None]

        def phi(a):
            nonlocal evals
            f, gtr = fn(x + a * p)
            evals += 1
            gt[0] = gtr
            return f, float(gtr.dot(p))

        accepted, f_acc = -1.0, 0.0
        a_prev, f_prev, d_prev = 0.0, f0, dphi0
        a = min(1.0, 1.0 / max(gn, 1e-12)) if not self.pairs else 1.0
        lo = hi = -1.0
        f_lo = d_lo = f_hi = 0.0
        zooming = False
        while evals < c.max_line_search:
            if not zooming:
                f, d = phi(a)
                if f > f0 + c.c1 * a * dphi0 or (evals > 1 and f >= f_prev):
                    lo, f_lo, d_lo, hi, f_hi, zooming = a_prev, f_prev, d_prev, a, f, True
                    continue
                if abs(d) <= -c.c2 * dphi0:
                    accepted, f_acc = a, f
                    break
                if d >= 0.0:
                    lo, f_lo, d_lo, hi, f_hi, zooming = a, f, d, a_prev, f_prev, True
                    continue
                a_prev, f_prev, d_prev = a, f, d
                a *= 2.0
            else:
                dd = hi - lo
                denom = f_hi - f_lo - d_lo * dd
                trial = 0.5 * (lo + hi) if abs(denom) < 1e-300 else lo - 0.5 * d_lo * dd * dd / denom
                span = abs(hi - lo)
                if not (min(lo, hi) + 0.1 * span <= trial <= max(lo, hi) - 0.1 * span):
                    trial = 0.5 * (lo + hi)
                f, d = phi(trial)
                if f > f0 + c.c1 * trial * dphi0 or f >= f_lo:
                    hi, f_hi = trial, f
                else:
                    if abs(d) <= -c.c2 * dphi0:
                        accepted, f_acc = trial, f
                        break
                    if d * (hi - lo) >= 0.0:
                        hi, f_hi = lo, f_lo
                    lo, f_lo, d_lo = trial, f, d
                if span < 1e-16 * max(1.0, abs(lo)):
                    break
        if accepted < 0.0:
            self.pairs.clear()
            self.have_grad = False
            res["line_search_failed"] = True
            return res
        x_new = x + accepted * p
        s, y = x_new - x, gt[0] - g
        sy = float(s.dot(y))
        if sy > c.curvature_floor:
            self.pairs.append((s, y, 1.0 / sy))
            while len(self.pairs) > c.history:
                self.pairs.pop(0)
        x.copy_(x_new)
        self.last_grad, self.last_loss, self.have_grad = gt[0], f_acc, True
        res["loss"], res["grad_norm"] = f_acc, float(gt[0].norm())
        return res


def lbfgs_refine(worker, params, lambdas, iters: int, cfg: LbfgsConfig = LbfgsConfig(),
                 poynting_weight: float = 0.0, stream=None, group=None, world: int = 1, n_total: int = 0):
    """The quasi-Newton phase of train() (trainer.cpp:558-617). params: float32/
    float64 device tensor (updated in place, float32 view kept in sync). Returns
    (float64 params, records) with one (l_pde, l_ic, l_bc) record per iteration,
    as MetricsRecord logs them.

    The reference runs it full batch on one worker holding the whole interior.
    Sharded: `worker` may be a list of shard workers on this device and `world`
    > 1 ranks may each hold shards (process group `group`, `n_total` interior
    points overall). Every shard's gradient and losses are weighted by its share
    n_r / N and summed (one all-reduce of [grad | losses] per objective), which is
    exactly the full-batch mean objective: the PDE term is a mean over all
    points and the IC/BC/penalty terms are replicated on every shard. All ranks
    then take identical L-BFGS steps. (Causality weights stay per shard, as in
    the data-parallel Adam epochs, trainer.cpp:361-367.)"""
    import torch
    dev = params.device
    workers = list(worker) if isinstance(worker, (list, tuple)) else [worker]
    sharded = len(workers) > 1 or world > 1
    if sharded:
        n_loc = [getattr(w, "n_interior", 0) for w in workers]
        if world == 1 and not n_total:
            n_total = sum(n_loc)
        if not n_total or not all(n_loc):
            raise ValueError("lbfgs_refine: sharded objective needs every shard's interior size and n_total")
    x = params.detach().double().clone()
    p32 = torch.empty(x.numel(), dtype=torch.float32, device=dev)
    g32 = torch.empty_like(p32)
    losses = torch.zeros(3, dtype=torch.float64, device=dev)
    acc = torch.zeros(x.numel() + 4, dtype=torch.float64, device=dev)  # [grad | l_pde l_ic l_bc pen]
    lam = tuple(float(v) for v in lambdas)
    last = {}
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream

    def objective(v):
        p32.copy_(v)
        if not sharded:
            w = workers[0]
            w.step_device(p32, g32, lam, losses, stream=st)
            torch.cuda.synchronize(dev)
            w.check()
            l = losses.tolist()
            pen = w.penalty() if poynting_weight > 0.0 else 0.0
            grad = g32.double()
        else:
            acc.zero_()
            for w, n in zip(workers, n_loc):
                w.step_device(p32, g32, lam, losses, stream=st)
                torch.cuda.synchronize(dev)
                w.check()
                share = n / n_total
                acc[:-4].add_(g32.double(), alpha=share)
                acc[-4:-1].add_(losses, alpha=share)
                if poynting_weight > 0.0:
                    acc[-1] += share * w.penalty()
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
            l = acc[-4:-1].tolist()
            pen = float(acc[-1])
            grad = acc[:-4].clone()
        f = lam[0] * l[0] + lam[1] * l[1] + lam[2] * l[2]
        if poynting_weight > 0.0:
            f += poynting_weight * pen
        last["losses"] = l
        return f, grad

    lb = Lbfgs(cfg)
    records = []
    for _ in range(iters):
        r = lb.step(x, objective)
        records.append(tuple(last["losses"]))
        if r["converged"] or r["line_search_failed"]:
            break
    params.copy_(x.to(params.dtype))
    return x, records
