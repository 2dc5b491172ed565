"""Data-parallel train step across processes, one per GPU (torch.distributed).

Reference protocol (in-process threads there, processes + NCCL here):
* interior shards: contiguous, last shard takes the remainder   trainer.cpp:143-154
* IC/BC sets replicated on every rank                           trainer.cpp:225-232
* gradient average: rank-ordered sum, then x 1/W                trainer.cpp:264-281
* identical Adam update on every replica                        trainer.cpp:626-638
* replica consistency hash (FNV-1a) after each step             trainer.cpp:22-35, 540-544

The only collective is one all-reduce per step of the packed
[grad (P) | l_pde, l_ic, l_bc, pen] float32 buffer (the points are partitioned,
not exchanged); the 1/W scale is fused into the device Adam kernel
(pnx_adam_step_device). The C-ABI equivalent for a C++ host is pnx_dp
(include/pnx.h, paper_2604_15645_b200.pinn.DataParallelGroup).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .pinn import param_layout, shard_interior


def rank_shard(n_total: int, world: int, rank: int):
    """[lo, hi) of this rank's interior shard (shard_interior semantics)."""
    return shard_interior(n_total, world)[rank]


def allreduce_sum_(t, world: int, group=None):
    """Sum a gradient buffer over ranks in place (NCCL on GPU, gloo on CPU)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_average_(t, world: int, group=None):
    """average_grads (trainer.cpp:264-281): sum over ranks, then scale by 1/W."""
    allreduce_sum_(t, world, group)
    if world > 1:
        t.mul_(1.0 / world)
    return t


def param_hash(spec, flat: np.ndarray) -> int:
    """FNV-1a over (name bytes, little-endian float64 bytes) per tensor in
    trainable() order -- param_hash (trainer.cpp:22-35)."""
    h = 1469598103934665603
    at = 0
    flat = np.asarray(flat, dtype="<f8")
    for name, shape in param_layout(spec):
        n = int(np.prod(shape)) if shape else 1
        for b in name.encode() + flat[at:at + n].tobytes():
            h ^= b
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        at += n
    return h


def replica_hashes(spec, params, world: int, group=None) -> Sequence[int]:
    """on_sync hook payload: every rank's parameter hash (all_gather)."""
    h = param_hash(spec, np.asarray(params, dtype=np.float64))
    if world == 1:
        return [h]
    import torch
    import torch.distributed as dist
    # NCCL gathers device tensors; gloo (CPU tests) host tensors
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
    t = torch.tensor([h & 0x7FFFFFFFFFFFFFFF, h >> 63], dtype=torch.int64, device=dev)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(o[0]) | (int(o[1]) << 63) for o in out]


class DataParallelTrainer:
    """Synchronized Adam steps (trainer.cpp:419-555): per-worker device step ->
    all-reduce -> fused Adam(1/W). `worker` is one Worker (one GPU per process)
    or a list of local workers (several replicas in one process, e.g. to run a
    W-worker reference case on one GPU); W = world x local workers.

    Loss balancing (BalancingConfig, trainer.hpp:45-49): on epochs with
    epoch % update_period == 0 the workers return the per-term gradients
    (pnx_step_terms_device), the averaged term norms update the lambdas
    (update_global_weights, losses.cpp:154-162; two-term rule without BC,
    trainer.cpp:477-483) and the step uses lambda_k' g_k with the NEW weights --
    or, with a Poynting penalty, the total gradient under the old weights
    (trainer.cpp:491-498)."""

    def __init__(self, worker, params0: np.ndarray, world: int = 1, lr: float = 1e-3, gamma: float = 1.0,
                 betas=(0.9, 0.999), eps: float = 1e-8, device=None, group=None, balancing=None,
                 has_bc: bool = True, poynting: bool = False, graph: bool = False, check_every: int = 100):
        import torch
        self.torch = torch
        self.workers = list(worker) if isinstance(worker, (list, tuple)) else [worker]
        self.worker = self.workers[0]
        self.world, self.group = world, group
        self.W = world * len(self.workers)
        self.lr, self.gamma, self.betas, self.eps = lr, gamma, betas, eps
        self.balancing, self.has_bc, self.poynting = balancing, has_bc, poynting
        self.lam = [1.0, 1.0, 1.0]
        dev = device or torch.device("cuda", self.worker.device)
        self.params = torch.tensor(np.asarray(params0), dtype=torch.float32, device=dev)
        P = self.params.numel()
        # one packed all-reduce per step: [grad (P) | l_pde, l_ic, l_bc, pen]
        self.pack = torch.zeros(P + 4, dtype=torch.float32, device=dev)
        self.grad = self.pack[:P]
        self._wgrad = [self.grad] + [torch.zeros_like(self.params) for _ in self.workers[1:]]
        self._wloss = [torch.zeros(3, dtype=torch.float64, device=dev) for _ in self.workers]
        self._g3 = None
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.losses = torch.zeros(3, dtype=torch.float64, device=dev)
        self.t = 0
        self.epoch = 0
        # CUDA-graph mode: Adam keeps (steps, epoch) on the device so one captured
        # step (worker steps + the NCCL all-reduce + Adam) replays; a gloo
        # collective (CPU tests) cannot be captured
        backend = None
        if world > 1:
            import torch.distributed as dist
            backend = dist.get_backend(group)
        self.graph = graph and (world == 1 or backend == "nccl")
        self.state = torch.zeros(2, dtype=torch.float64, device=dev)
        self._graph = None
        self._glam = None
        self._warm = False
        self.loss_history = []
        # non-finite residuals / gradients (losses.cpp:86-90, optim.cpp:16-22) are
        # flagged on the device (the update is skipped) and raised here every
        # `check_every` steps and before parameters are read back
        self.check_every = check_every

    def _total(self, lam, st):
        """Every local worker's step, summed into the pack (gradient and loss
        terms), then ONE all-reduce of the pack."""
        P = self.params.numel()
        for i, (w, gb, lb) in enumerate(zip(self.workers, self._wgrad, self._wloss)):
            w.step_device(self.params, gb, lam, lb, stream=st)
            if i > 0:
                self.grad.add_(gb)
        ls = self._wloss[0].clone()
        for lb in self._wloss[1:]:
            ls.add_(lb)
        self.pack[P:P + 3].copy_(ls)
        allreduce_sum_(self.pack, self.world, self.group)

    def _balance(self, st):
        torch = self.torch
        P = self.params.numel()
        if self._g3 is None:
            self._g3 = [torch.zeros(3 * P, dtype=torch.float32, device=self.params.device) for _ in self.workers]
        for w, g3, lb in zip(self.workers, self._g3, self._wloss):
            w.step_terms_device(self.params, g3, lb, stream=st)
        # one all-reduce of [g_pde | g_ic | g_bc | l_pde, l_ic, l_bc] (trainer.cpp:469-498)
        gs = torch.zeros(3 * P + 3, dtype=torch.float32, device=self.params.device)
        for g3 in self._g3:
            gs[:3 * P].add_(g3)
        for lb in self._wloss:
            gs[3 * P:].add_(lb)
        allreduce_sum_(gs, self.world, self.group)
        terms = gs[:3 * P].view(3, P)
        self.pack[P:P + 3].copy_(gs[3 * P:])
        avg = terms.double() * (1.0 / self.W)
        norms = [float(avg[k].norm()) for k in range(3)]
        a, lam = self.balancing.alpha, self.lam
        if self.has_bc:
            tot = norms[0] + norms[1] + norms[2]
            self.lam = [a * lam[k] + (1.0 - a) * (tot / max(norms[k], 1e-9)) for k in range(3)]
        else:
            tot = norms[0] + norms[1]
            self.lam = [a * lam[0] + (1.0 - a) * (tot / max(norms[0], 1e-9)),
                        a * lam[1] + (1.0 - a) * (tot / max(norms[1], 1e-9)), lam[2]]
        if self.poynting:
            self._total(lam, st)  # total gradient under the previous weights
        else:
            self.grad.copy_(terms[0]).mul_(self.lam[0]).add_(terms[1], alpha=self.lam[1])
            if self.has_bc:
                self.grad.add_(terms[2], alpha=self.lam[2])

    def _finish(self, st):
        P = self.params.numel()
        self.losses.copy_(self.pack[P:P + 3])
        self.losses.mul_(1.0 / self.W)  # MetricsRecord: mean over workers (trainer.cpp:517-526)
        if self.graph:
            self.worker.adam_step_device_state(self.params, self.grad, self.m, self.v, self.state, self.lr,
                                               self.gamma, self.betas[0], self.betas[1], self.eps,
                                               grad_scale=1.0 / self.W, stream=st)
        else:
            lr = self.lr * self.gamma ** self.epoch  # ExponentialLr::at (optim.cpp:71-73)
            self.worker.adam_step_device(self.params, self.grad, self.m, self.v, self.t + 1, lr, self.betas[0],
                                         self.betas[1], self.eps, grad_scale=1.0 / self.W, stream=st)

    def _capture(self):
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.params.device)
        side.wait_stream(torch.cuda.current_stream(self.params.device))
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                cs = torch.cuda.current_stream(self.params.device).cuda_stream
                self._total(tuple(self.lam), cs)
                self._finish(cs)
        torch.cuda.current_stream(self.params.device).wait_stream(side)
        self._graph, self._glam = g, tuple(self.lam)

    def step(self, lambdas=None, stream=None, eager: bool = False):
        st = stream if stream is not None else self.torch.cuda.current_stream(self.params.device).cuda_stream
        b = self.balancing
        if lambdas is not None:
            self.lam = list(lambdas)
        balance_now = b is not None and b.enabled and b.update_period > 0 and self.epoch % b.update_period == 0
        if self.graph and not balance_now and self._warm and not eager:
            if self._graph is None or self._glam != tuple(self.lam):
                self._capture()  # the capture itself enqueues no work
            self._graph.replay()
        else:
            if balance_now:
                self._balance(st)
            else:
                self._total(tuple(self.lam), st)
            self._finish(st)
            self._warm = True
        self.t += 1
        self.epoch += 1
        if self.check_every and self.t % self.check_every == 0:
            self.check()
        return self.losses

    def check(self):
        """Raise TensorError for a non-finite residual or gradient since the last
        check and, with several ranks, if the replicas' parameter hashes differ
        (param_hash / on_sync, trainer.cpp:540-544)."""
        for w in self.workers:
            w.check()
        if self.world > 1:
            from .pinn import TensorError
            hs = replica_hashes(self.worker.spec, self.params.double().cpu().numpy(), self.world, self.group)
            if len(set(hs)) != 1:
                raise TensorError(f"data parallel: replica parameter hashes differ after step {self.t}: {hs}")

    def should_switch(self, policy) -> bool:
        """SwitchPolicy check after a step (trainer.cpp:532-554): the history is
        lambda . (l_pde, l_ic, l_bc) per epoch, as the reference records it."""
        l = self.losses.tolist()
        self.loss_history.append(self.lam[0] * l[0] + self.lam[1] * l[1] + self.lam[2] * l[2])
        return policy.should_switch(self.epoch - 1, self.loss_history)

    def params_host(self) -> np.ndarray:
        self.check()
        return self.params.double().cpu().numpy()
