"""Data-parallel train step across processes, one per GPU (torch.distributed).

Reference protocol (in-process threads there, processes + NCCL here):
* interior shards: contiguous, last shard takes the remainder   trainer.cpp:143-154
* IC/BC sets replicated on every rank                           trainer.cpp:225-232
* gradient average: rank-ordered sum, then x 1/W                trainer.cpp:264-281
* identical Adam update on every replica                        trainer.cpp:626-638
* replica consistency hash (FNV-1a) after each step             trainer.cpp:22-35, 540-544

The only collective is one all-reduce of the flat gradient per step (the
points are partitioned, not exchanged); the 1/W scale is fused into the device
Adam kernel (pnx_adam_step_device).
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
    t = torch.tensor([h & 0x7FFFFFFFFFFFFFFF, h >> 63], dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(o[0]) | (int(o[1]) << 63) for o in out]


class DataParallelTrainer:
    """Synchronized Adam steps on one GPU per process (trainer.cpp:419-555 with
    balancing off): device step -> NCCL all-reduce -> fused Adam(1/W)."""

    def __init__(self, worker, params0: np.ndarray, world: int = 1, lr: float = 1e-3, gamma: float = 1.0,
                 betas=(0.9, 0.999), eps: float = 1e-8, device=None, group=None):
        import torch
        self.torch = torch
        self.worker, self.world, self.group = worker, world, group
        self.lr, self.gamma, self.betas, self.eps = lr, gamma, betas, eps
        dev = device or torch.device("cuda", worker.device)
        self.params = torch.tensor(np.asarray(params0), dtype=torch.float32, device=dev)
        self.grad = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.losses = torch.zeros(3, dtype=torch.float64, device=dev)
        self.t = 0
        self.epoch = 0

    def step(self, lambdas=(1.0, 1.0, 1.0), stream=None):
        st = stream if stream is not None else self.torch.cuda.current_stream(self.params.device).cuda_stream
        self.worker.step_device(self.params, self.grad, lambdas, self.losses, stream=st)
        allreduce_sum_(self.grad, self.world, self.group)
        self.t += 1
        lr = self.lr * self.gamma ** self.epoch  # ExponentialLr::at (optim.cpp:71-73)
        self.worker.adam_step_device(self.params, self.grad, self.m, self.v, self.t, lr, self.betas[0],
                                     self.betas[1], self.eps, grad_scale=1.0 / self.world, stream=st)
        self.epoch += 1
        return self.losses

    def params_host(self) -> np.ndarray:
        return self.params.double().cpu().numpy()
