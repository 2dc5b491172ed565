"""The BASELINE.json workloads as concrete specs.

C1 Burgers tanh 4x64, 100x100 grid (the reference's CPU-runnable case)
C2 Burgers + RFF(128, sigma 10) + RWF(1, 0.1), 4x128, 256x256
C3 steady NS lid-driven cavity (Re 100), 5x128, out 3, 512x512 (extension)
C4 Maxwell TE (Ez, Hx, Hy) 6x256, 128x128x64 = 1,048,576 points
C5 C4's model, weak scaling: points_per_gpu x n_gpus
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .pinn import ModelSpec, ResidualSpec, RFFSpec, RWFSpec


@dataclass
class Workload:
    name: str
    spec: ModelSpec
    res: ResidualSpec
    bc: str
    domain: List[Tuple[float, float]]
    dims: List[int]
    initial: str
    n_ic: int = 128
    n_bc: int = 64
    description: str = ""

    @property
    def n_interior(self) -> int:
        return int(np.prod(self.dims))

    def streams(self) -> int:
        return {"advection": 3, "burgers": 3, "allen_cahn": 4, "maxwell_te": 4, "maxwell_te_eh": 4,
                "ns_steady": 5}[self.res.id]

    def sum_in_out(self) -> int:
        s = self.spec
        dims = [s.first_layer_width()] + [s.hidden_dim] * s.depth + [s.out_dim]
        return sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))

    def flops_per_point(self) -> int:
        """Algorithmic F_pt = 3 * 2 * S * sum_l in_l*out_l:
        forward jets + dX + dW contractions; elementwise work excluded."""
        return 6 * self.streams() * self.sum_in_out()


def _initial(name: str, xs: np.ndarray, fields: int) -> np.ndarray:
    if name == "sin_pi_x":
        return np.sin(math.pi * xs[:, :1])
    if name == "gauss25":
        out = np.zeros((xs.shape[0], fields))
        out[:, 0] = np.exp(-25.0 * (xs[:, 0] ** 2 + xs[:, 1] ** 2))
        return out
    if name == "lid":  # NS walls: targets handled by bc traces; IC unused
        return np.zeros((xs.shape[0], fields))
    return np.zeros((xs.shape[0], fields))


def linspace(lo, hi, n):  # sampling.cpp:10-20
    if n == 1:
        return np.array([lo], dtype=np.float64)
    v = lo + np.arange(n, dtype=np.float64) * ((hi - lo) / (n - 1))
    v[-1] = hi
    return v


def grid(bounds, dims) -> np.ndarray:
    """sample_uniform (sampling.cpp:22-54): tensor grid, last axis fastest."""
    axes = [linspace(b[0], b[1], n) for b, n in zip(bounds, dims)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)


def collocation(w: Workload, dims: Optional[List[int]] = None, with_interior: bool = True):
    """build_collocation, uniform mode (trainer.cpp:47-128). Returns dict of
    interior, ic_points, ic_targets, bc_a, bc_b, bc_targets (numpy float64);
    with_interior=False leaves the interior to a device design (pnx_sample_points)."""
    dims = dims or w.dims
    b = w.domain
    F = w.spec.out_dim
    out = {"interior": grid(b, dims) if with_interior else None}
    if w.res.id == "ns_steady":
        # steady: no time axis and no IC; 4-wall Dirichlet with lid u = 1
        n = w.n_bc
        s = linspace(0.0, 1.0, n)
        walls = [np.stack([np.zeros(n), s], 1), np.stack([np.ones(n), s], 1),
                 np.stack([s, np.zeros(n)], 1), np.stack([s, np.ones(n)], 1)]
        pts = np.concatenate(walls)
        tg = np.zeros((4 * n, F))
        tg[3 * n:, 0] = 1.0
        out.update(ic_points=np.zeros((0, 2)), ic_targets=np.zeros((0, F)), bc_a=pts, bc_b=None, bc_targets=tg)
        return out
    d = len(b)
    spatial = d - 1
    if spatial == 1:
        ic = linspace(b[0][0], b[0][1], w.n_ic)[:, None]
    else:
        per = int(math.ceil(w.n_ic ** (1.0 / spatial)))
        ic = grid(b[:-1], [per] * spatial)
    ic = np.concatenate([ic, np.zeros((ic.shape[0], 1))], axis=1)
    out.update(ic_points=ic, ic_targets=_initial(w.initial, ic[:, :spatial], F), bc_a=None, bc_b=None,
               bc_targets=None)
    if w.bc != "hard":
        ts = linspace(b[-1][0], b[-1][1], w.n_bc)

        def trace(xv):
            cols = [np.full(w.n_bc, xv)] + [np.full(w.n_bc, 0.5 * (b[a][0] + b[a][1])) for a in range(1, spatial)]
            return np.stack(cols + [ts], axis=1)

        ta, tb = trace(b[0][0]), trace(b[0][1])
        if w.bc == "dirichlet_zero":
            out["bc_a"] = np.concatenate([ta, tb])
            out["bc_targets"] = np.zeros((2 * w.n_bc, F))
        else:
            out["bc_a"], out["bc_b"] = ta, tb
    return out


CONFIGS = {
    "c1": Workload("c1_burgers_4x64", ModelSpec(2, 64, 4, 1, "tanh"), ResidualSpec("burgers"),
                   "dirichlet_zero", [(0.0, 2.0), (0.0, 1.0)], [100, 100], "sin_pi_x",
                   description="1D inviscid Burgers, tanh MLP 4x64, 10k pts (PAPER.md:742-744)"),
    "c2": Workload("c2_burgers_rff_rwf_4x128",
                   ModelSpec(2, 128, 4, 1, "tanh", rff=RFFSpec(128, 10.0, 0.0), rwf=RWFSpec(1.0, 0.1)),
                   ResidualSpec("burgers"), "dirichlet_zero", [(0.0, 2.0), (0.0, 1.0)], [256, 256], "sin_pi_x",
                   description="Burgers + RFF(128, sigma 10) + RWF, 4x128, 64k pts"),
    "c3": Workload("c3_ns_cavity_5x128", ModelSpec(2, 128, 5, 3, "tanh"), ResidualSpec("ns_steady", reynolds=100.0),
                   "dirichlet_zero", [(0.0, 1.0), (0.0, 1.0)], [512, 512], "lid", n_bc=64,
                   description="2D steady NS lid-driven cavity Re=100, 5x128, 256k pts (extension)"),
    "c4": Workload("c4_maxwell_te_6x256", ModelSpec(3, 256, 6, 3, "tanh"),
                   ResidualSpec("maxwell_te", epsilon=1.0, mu=1.0), "hard",
                   [(-1.0, 1.0), (-1.0, 1.0), (0.0, 1.5)], [128, 128, 64], "gauss25", n_ic=144,
                   description="2D Maxwell TE pulse (PAPER.md:1023-1046), 6x256, 1M pts"),
}


def get_config(name: str) -> Workload:
    return CONFIGS[name]


def weak_scaling_dims(points_per_gpu: int, n_gpus: int) -> List[int]:
    """C5: C4's 128x128 spatial grid with the time axis stretched so the box
    holds points_per_gpu * n_gpus points (weak scaling, fixed work per GPU)."""
    total = points_per_gpu * n_gpus
    nt = max(1, total // (128 * 128))
    return [128, 128, nt]
