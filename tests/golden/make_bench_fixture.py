"""FP64 gradient of the bench workload at full size (test fixture generator).

The headline bench line is C4/C5 at 1,048,576 interior points (Maxwell TE,
tanh 6x256, configs.weak_scaling_dims(2**20, 1) = 128 x 128 x 64, parameters
pk.init_params(seed=0)). This script computes that step's losses and flat
gradient in float64 with the numpy restatement of the reference
(oracle/pinn_oracle.py, pinned to oracle/_ref at 1e-12 by tests/test_oracle.py),
so the GPU parity test can compare the tensor-core path at the bench size
against FP64, not against another FP32 engine.

The full-batch PDE term is assembled from equal-size chunks: with per-chunk
mean losses l_c and gradients g_c over n_c points, the whole-set values are
sum_c (n_c / N) l_c and sum_c (n_c / N) g_c -- the equal-shard identity the
reference states for data_parallel_gradient (trainer.cpp:264-281).
The replicated IC term (trainer.cpp:225-232) is added once. Only oracle code
runs here; nothing of the product path.

    python tests/golden/make_bench_fixture.py [--procs 4]

writes tests/golden/bench_c4_1M_fp64.npz (gradient, losses, and hashes of the
inputs so the test can check it regenerated the same points and parameters).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "bench_c4_1M_fp64.npz")
CHUNK = 8192
DIMS = [128, 128, 64]
SEED = 0


def inputs():
    """The bench's own workload construction (bench.py: workload + init_params)."""
    import paper_2604_15645_b200 as pk
    from paper_2604_15645_b200 import configs
    wl = configs.get_config("c4")
    col = configs.collocation(wl, DIMS)
    flat, rffB = pk.init_params(wl.spec, seed=SEED)
    return wl, col, flat, rffB


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def _oracle_objs(wl, col):
    from oracle import pinn_oracle as po
    spec = po.ModelSpec(wl.spec.in_dim, wl.spec.hidden_dim, wl.spec.depth, wl.spec.out_dim, wl.spec.activation)
    res = po.ResidualSpec(wl.res.id, wl.res.advection_c, wl.res.epsilon, wl.res.mu, wl.res.reynolds)
    ocol = po.Collocation(col["interior"], col["ic_points"], col["ic_targets"], col["bc_a"], col["bc_b"],
                          col["bc_targets"])
    return po, spec, res, ocol


def _chunk(args):
    lo, hi = args
    wl, col, flat, rffB = inputs()
    po, spec, res, ocol = _oracle_objs(wl, col)
    o = po.worker_step(spec, flat, rffB, res, col["interior"][lo:hi], ocol, wl.bc, (1.0, 0.0, 0.0))
    return lo, hi, o["pde"], o["grad"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=4)
    a = ap.parse_args()
    wl, col, flat, rffB = inputs()
    N = len(col["interior"])
    po, spec, res, ocol = _oracle_objs(wl, col)
    # replicated IC term (value stream), computed once on a small interior slice
    icb = po.worker_step(spec, flat, rffB, res, col["interior"][:256], ocol, wl.bc, (0.0, 1.0, 1.0))
    spans = [(lo, min(N, lo + CHUNK)) for lo in range(0, N, CHUNK)]
    g = np.zeros_like(icb["grad"])
    l_pde = 0.0
    t0 = time.time()
    with ProcessPoolExecutor(a.procs) as ex:
        parts = sorted(ex.map(_chunk, spans))
    for lo, hi, lp, gc in parts:  # fixed (row) order
        w = (hi - lo) / N
        g += w * gc
        l_pde += w * lp
    g += icb["grad"]
    np.savez_compressed(OUT, grad=g, losses=np.array([l_pde, icb["ic"], icb["bc"]]), n_interior=N,
                        dims=np.array(DIMS), seed=SEED, params_sha256=digest(flat),
                        interior_sha256=digest(col["interior"]))
    print(f"wrote {OUT}: N={N} l_pde={l_pde:.17g} l_ic={icb['ic']:.17g} |g|={np.linalg.norm(g):.6g} "
          f"({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
