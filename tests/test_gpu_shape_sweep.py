"""GPU: a deterministic sweep of model shapes and objective options against the
FP64 oracle (pinned to the compiled reference, test_oracle.py).

The goldens fix a handful of shapes; this sweep varies what selects kernel
paths -- width (multiples of 32 or not: tensor-core, single-kernel and FFMA
paths), depth, activation, RFF / RWF / periodic embeddings (trainable period),
PDE, boundary mode, ragged point counts (partial 128/256-row tiles), several
workers -- and holds every case to the parity bar of test_gpu_parity.py:
gradient rel-L2 and SURVEY 8(c)'s elementwise bound at 1e-5, losses at 1e-5.
"""
import numpy as np
import pytest

import golden_io as gi
from oracle import pinn_oracle as po

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-5
LOSS_RTOL = 1e-5

PDES = ["burgers", "advection", "allen_cahn", "maxwell_te", "maxwell_te_eh"]
WIDTHS = [8, 20, 32, 48, 64, 96, 128, 160, 256]
ACTS = ["tanh", "tanh", "sine", "swish"]


def _cases(n=96, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        pde = PDES[i % len(PDES)]
        c = {
            "pde": pde,
            "width": int(rng.choice(WIDTHS)),
            "depth": int(rng.integers(1, 4)),
            "act": str(rng.choice(ACTS)),
            "rff": int(rng.choice([0, 0, 8, 16])),
            "rwf": bool(rng.random() < 0.3),
            "periodic": bool(pde not in ("maxwell_te", "maxwell_te_eh") and rng.random() < 0.3),
            "trainable": bool(rng.random() < 0.5),
            "bc": str(rng.choice(["hard", "dirichlet_zero", "soft_periodic"])),
            "n": int(rng.choice([1, 7, 31, 129, 255, 257]) if rng.random() < 0.25 else rng.integers(90, 1500)),
            "workers": int(rng.choice([1, 1, 2, 3])),
            "engine": str(rng.choice(["auto", "auto", "ffma"])),
            "seed": int(rng.integers(0, 1 << 30)),
        }
        c["workers"] = min(c["workers"], c["n"])
        if c["periodic"]:
            c["rff"] = 0  # the reference applies RFF to the raw coordinates or the embedding; keep one
        out.append(c)
    return out


def _fixed():
    """Hand-picked cases for the tensor-core paths (tanh at width 128 / 256)."""
    base = dict(rff=0, rwf=False, periodic=False, trainable=False, workers=1, engine="auto")
    out = [
        dict(base, pde="maxwell_te", width=256, depth=2, act="tanh", bc="hard", n=700, seed=11),      # pair fwd, tc5 MX bwd
        dict(base, pde="burgers", width=256, depth=3, act="tanh", bc="dirichlet_zero", n=600, seed=12),  # tc5 XT bwd
        dict(base, pde="allen_cahn", width=256, depth=2, act="tanh", bc="soft_periodic", n=520, seed=13),  # S=4 second order
        dict(base, pde="maxwell_te_eh", width=256, depth=2, act="tanh", bc="dirichlet_zero", n=333, seed=14, workers=2),
        dict(base, pde="burgers", width=128, depth=3, act="tanh", bc="hard", n=777, seed=15, rff=64, rwf=True),  # C2-like
        dict(base, pde="allen_cahn", width=128, depth=2, act="tanh", bc="dirichlet_zero", n=450, seed=16, workers=3),
        dict(base, pde="maxwell_te", width=128, depth=3, act="tanh", bc="soft_periodic", n=390, seed=17, engine="tc3xtf32"),
        dict(base, pde="advection", width=256, depth=1, act="tanh", bc="hard", n=257, seed=18, periodic=True,
             trainable=True),
        dict(base, pde="maxwell_te", width=512, depth=2, act="tanh", bc="hard", n=300, seed=19),  # beyond the tc widths
        dict(base, pde="burgers", width=384, depth=1, act="sine", bc="dirichlet_zero", n=200, seed=20),
        dict(base, pde="allen_cahn", width=1, depth=1, act="tanh", bc="hard", n=50, seed=21),
        dict(base, pde="burgers", width=64, depth=6, act="tanh", bc="soft_periodic", n=513, seed=22),  # deep narrow
    ]
    return out


CASES = _cases() + _fixed()


def _build(c):
    import paper_2604_15645_b200 as pk
    rng = np.random.default_rng(c["seed"])
    pde = c["pde"]
    res = pk.ResidualSpec(pde, advection_c=0.7, epsilon=1.3, mu=0.8)
    d = res.coord_count()
    F = res.field_count()
    spec = pk.ModelSpec(in_dim=d, hidden_dim=c["width"], depth=c["depth"], out_dim=F, activation=c["act"],
                        sine_w0=1.5 if c["act"] == "sine" else 1.0)
    if c["periodic"]:
        spec.periodic_axes = [pk.pinn.AxisPeriodic(True, 2.0, c["trainable"]), pk.pinn.AxisPeriodic(False, 0.0)]
    if c["rff"]:
        spec.rff = pk.RFFSpec(c["rff"], 1.0, 0.0)
    if c["rwf"]:
        spec.rwf = pk.RWFSpec(1.0, 0.1)
    flat, rffB = pk.init_params(spec, seed=c["seed"] % 1000)
    lo = np.array([-1.0] * (d - 1) + [0.0])
    hi = np.array([1.0] * (d - 1) + [1.0])
    interior = lo + (hi - lo) * rng.random((c["n"], d))
    n_ic = 24
    ic = np.concatenate([lo[:-1] + (hi[:-1] - lo[:-1]) * rng.random((n_ic, d - 1)), np.zeros((n_ic, 1))], axis=1)
    ic_t = rng.normal(0.0, 0.5, size=(n_ic, F))
    bc_a = bc_b = bc_t = None
    ts = rng.random(16)
    if c["bc"] == "dirichlet_zero":
        side = lambda x: np.stack([np.full(16, x)] + [np.zeros(16)] * (d - 2) + [ts], axis=1)  # noqa: E731
        bc_a = np.concatenate([side(-1.0), side(1.0)])
        bc_t = np.zeros((32, F))
    elif c["bc"] == "soft_periodic":
        side = lambda x: np.stack([np.full(16, x)] + [np.zeros(16)] * (d - 2) + [ts], axis=1)  # noqa: E731
        bc_a, bc_b = side(-1.0), side(1.0)
    return pk, spec, res, flat, rffB, dict(interior=interior, ic_points=ic, ic_targets=ic_t, bc_a=bc_a, bc_b=bc_b,
                                           bc_targets=bc_t)


def _oracle(spec, res, flat, rffB, col, bc, workers):
    import test_gpu_parity as tp
    ospec = gi.spec_from_json(tp._spec_json(spec))
    ores = po.ResidualSpec(res.id, res.advection_c, res.epsilon, res.mu)
    ocol = po.Collocation(col["interior"], col["ic_points"], col["ic_targets"], col["bc_a"], col["bc_b"],
                          col["bc_targets"])
    return po.data_parallel_gradient(ospec, flat, rffB, ores, ocol, bc, workers)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "{pde}-w{width}d{depth}-{act}-rff{rff}{r}{p}-{bc}-n{n}W{workers}-{engine}"
                         .format(r="-rwf" if c["rwf"] else "", p="-per" if c["periodic"] else "", **c))
def test_shape_sweep_vs_oracle(case):
    pk, spec, res, flat, rffB, col = _build(case)
    bc = case["bc"]
    ref, outs = _oracle(spec, res, flat, rffB, col, bc, case["workers"])
    grad, losses = pk.data_parallel_gradient(spec, res, bc, flat, rffB, workers=case["workers"],
                                             engine=case["engine"], **col)
    tol = 2e-5 if case["engine"] == "tc3xtf32" else GRAD_RTOL  # the opt-in engine's stated bound
    err = float(np.linalg.norm(grad - ref) / max(np.linalg.norm(ref), 1e-300))
    assert err <= tol, err
    bound = tol * np.max(np.abs(ref)) + tol * np.abs(ref)
    assert np.all(np.abs(grad - ref) <= bound + 1e-300), float(np.max(np.abs(grad - ref) / (bound + 1e-300)))
    for o, r in zip(losses, outs):
        for k in ("pde", "ic", "bc"):
            assert abs(o[k] - r[k]) <= LOSS_RTOL * abs(r[k]) + 1e-12, (k, o[k], r[k])
