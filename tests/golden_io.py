"""Load tests/golden fixtures into oracle objects (test helper)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import pinn_oracle as po  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def spec_from_json(j: dict) -> po.ModelSpec:
    s = po.ModelSpec(in_dim=j["in_dim"], hidden_dim=j["hidden_dim"], depth=j["depth"],
                     out_dim=j["out_dim"], activation=j["activation"], sine_w0=j.get("sine_w0", 1.0))
    for a in j.get("periodic_axes", []):
        s.periodic_axes.append(po.AxisPeriodic(a["periodic"], a["period"], a.get("trainable", False)))
    if "rff" in j:
        s.rff = po.RFFSpec(j["rff"]["width"], j["rff"].get("sigma", 10.0), j["rff"].get("mean", 0.0))
    if "rwf" in j:
        s.rwf = po.RWFSpec(j["rwf"].get("mean", 1.0), j["rwf"].get("stddev", 0.1))
    return s


def res_from_json(j: dict) -> po.ResidualSpec:
    return po.ResidualSpec(id=j["id"], advection_c=j.get("advection_c", 1.0),
                           epsilon=j.get("epsilon", 1.0), mu=j.get("mu", 1.0))


def load(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(z["meta"]))
    case = meta["case"]
    spec = spec_from_json(case["model"])
    res = res_from_json(case["pde"])
    bc = case.get("bc", "hard")
    col = po.Collocation(z["interior"], z["ic_points"], z["ic_targets"])
    if bc == "dirichlet_zero":
        col.bc_a = z["bc_a"]
        col.bc_targets = np.zeros((z["bc_a"].shape[0], spec.out_dim))
    elif bc == "soft_periodic":
        col.bc_a, col.bc_b = z["bc_a"], z["bc_b"]
    rffB = z["rffB"] if spec.rff else None
    dom = case["domain"]
    causality = poynting = balancing = None
    if case.get("causality", {}).get("enabled", False):
        causality = po.Causality(case["causality"].get("segments", 10), case["causality"].get("epsilon", 1.0),
                                 dom[-1][0], dom[-1][1])
    if case.get("poynting", {}).get("weight", 0.0) > 0.0:
        pj = case["poynting"]
        poynting = po.Poynting(pj["weight"], pj.get("grid", 32), pj.get("time_samples", 4),
                               tuple(dom[0]), tuple(dom[1]), tuple(dom[-1]))
    t = case.get("train", {})
    if t.get("balancing", False):
        balancing = po.Balancing(True, t.get("alpha", 0.9), t.get("update_period", 100))
    switch = lbfgs_cfg = None
    if "switch" in t:
        sw = t["switch"]
        switch = po.SwitchPolicy(sw.get("trigger", "none"), sw.get("epoch_threshold", 0), sw.get("plateau_window", 0),
                                 sw.get("plateau_rel_improvement", 0.0))
        lbfgs_cfg = po.LbfgsConfig(**t.get("lbfgs", {}))
    out = {"meta": meta, "case": case, "spec": spec, "res": res, "bc": bc, "col": col,
           "params": z["params"], "rffB": rffB, "causality": causality, "poynting": poynting,
           "balancing": balancing, "switch": switch, "lbfgs_cfg": lbfgs_cfg,
           "lbfgs_max_iters": t.get("lbfgs_max_iters", 0)}
    for k in z.files:
        if k not in out:
            out[k] = z[k]
    return out


CASE_NAMES = sorted(n[:-4] for n in os.listdir(GOLDEN)
                    if n.endswith(".npz") and not n.startswith(("traj_", "ckpt_", "bench_")))
CKPT_NAMES = sorted(n[:-4] for n in os.listdir(GOLDEN) if n.startswith("ckpt_") and n.endswith(".npz"))
TRAJ_NAMES = sorted(n[:-4] for n in os.listdir(GOLDEN) if n.startswith("traj_") and n.endswith(".npz"))
