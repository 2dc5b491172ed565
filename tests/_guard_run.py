"""Workloads for test_gpu_guard.py (run in a subprocess with PNX_GUARD set): every
kernel family steps once and pnx_check verifies the buffer guards."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import golden_io as gi  # noqa: E402
import paper_2604_15645_b200 as pk  # noqa: E402
from paper_2604_15645_b200 import configs  # noqa: E402


def golden(name, engine):
    g = gi.load(name)
    c = g["case"]
    p = c["pde"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    col = g["col"]
    kw = {}
    if g["causality"] is not None:
        o = g["causality"]
        kw["causality"] = pk.CausalityConfig(o.segments, o.epsilon, o.t_lo, o.t_hi)
    if g["poynting"] is not None:
        o = g["poynting"]
        kw["poynting"] = pk.PoyntingConfig(o.weight, o.grid, o.time_samples, tuple(o.xb) + tuple(o.yb) + tuple(o.tb))
    w = pk.make_worker(spec, res, g["bc"], g["rffB"], col.interior, col.ic_points, col.ic_targets, col.bc_a, col.bc_b,
                       col.bc_targets, engine=engine, **kw)
    w.step(g["params"])
    w.step_terms(g["params"])
    w.check()


names = [n for n in gi.CASE_NAMES]
for n in names:
    for eng in ("auto", "ffma"):
        golden(n, eng)
for cfg, dims in (("c1", [40, 30]), ("c2", [32, 24]), ("c3", [24, 20]), ("c4", [12, 10, 8])):
    wl = configs.get_config(cfg)
    col = configs.collocation(wl, dims)
    flat, rffB = pk.init_params(wl.spec, seed=1)
    for eng in ("auto", "tc3xtf32", "ffma"):
        w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, engine=eng, **col)
        w.step(flat)
        w.set_chunk_rows(512)
        w.step(flat)
        w.check()
# device designs and chunked rows at a larger size
wl = configs.get_config("c4")
col = configs.collocation(wl, [10, 10, 6], with_interior=False)
flat, rffB = pk.init_params(wl.spec, seed=2)
w = pk.Worker(wl.spec, wl.res, wl.bc, rffB)
w.sample_points("lhs", wl.domain, n=70000, seed=3)
w.set_ic(col["ic_points"], col["ic_targets"])
w.step(flat)
w.set_chunk_rows(16384)
w.step(flat)
w.check()
print("guards ok")
