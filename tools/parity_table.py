"""Gradient rel-L2 of the default engine per BASELINE config (dev tool; the
numbers in BASELINE.md §5). C1/C2/C4: reference goldens at the config's model
(oracle/_ref, tests/golden); C3: the NS extension vs the FP64 numpy oracle (no
reference code exists for it); C5: the bench step itself vs its FP64 fixture."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import golden_io as gi
import paper_2604_15645_b200 as pk
from oracle import pinn_oracle as po
import test_gpu_parity as tp


def golden(name):
    g = gi.load(name)
    c = g["case"]
    p = c["pde"]
    spec = pk.ModelSpec.from_json(c["model"])
    res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
    col = g["col"]
    gr, _ = pk.data_parallel_gradient(spec, res, g["bc"], g["params"], g["rffB"], col.interior, col.ic_points,
                                      col.ic_targets, col.bc_a, col.bc_b, col.bc_targets, workers=1)
    return tp.rel_l2(gr, g["grad_w1"]), len(col.interior)


rows = []
for cfg, name in (("C1", "burgers_c1_full"), ("C2", "burgers_c2_shape"), ("C4", "maxwell_c4_shape")):
    e, n = golden(name)
    rows.append((cfg, f"reference golden {name} ({n} pts)", e))
wl, col, flat, rffB, ospec, ores, ocol = tp._workload_case("c3", [24, 20])
ref, _ = po.data_parallel_gradient(ospec, flat, rffB, ores, ocol, wl.bc, 1)
g, _ = pk.data_parallel_gradient(wl.spec, wl.res, wl.bc, flat, rffB, workers=1, **col)
rows.append(("C3", "FP64 numpy oracle (NS extension, 480 pts)", tp.rel_l2(g, ref)))
wl, col, flat, rffB, z = tp._bench_fixture()
w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, **col)
g, _ = w.step(flat)
rows.append(("C4/C5", "FP64 fixture of the bench step (1,048,576 pts)", tp.rel_l2(g, z["grad"])))
for r in rows:
    print(f"{r[0]:6s} {r[2]:.2e}  {r[1]}")
