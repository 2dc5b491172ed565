"""Largest elementwise gradient error relative to SURVEY 8(c)'s bound |d_i| <= 1e-5 max|g| + 1e-5 |g_i|
for every golden (ffma, auto) and the bench-size FP64 fixture (dev tool)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import golden_io as gi
import paper_2604_15645_b200 as pk
import test_gpu_parity as tp
def ratio(g, r):
    return float(np.max(np.abs(g - r) / (1e-5 * np.max(np.abs(r)) + 1e-5 * np.abs(r))))
worst = 0
for name in gi.CASE_NAMES:
    g = gi.load(name); case = g["case"]; caus, poy = tp._objective(g)
    for eng in ("ffma", "auto"):
        for w in g["meta"]["workers"]:
            grad, _ = pk.data_parallel_gradient(tp._spec(case), tp._res(case), g["bc"], g["params"], g["rffB"], workers=w,
                                                engine=eng, causality=caus, poynting=poy, **tp._col_args(g))
            q = ratio(grad, g[f"grad_w{w}"]); worst = max(worst, q)
            if q > 0.3: print(name, eng, w, f"{q:.3f}")
wl, col, flat, rffB, z = tp._bench_fixture()
for eng in ("auto", "tc3xtf32", "ffma"):
    w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, engine=eng, **col)
    g, _ = w.step(flat)
    print("bench", eng, f"{ratio(g, z['grad']):.3f}", f"rel-L2 {tp.rel_l2(g, z['grad']):.2e}")
print("worst golden ratio", worst)
