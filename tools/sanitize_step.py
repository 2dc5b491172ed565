"""One worker step per engine path, small sizes, for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per run): C1 on the single-kernel narrow path
(auto) and the multi-kernel FFMA path, and the C4 model (6x256) on the tcgen05
3xFP16 kernels (auto), plus a device Adam step and a device LHS design."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200 import configs

for cfg, dims, engines in (("c1", [24, 20], ("auto", "ffma")), ("c4", [12, 10, 8], ("auto",))):
    wl = configs.get_config(cfg)
    col = configs.collocation(wl, dims)
    flat, rffB = pk.init_params(wl.spec, seed=1)
    for eng in engines:
        w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, engine=eng, **col)
        g, l = w.step(flat)
        print(cfg, eng, "grad norm", float(np.linalg.norm(g)), l, "launches", w.launch_count(), flush=True)
    w.sample_points("lhs", wl.domain, n=777, seed=3)
    g, l = w.step(flat)
    print(cfg, "device LHS design", float(np.linalg.norm(g)), flush=True)
print("sanitize_step done")
