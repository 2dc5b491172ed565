"""Per-tensor comparison of the single-kernel narrow step (engine auto) with the
multi-kernel FFMA path and the FP64 oracle, on a golden case (dev tool)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import golden_io as gi
import paper_2604_15645_b200 as pk
from oracle import pinn_oracle as po
name = sys.argv[1] if len(sys.argv) > 1 else "traj_maxwell"
g = gi.load(name)
c = g["case"]
spec = pk.ModelSpec.from_json(c["model"])
p = c["pde"]
res = pk.ResidualSpec(p["id"], p.get("advection_c", 1.0), p.get("epsilon", 1.0), p.get("mu", 1.0))
col = g["col"]
W = c.get("workers", 1) if isinstance(c.get("workers", 1), int) else 1
outs = {}
for eng in ("auto", "ffma"):
    gr, l = pk.data_parallel_gradient(spec, res, g["bc"], g["params"], g["rffB"], col.interior, col.ic_points,
                                      col.ic_targets, col.bc_a, col.bc_b, col.bc_targets, workers=W, engine=eng)
    outs[eng] = (gr, l)
ref, ro = po.data_parallel_gradient(g["spec"], g["params"], g["rffB"], g["res"], col, g["bc"], W)
at = 0
for nm, shape in pk.param_layout(spec):
    n = int(np.prod(shape)) if shape else 1
    r = ref[at:at + n]
    a = outs["auto"][0][at:at + n]
    f = outs["ffma"][0][at:at + n]
    sc = np.max(np.abs(r)) + 1e-30
    print(f"{nm:12s} |ref|max {sc:.3e}  auto err {np.max(np.abs(a - r)) / sc:.2e}  ffma err {np.max(np.abs(f - r)) / sc:.2e}"
          f"  auto-vs-ffma {np.max(np.abs(a - f)) / sc:.2e}")
    at += n
print("losses auto", outs["auto"][1], "ffma", outs["ffma"][1], "ref", [(o["pde"], o["ic"], o["bc"]) for o in ro])
for eng in ("auto", "ffma"):
    gr = outs[eng][0]
    flip = np.nonzero(np.sign(gr) != np.sign(ref))[0]
    print(eng, "sign flips:", len(flip), [(int(i), float(ref[i]), float(gr[i])) for i in flip[:8]])
# trajectory: losses per epoch vs the fixture, both engines
if "metrics" in g:
    import torch
    from paper_2604_15645_b200.dist import DataParallelTrainer
    t = c["train"]
    for eng in ("auto", "ffma"):
        ws = []
        for lo, hi in pk.shard_interior(len(col.interior), c["workers"]):
            ws.append(pk.make_worker(spec, res, g["bc"], g["rffB"], col.interior[lo:hi], col.ic_points, col.ic_targets,
                                     col.bc_a, col.bc_b, col.bc_targets, engine=eng))
        tr = DataParallelTrainer(ws, g["params"], world=1, lr=t["lr"], gamma=t["gamma"], device=torch.device("cuda:0"),
                                 has_bc=g["bc"] != "hard")
        errs = []
        for ep in range(t["epochs"]):
            l = tr.step().cpu().numpy()
            errs.append(np.max(np.abs(l[:2] - g["metrics"][ep, 1:3]) / np.abs(g["metrics"][ep, 1:3])))
        print(eng, "traj rel err per epoch:", " ".join(f"{e:.1e}" for e in errs))
