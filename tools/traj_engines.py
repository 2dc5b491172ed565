"""Loss trajectories of the three engines over 300 device-Adam steps (dev tool)."""
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200.dist import DataParallelTrainer
import test_gpu_parity as T
wl, col, flat, rffB, *_ = T._workload_case("c4", [20, 16, 12])
L = {}
for engine in ("ffma", "auto", "tc3xtf32"):
    w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, engine=engine, **col)
    tr = DataParallelTrainer([w], flat, world=1, lr=1e-3, gamma=1.0, device=torch.device("cuda:0"), has_bc=wl.bc != "hard", graph=True)
    L[engine] = np.array([tr.step().cpu().numpy()[:3] for _ in range(300)])
for e in ("auto", "tc3xtf32"):
    for k, name in ((0, "pde"), (1, "ic")):
        rel = np.abs(L[e][:, k] - L["ffma"][:, k]) / np.abs(L["ffma"][:, k])
        print(e, name, "max rel dev per 50 steps:", ["%.1e" % rel[i:i+50].max() for i in range(0, 300, 50)])
print("ffma loss first/last", L["ffma"][0], L["ffma"][-1])
