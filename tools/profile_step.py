"""Run a few worker steps of a config (for ncu captures). Dev tool."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200 import configs
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--points", type=int, default=262144)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--engine", default="auto")
a = ap.parse_args()
wl = configs.get_config(a.config)
dims = configs.weak_scaling_dims(a.points, 1) if a.config == "c4" else wl.dims
col = configs.collocation(wl, dims)
flat, rffB = pk.init_params(wl.spec, 0)
w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, engine=a.engine, **col)
p = torch.tensor(flat, dtype=torch.float32, device="cuda")
g = torch.zeros_like(p)
st = torch.cuda.current_stream().cuda_stream
for _ in range(a.steps):
    w.step_device(p, g, stream=st)
torch.cuda.synchronize()
w.check()
print("ok", len(col["interior"]), w.launch_count())
