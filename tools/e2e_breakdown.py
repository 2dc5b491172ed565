"""Where the end-to-end C5 step spends its host time (dev tool): set_points
(host -> device copy of the 1M-point batch), pnx_step (params H2D, device step,
gradient D2H, FP64 conversions) and the C++ host Adam, each timed by wall clock
around the call, median of N steps."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200 import configs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
wl = configs.get_config("c4" if cfg == "c5" else cfg)
dims = configs.weak_scaling_dims(1 << 20, 1) if cfg == "c5" else wl.dims
col = configs.collocation(wl, dims)
flat, rffB = pk.init_params(wl.spec, seed=0)
w = pk.make_worker(wl.spec, wl.res, wl.bc, rffB, **col)
P = w.n_params
pinned = torch.from_numpy(np.ascontiguousarray(col["interior"].T)).pin_memory()
pts = pinned.numpy()
hl = ctypes.CDLL(os.path.join(ROOT, "host", "libpinnlab_b200.so"))
dp = ctypes.POINTER(ctypes.c_double)
hl.pinnlab_adam_step.argtypes = [dp, dp, dp, dp, ctypes.c_int64] + [ctypes.c_double] * 4 + [ctypes.c_int64]
m = np.zeros(P)
v = np.zeros(P)
p = flat.copy()
rows = []
for k in range(1, N + 4):
    t0 = time.perf_counter()
    w.set_points(pts, axis_major=True)
    t1 = time.perf_counter()
    g, l = w.step(p)
    t2 = time.perf_counter()
    g = np.ascontiguousarray(g)
    hl.pinnlab_adam_step(p.ctypes.data_as(dp), m.ctypes.data_as(dp), v.ctypes.data_as(dp), g.ctypes.data_as(dp), P,
                         1e-3, 0.9, 0.999, 1e-8, k)
    t3 = time.perf_counter()
    if k > 3:
        rows.append((t1 - t0, t2 - t1, t3 - t2, t3 - t0))
r = np.median(np.array(rows), axis=0) * 1e3
print(f"set_points {r[0]:.3f} ms  step {r[1]:.3f} ms  host_adam {r[2]:.3f} ms  total {r[3]:.3f} ms  (P={P})")

# the same step with device-resident params (eager launches, wall clock with syncs)
from paper_2604_15645_b200.dist import DataParallelTrainer
dev = torch.device("cuda", 0)
tr = DataParallelTrainer(w, flat, world=1, lr=1e-3, device=dev, graph=False)
st = torch.cuda.current_stream(dev).cuda_stream
ts = []
for k in range(N + 3):
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    tr.step((1.0, 1.0, 1.0), stream=st, eager=True)
    torch.cuda.synchronize(dev)
    if k >= 3:
        ts.append(time.perf_counter() - t0)
print(f"device-resident step (eager, + device Adam) {np.median(ts) * 1e3:.3f} ms")
