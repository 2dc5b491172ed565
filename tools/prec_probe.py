"""Per-contraction precision ablation (dev tool): rel-L2 of the GPU gradient vs
the FP64 oracle with the tcgen05 path enabled per GEMM type (PNX_TC_MASK)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, "%s"); sys.path.insert(0, "%s/tests")
import golden_io as gi
from oracle import pinn_oracle as po
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200 import configs
import test_gpu_parity as T
for cfg, dims in [("c2", [32, 24]), ("c3", [24, 20]), ("c4", [12, 10, 8]), ("c4", [40, 40, 16])]:
    wl, col, flat, rffB, ospec, ores, ocol = T._workload_case(cfg, dims)
    ref, outs = po.data_parallel_gradient(ospec, flat, rffB, ores, ocol, wl.bc, 1)
    g, l = pk.data_parallel_gradient(wl.spec, wl.res, wl.bc, flat, rffB, workers=1, engine=sys.argv[1], **col)
    e = np.abs(g - ref)
    print(cfg, dims, sys.argv[1], "mask", sys.argv[2], "rel_l2 %%.2e  max_rel_elem %%.2e" %% (T.rel_l2(g, ref), (e / (np.abs(ref).max())).max()), flush=True)
''' % (ROOT, ROOT)
for eng, mask in [("ffma", "0"), ("auto", "1"), ("auto", "2"), ("auto", "4"), ("auto", "7"), ("tc3xf16", "1"), ("tc3xf16", "7")]:
    env = dict(os.environ, PNX_TC_MASK=mask)
    subprocess.run([sys.executable, "-c", code, eng, mask], env=env)
