"""Dev tool: weight-gradient rows per CTA (PNX_WG_ROWS) -- gradient deviation
from the FFMA engine at the C5 model and ~1M points (a long FP32 accumulation
in TMEM is the accuracy risk of longer tiles). Run under gpurun."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, "%s")
import paper_2604_15645_b200 as pk
from paper_2604_15645_b200 import configs
wl = configs.get_config("c4")
col = configs.collocation(wl, [102, 102, 100])
flat, rffB = pk.init_params(wl.spec, seed=1)
g, l = pk.data_parallel_gradient(wl.spec, wl.res, wl.bc, flat, rffB, workers=1, engine=sys.argv[1], **col)
np.save(sys.argv[2], g)
''' % ROOT
os.makedirs("gpurun_out/wg", exist_ok=True)
# tokens: "wr" or "engine:wr[:tc_mask]"
runs = [("ffma", "", "")]
for a in sys.argv[1:]:
    p = a.split(":") if ":" in a else ["auto", a]
    runs.append((p[0], p[1], p[2] if len(p) > 2 else ""))
import numpy as np
ref = None
for eng, wr, mask in runs:
    env = dict(os.environ)
    if wr:
        env["PNX_WG_ROWS"] = wr
    if mask:
        env["PNX_TC_MASK"] = mask
    out = f"gpurun_out/wg/g_{eng}_{wr or 'default'}_{mask}.npy"
    subprocess.run([sys.executable, "-c", code, eng, out], env=env, check=True)
    g = np.load(out)
    if ref is None:
        ref = g
        continue
    print(f"engine={eng} wg_rows={wr or 'default'} tc_mask={mask or 'all'} rel_l2_vs_ffma={np.linalg.norm(g - ref) / np.linalg.norm(ref):.3e}", flush=True)
