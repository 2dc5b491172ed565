#!/bin/bash
# A/B of two builds of libpnx on the same box: ab_base/libpnx.so (PNX_LIB_PATH) vs the in-tree one
for lib in ab_base/libpnx.so "" ab_base/libpnx.so ""; do
  PNX_LIB_PATH=$lib python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ablib.json 2>&1
  python - "${lib:-new}" <<'PY'
import json, sys
l = json.loads(open("gpurun_out/ablib.json").read().strip().split("\n")[-1])
print(sys.argv[1], "%.2f ms" % l["ms_per_step"], {k: round(v, 2) for k, v in l["kernel_ms_per_step"].items() if v},
      "clk", l["clocks"]["sm_mhz"])
PY
done
