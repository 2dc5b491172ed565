#!/bin/bash
# A/B: persistent backward (default) vs one tile per CTA (PNX_TC5_ONESHOT=1), same box
for v in ${VARIANTS:-"" "PNX_TC5_ONESHOT=1" "" "PNX_TC5_ONESHOT=1"}; do
  env $v python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/abp.json 2>&1
  python - "$v" <<'PY'
import json, sys
l = json.loads(open("gpurun_out/abp.json").read().strip().split("\n")[-1])
print(sys.argv[1] or "persistent", "%.2f ms" % l["ms_per_step"], {k: round(v, 2) for k, v in l["kernel_ms_per_step"].items() if v},
      "clk", l["clocks"]["sm_mhz"])
PY
done
