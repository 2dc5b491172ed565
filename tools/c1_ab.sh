#!/bin/bash
# C1 single-kernel step A/B (CUDA-graph replays): 16 vs 32 warps per CTA
for v in ${VARIANTS:-"X=1" "PNX_SMALL_NT1024=1" "X=1" "PNX_SMALL_NT1024=1"}; do
  env $v python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/c1ab.json 2>&1
  python - "$v" <<'PY'
import json, sys
l = json.loads(open("gpurun_out/c1ab.json").read().strip().split("\n")[-1])
print(sys.argv[1], "%.4f ms" % l["ms_per_step"], {k: round(v, 4) for k, v in l["kernel_ms_per_step"].items() if v})
PY
done
