#!/bin/bash
# C1 single-kernel step A/B: bench eager + graph, with and without the fused finalize
for v in ""; do
  for g in "" "--graph"; do
    env $v python bench.py --config c1 --no-cpu-baseline --no-e2e $g > gpurun_out/c1ab.json 2>&1
    python - "$v" "$g" <<'PY'
import json, sys
l = json.loads(open("gpurun_out/c1ab.json").read().strip().split("\n")[-1])
print(sys.argv[1] or "fused", sys.argv[2] or "eager", "%.4f ms" % l["ms_per_step"], {k: round(v, 4) for k, v in l["kernel_ms_per_step"].items() if v})
PY
  done
done
