#!/bin/bash
# A/B of the weight-gradient drain segment (PNX_WG_SEG): bench ms/step, the
# weight-gradient class time, and the bench-size gradient error vs FP64.
for seg in ${SEGS:-256 512 1024}; do
  PNX_WG_SEG=$seg python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_seg_$seg.json 2>&1
  python - "$seg" <<'PY'
import json, sys
l = json.loads(open(f"gpurun_out/ab_seg_{sys.argv[1]}.json").read().strip().split("\n")[-1])
print("seg", sys.argv[1], "ms/step %.2f" % l["ms_per_step"], {k: round(v, 2) for k, v in l["kernel_ms_per_step"].items()},
      "clk", l["clocks"]["sm_mhz"])
PY
  PNX_WG_SEG=$seg python -m pytest tests/test_gpu_parity.py -q -s -k "bench_scale and auto" 2>&1 | grep "rel-L2"
done
