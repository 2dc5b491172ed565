#!/bin/bash
# same-box A/B of ab_base/libpnx.so vs the in-tree build on one config ($1, default c3)
cfg=${1:-c3}
for rep in 1 2; do for lib in ab_base/libpnx.so ""; do
PNX_LIB_PATH=$lib python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/abcfg.json 2>&1
tail -c 100000 gpurun_out/abcfg.json | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('${lib:-new}', '$cfg', round(l['ms_per_step'],4), {k:round(v,4) for k,v in l['kernel_ms_per_step'].items() if v})"
done; done
