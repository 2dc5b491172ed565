for rep in 1 2; do for lib in ab_base/libpnx.so ""; do
PNX_LIB_PATH=$lib python bench.py --config c1 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/c1ab.json 2>&1
tail -c 100000 gpurun_out/c1ab.json | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('${lib:-new}', round(l['ms_per_step'],4), {k:round(v,4) for k,v in l['kernel_ms_per_step'].items() if v})"
done; done
