# A/B of one env setting ($1, e.g. PNX_WG_STREAM=1) against the default, alternating
for v in "" "$1" "" "$1"; do
  env $v timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('[$v]', round(d['ms_per_step'],2), {a:round(b,2) for a,b in k.items() if b}, d['clocks']['sm_mhz'])"
done
