# A/B of the weight-gradient rows per CTA (run under gpurun): step time and accuracy
mkdir -p gpurun_out
for wr in "" 2048 3552 7096 "" 2048 3552 7096; do
  env ${wr:+PNX_WG_ROWS=$wr} timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('[wr=${wr:-default}]', round(d['ms_per_step'],2), {a:round(b,2) for a,b in k.items() if b}, d['clocks']['sm_mhz'])"
done
timeout 600 python tools/wg_rows_ab.py "" 2048 3552 7096 14192
