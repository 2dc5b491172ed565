# accuracy split (which contraction dominates the 1M-point gradient error) + 512-row timing
mkdir -p gpurun_out
timeout 900 python tools/wg_rows_ab.py "auto::3" "auto:512" "auto:" "tc3xtf32:" "tc3xtf32:512" "ffma::"
for wr in "" 512 "" 512; do
  env ${wr:+PNX_WG_ROWS=$wr} timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('[wr=${wr:-default}]', round(d['ms_per_step'],2), {a:round(b,2) for a,b in k.items() if b}, d['clocks']['sm_mhz'])"
done
