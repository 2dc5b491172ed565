for n in A B A B; do
  if [ $n = B ]; then export PNX_LIB_PATH=$PWD/build_var/libpnx_B.so; else unset PNX_LIB_PATH; fi
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('$n', round(d['ms_per_step'],2), {a:round(b,2) for a,b in k.items() if b}, d['clocks']['sm_mhz'])"
done
