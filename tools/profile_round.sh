#!/bin/bash
# ncu evidence for the current kernels (run under gpurun; writes gpurun_out/ncu/).
#   1. launch list of two C5 train steps (per-launch durations, --clock-control none)
#   2. one --set full capture per hot kernel class (launch 3 of each: a middle layer)
set -u
mkdir -p gpurun_out/ncu
CMD="python tools/profile_step.py --config c4 --points 1048576 --steps 2 ${ENGINE:+--engine $ENGINE}"
timeout 300 $CMD > gpurun_out/ncu/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ncu/launches.csv $CMD > gpurun_out/ncu/launches.log 2>&1
for k in k_tc4_fwd k_tc5_bwd k_tc2_wgrad k_head k_layer0_wgrad_stream; do
    timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
        -o gpurun_out/ncu/full_$k -f $CMD > gpurun_out/ncu/full_$k.log 2>&1
done
ls -la gpurun_out/ncu
