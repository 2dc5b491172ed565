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
# hidden-layer kernels launch 5x per step: skip 2 (a middle layer of step 1);
# once-per-step kernels: skip 1 (step 2)
for k in k_tc4_fwd:2 k_tc5_bwd:2 k_tc2_wgrad:2 k_head:1 k_layer0_wgrad_stream:1 k_layer0_fwd:1; do
    name=${k%%:*}; skip=${k#*:}
    timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$name" -s $skip -c 1 \
        -o gpurun_out/ncu/full_$name -f $CMD > gpurun_out/ncu/full_$name.log 2>&1
done
ls -la gpurun_out/ncu
# text summaries on the box (reports are ~20 MB each; gpurun copies back <= 64 MiB)
for f in gpurun_out/ncu/full_*.ncu-rep; do
    python tools/ncu_summary.py "$f" > "${f%.ncu-rep}.txt" 2>&1
    python tools/ncu_lines.py "$f" 25 > "${f%.ncu-rep}_lines.txt" 2>&1
done
python tools/ncu_launches.py gpurun_out/ncu/launches.csv 2 \
    "# ncu launch list: tools/profile_step.py --config c4 --points 1048576 --steps 2 (C5 workload, 1 GPU, engine ${ENGINE:-auto})" \
    > gpurun_out/ncu/launches_summary.txt 2>&1
[ -n "${KEEP_REPORTS:-}" ] || rm -f gpurun_out/ncu/*.ncu-rep
