#!/bin/bash
# Round-2 ncu evidence (under gpurun, 1 GPU; writes gpurun_out/ncu2/):
#   1. launch list of the bench command itself (C5 @ 1M, 2 timed steps)
#   2. --set full of the hot kernels (a middle layer of step 1)
set -u
mkdir -p gpurun_out/ncu2
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $BENCH > gpurun_out/ncu2/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ncu2/launches_bench.csv $BENCH > gpurun_out/ncu2/launches_bench.log 2>&1
CMD="python tools/profile_step.py --config c4 --points 1048576 --steps 2"
timeout 300 $CMD > gpurun_out/ncu2/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for k in k_tc2_wgrad:2 k_tc5_bwd:2 k_tc4_fwd:2; do
    name=${k%%:*}; skip=${k#*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$name" -s $skip -c 1 \
        -o gpurun_out/ncu2/full_$name -f $CMD > gpurun_out/ncu2/full_$name.log 2>&1
done
for f in gpurun_out/ncu2/full_*.ncu-rep; do
    python tools/ncu_summary.py "$f" > "${f%.ncu-rep}.txt" 2>&1
    python tools/ncu_lines.py "$f" 25 > "${f%.ncu-rep}_lines.txt" 2>&1
done
python tools/ncu_launches.py gpurun_out/ncu2/launches_bench.csv 6 \
    "# ncu launch list of: $BENCH (C5 @ 1,048,576 points, 1 GPU, engine auto; CUDA-graph mode: 1 warm-up + 1 eager + 2 eager per-class profiling + 2 timed graph replays = 6 steps; ncu profiles graph nodes as launches)" \
    > gpurun_out/ncu2/launches_bench_summary.txt 2>&1
[ -n "${KEEP_REPORTS:-}" ] || rm -f gpurun_out/ncu2/*.ncu-rep
ls -la gpurun_out/ncu2
