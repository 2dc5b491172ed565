#!/bin/bash
# Driver-style bench lines for every BASELINE config (1 GPU): the headline C5 @ 1M
# (with the CPU reference beside it), C1/C2/C3/C4, the C5 sweep at 8M/16M/64M
# points per GPU, and the reference CPU arm.
mkdir -p gpurun_out/lines
run() { local tag=$1; shift; echo "== $tag: $*"; timeout 900 python bench.py "$@" > gpurun_out/lines/$tag.json 2> gpurun_out/lines/$tag.err; echo "rc=$?"; tail -c 400 gpurun_out/lines/$tag.json; echo; }
run c5_1M
run c1 --config c1
run c2 --config c2 --no-cpu-baseline
run c3 --config c3 --no-cpu-baseline
run c4 --config c4 --no-cpu-baseline
run c5_8M --points-per-gpu 8388608 --no-cpu-baseline --steps 5
run c5_16M --points-per-gpu 16777216 --no-cpu-baseline --steps 4
run c5_64M --points-per-gpu 67108864 --no-cpu-baseline --no-e2e --steps 3
run reference_c5 --impl reference
