#!/bin/bash
# One gpurun call: bench line, ncu launch list, ncu --set full of the top kernel.
# usage: tools/gpu_bench_profile.sh <tag> [config]
set -u
TAG=${1:-r01}; CFG=${2:-c3}
mkdir -p gpurun_out
python bench.py --config $CFG > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
SMALL="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --no-pruned --no-extras"
$SMALL > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $SMALL > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
$SMALL > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${3:-nn_fused} -s 1 -c 1 -o gpurun_out/prof_$TAG $SMALL > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
