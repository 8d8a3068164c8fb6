#!/bin/bash
# ncu launch list only. usage: tools/gpu_launches.sh <tag> [config]
TAG=${1:-x}; CFG=${2:-c3}
mkdir -p gpurun_out
SMALL="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --no-pruned --no-extras --no-tc --no-bwd-roofline"
$SMALL > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $SMALL > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?"
