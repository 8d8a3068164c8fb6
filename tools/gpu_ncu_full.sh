#!/bin/bash
# ncu --set full of one kernel (after a plain run of the same command exits 0).
# usage: tools/gpu_ncu_full.sh <tag> <config> <kernel-regex>
TAG=${1:-x}; CFG=${2:-c3}; K=${3:-nn_fused}
mkdir -p gpurun_out
SMALL="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --no-pruned --no-extras --no-tc --no-bwd-roofline"
$SMALL > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$TAG $SMALL > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
