#!/bin/bash
# ncu --set full of one kernel of an arbitrary python command (plain run first, same command).
# usage: tools/gpu_ncu_kernel.sh <tag> <kernel-regex> <skip> <python args...>
TAG=$1; K=$2; S=$3; shift 3
mkdir -p gpurun_out
python "$@" > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/prof_$TAG python "$@" > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
