#!/bin/bash
# Per-kernel device times of one pruned forward (ncu launch list): tools/time_pruned_kernels.sh <config> [variant...]
CFG=$1; shift
for v in "$@"; do
  CD_LIB_VARIANT=$v python tools/run_forward.py $CFG pruned 1 > /dev/null && \
  CD_LIB_VARIANT=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ptk_$v.csv python tools/run_forward.py $CFG pruned 1 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/ptk_$v.csv gpurun_out/ptk_$v.txt "variant [$v] $CFG" > /dev/null
  echo "== variant [$v]"; awk 'NR>2 {printf "%s %s; ", $2, $3} END {print ""}' gpurun_out/ptk_$v.txt
done
