#!/bin/bash
# Round-2 evidence call: GPU suite, race stress, per-launch time + DRAM bytes of every step kernel
# (c3, c5), ncu --set full of the dominant kernel and of the epilogue at c3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ev_tests.log
timeout 900 python tools/race_stress.py 50 > gpurun_out/ev_race.log 2>&1; echo "race rc=$?"; tail -2 gpurun_out/ev_race.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for CFG in c3 c5; do
  SMALL="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --no-pruned --no-extras --no-tc --no-bwd-roofline --no-graph"
  $SMALL > gpurun_out/ev_plain_$CFG.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ev_launches_$CFG.csv $SMALL > gpurun_out/ev_ncu_$CFG.log 2>&1
  echo "launches $CFG rc=$?"
done
bash tools/gpu_ncu_full.sh r2fused c3 nn_fused
bash tools/gpu_ncu_full.sh r2epi c3 nn_epilogue
