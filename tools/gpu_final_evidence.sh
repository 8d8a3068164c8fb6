#!/bin/bash
# End-of-round evidence at HEAD: GPU suite, randomised cross-checks, race reruns, bench lines for every
# config (+ the two-rank gloo runs and the reference arm), per-launch lists of one c3 / c5 step, and
# ncu --set full of the kernels changed this round.  usage: tools/gpu_final_evidence.sh <tag>
TAG=${1:-fin}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 900 python tools/stress.py 1000 31 > gpurun_out/${TAG}_stress.log 2>&1; echo "stress rc=$?"; tail -1 gpurun_out/${TAG}_stress.log
timeout 600 python tools/stress_p2s.py 300 37 > gpurun_out/${TAG}_stress_p2s.log 2>&1; echo "stress_p2s rc=$?"; tail -1 gpurun_out/${TAG}_stress_p2s.log
timeout 900 python tools/race_stress.py 50 > gpurun_out/${TAG}_race.log 2>&1; echo "race rc=$?"; tail -1 gpurun_out/${TAG}_race.log
CFGS="c1 c2 c3 c4 c5" bash tools/gpu_allcfg.sh $TAG
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for CFG in c3 c5; do
  SMALL="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --no-pruned --no-extras --no-tc --no-bwd-roofline --no-graph"
  $SMALL > gpurun_out/${TAG}_plain_$CFG.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$CFG.csv $SMALL > gpurun_out/${TAG}_ncu_$CFG.log 2>&1
  echo "launches $CFG rc=$?"
done
bash tools/gpu_ncu_full.sh ${TAG}_fused c3 nn_fused
bash tools/gpu_ncu_kernel.sh ${TAG}_segg seg_sort_grad_kernel 1 tools/run_backward.py c3 2
bash tools/gpu_ncu_kernel.sh ${TAG}_pruned nn_pruned 1 tools/run_forward.py c4 pruned 2
