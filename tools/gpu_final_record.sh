#!/bin/bash
# End-of-round record: tools/gpu_round_record.sh + the backward launch lists with DRAM bytes (c3, c5)
# and ncu --set full of the backward's top kernels.  usage: tools/gpu_final_record.sh <tag>
TAG=${1:-fin}
mkdir -p gpurun_out
tools/gpu_round_record.sh $TAG
for c in c3 c5; do
  python tools/run_backward.py $c 1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/bwd_${TAG}_$c.csv python tools/run_backward.py $c 1 > /dev/null 2>&1; echo "bwd $c rc=$?"
done
tools/gpu_ncu_kernel.sh ${TAG}_seg seg_sort 0 tools/run_backward.py c3 1
tools/gpu_ncu_kernel.sh ${TAG}_bgr grad_kernel 0 tools/run_backward.py c5 1
tools/gpu_ncu_kernel.sh ${TAG}_bsc radix_scatter 1 tools/run_backward.py c5 1
tools/gpu_ncu_kernel.sh ${TAG}_tie ps_tie 0 tools/run_p2s.py pruned
