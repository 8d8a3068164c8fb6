#!/bin/bash
# Round record: bench lines for every config, the c3 launch list, ncu --set full of the three hot
# kernels (nn_fused c3, nn_pruned c4, p2s).  usage: tools/gpu_round_record.sh <tag>
TAG=${1:-rec}
mkdir -p gpurun_out
CFGS=${CFGS:-c1 c2 c3 c4 c5} tools/gpu_allcfg.sh $TAG
tools/gpu_launches.sh ${TAG}_l c3
tools/gpu_ncu_full.sh ${TAG}_fused c3 nn_fused
tools/gpu_ncu_kernel.sh ${TAG}_pruned nn_pruned 1 tools/run_forward.py c4 pruned 2
tools/gpu_ncu_kernel.sh ${TAG}_p2s p2s_kernel 1 tools/run_p2s.py brute
tools/gpu_ncu_kernel.sh ${TAG}_p2sp p2s_pruned_kernel 1 tools/run_p2s.py pruned
tools/gpu_ncu_kernel.sh ${TAG}_tc nn_tc_kernel 0 tools/run_tc.py c3 1
tools/gpu_ncu_kernel.sh ${TAG}_segg seg_sort_grad_kernel 1 tools/run_backward.py c3 2
tools/gpu_ncu_kernel.sh ${TAG}_gradc5 grad_kernel 1 tools/run_backward.py c5 2
tools/gpu_ncu_kernel.sh ${TAG}_scatc5 radix_scatter_kernel 1 tools/run_backward.py c5 2
