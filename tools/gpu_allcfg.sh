#!/bin/bash
# bench lines for every config + a 2-rank gloo run on one GPU (multi-rank code path smoke)
TAG=${1:-x}
mkdir -p gpurun_out
for c in ${CFGS:-c1 c2 c3 c4 c5}; do
  python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "$c rc=$?"
  python - <<PY
import json; d=json.load(open("gpurun_out/bench_${TAG}_$c.json"))
r=d["roofline"]; pr=d.get("pruned") or {}; print("$c next", json.dumps(d.get("next_rows"))); print("$c pruned ms %.4f eff %.4g speedup %.2f lossdiff %.2g" % (pr.get("ms_per_step",0), pr.get("value_effective",0), pr.get("speedup_vs_brute_step",0), pr.get("loss_rel_diff_vs_brute",0))); print("$c value %.4g ms/step %.4f kernel_ms %.4f frac %.3f eff%% %.1f e2e %.4g cpu %.4g launch %s clocks %s" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], d["pct_fp32_fma_peak_effective"], (d.get("e2e") or {}).get("value") or 0, (d.get("cpu_baseline") or {}).get("value") or 0, d["config"].get("launch"), d.get("clocks")))
PY
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c3 --steps 10 --warmup 3 --dist-backend gloo > gpurun_out/bench_${TAG}_dist_c3.json 2> gpurun_out/bench_${TAG}_dist_c3.err; echo "dist c3 rc=$?"; cut -c1-400 gpurun_out/bench_${TAG}_dist_c3.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo > gpurun_out/bench_${TAG}_dist_c5.json 2> gpurun_out/bench_${TAG}_dist_c5.err; echo "dist c5 (default N>1 config) rc=$?"; cut -c1-400 gpurun_out/bench_${TAG}_dist_c5.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config c4 --steps 5 --warmup 2 --dist-backend gloo > gpurun_out/bench_${TAG}_dist_c4.json 2> gpurun_out/bench_${TAG}_dist_c4.err; echo "dist c4 strong rc=$?"; cut -c1-400 gpurun_out/bench_${TAG}_dist_c4.json
python bench.py --impl reference --config c3 --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref_c3.json 2> gpurun_out/bench_${TAG}_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_${TAG}_ref_c3.json
