#!/bin/bash
# Iteration call: gpu tests (quick subset or all), bench line, optional ncu full of the top kernel.
# usage: tools/gpu_iter.sh <tag> [tests-k-expr|all|none] [ncu-kernel-regex|none] [config]
TAG=${1:-x}; TESTS=${2:-all}; K=${3:-nn_fused}; CFG=${4:-c3}
mkdir -p gpurun_out
if [ "$TESTS" = "all" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_$TAG.log
elif [ "$TESTS" != "none" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTS" > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_$TAG.log; fi
python bench.py --config $CFG --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json; d=json.load(open("gpurun_out/bench_$TAG.json"))
r=d["roofline"]; print("value %.4g ms/step %.4f kernel_ms %.4f frac %.3f eff%% %.1f e2e %.4g clocks %s" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], d["pct_fp32_fma_peak_effective"], (d.get("e2e") or {}).get("value") or 0, d.get("clocks")))
PY
if [ "$K" != "none" ]; then tools/gpu_ncu_full.sh $TAG $CFG $K; fi
