#!/bin/bash
# Same-box sweep of P1's budget (FRACTAL_BUDGET) on cfg3, fp32 and fp64 fast, interleaved.
# usage: tools/ab_budget.sh R -> gpurun_out/ab_budget.txt (ms per call)
set -u
mkdir -p gpurun_out
R=${1:-3}
for r in $(seq 1 $R); do
  for mode in FP32_FAST FP64_FAST; do
    for b in 24 32 40 48; do
      echo "$mode budget=$b $(FRACTAL_BUDGET=$b timeout 120 python tools/time_cfg.py cfg3 100 \
        $mode 2>&1 | tail -1)"
    done
  done
done > gpurun_out/ab_budget.txt
