#!/bin/bash
# cfg3 FP64_FAST: P1 budget x amortised P1 (KS 8, exact prefix 8), 3 interleaved rounds -> gpurun_out/ab_fp64.txt
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in "48 0 0" "32 0 0" "48 8 8" "32 8 8" "40 8 8" "64 8 8"; do
    set -- $v
    echo "FP64_FAST budget=$1 ks=$2 pre=$3 $(FRACTAL_BUDGET=$1 FRACTAL_P1_AMORT=$2 FRACTAL_P1_PRE=$3 timeout 120 python tools/time_cfg.py cfg3 100 FP64_FAST 2>&1 | tail -1)"
  done
done > gpurun_out/ab_fp64.txt
