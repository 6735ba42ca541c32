#!/bin/bash
# Same-box A/B of the amortised P1 (FRACTAL_P1_AMORT = 0 / 4 / 8 sub-blocks after an exact
# prefix of FRACTAL_P1_PRE = 0 / 8 / 16 iterations) on cfg3, interleaved.
# usage: tools/ab_p1.sh R [extra env...]  -> gpurun_out/ab_p1.txt (ms per call)
set -u
mkdir -p gpurun_out
R=${1:-3}; shift || true
for r in $(seq 1 $R); do
  for mode in FP32_FAST FP64_FAST; do
    for v in 0:0 4:8 8:8 4:16 8:16; do
      ks=${v%:*}; pre=${v#*:}
      for b in 48 64; do
        echo "$mode ks=$ks pre=$pre budget=$b $(env FRACTAL_P1_AMORT=$ks FRACTAL_P1_PRE=$pre \
          FRACTAL_BUDGET=$b "$@" \
          timeout 120 python tools/time_cfg.py cfg3 100 $mode 2>&1 | tail -1)"
      done
    done
  done
done > gpurun_out/ab_p1.txt
