#!/bin/bash
# Same-box A/B of one vs two tiles per P1 CTA (FRACTAL_P1_TILES) on cfg3, interleaved.
# usage: tools/ab_p1tiles.sh R -> gpurun_out/ab_p1tiles.txt (ms per call)
set -u
mkdir -p gpurun_out
R=${1:-3}
for r in $(seq 1 $R); do
  for mode in FP32_FAST FP32_STRICT FP64_FAST; do
    for t in 1 2; do
      echo "$mode tiles=$t $(FRACTAL_P1_TILES=$t timeout 120 python tools/time_cfg.py cfg3 100 \
        $mode 2>&1 | tail -1)"
    done
  done
done > gpurun_out/ab_p1tiles.txt
