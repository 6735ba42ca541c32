#!/bin/bash
# Same-box A/B of the fast two-orbit vote block in S2 and P1 (FRACTAL_VOTE_K = 4 / 2),
# cfg2 (S2) and cfg3 (P1 + P2), interleaved.  usage: tools/ab_votek.sh R -> gpurun_out/ab_votek.txt
set -u
mkdir -p gpurun_out
R=${1:-3}
for r in $(seq 1 $R); do
  for cfg in cfg2 cfg3; do
    for k in 4 2; do
      echo "$cfg K=$k $(FRACTAL_VOTE_K=$k timeout 120 python tools/time_cfg.py $cfg 200 \
        FP32_FAST 2>&1 | tail -1)"
    done
  done
done > gpurun_out/ab_votek.txt
