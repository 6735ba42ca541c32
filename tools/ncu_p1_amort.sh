#!/bin/bash
# Launch list (time + warp-instructions) of cfg3 fast with the exact and the amortised P1.
# usage: tools/ncu_p1_amort.sh -> gpurun_out/launches_p1_<KS>_<PRE>.csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_p1l.log 2>&1
for v in "0 0" "4 16" "8 0"; do
  set -- $v
  FRACTAL_P1_AMORT=$1 FRACTAL_P1_PRE=$2 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/launches_p1_$1_$2.csv python tools/time_cfg.py cfg3 5 FP32_FAST > gpurun_out/ncu_p1_$1_$2.log 2>&1
done
