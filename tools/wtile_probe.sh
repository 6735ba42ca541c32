#!/bin/bash
# Kernel S warp-tile shape probe: bench value + per-launch DRAM bytes for FRACTAL_WTILE.
# usage: tools/wtile_probe.sh [widths...]   (default 8 16)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_wt.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1"
for w in ${@:-8 16}; do
  FRACTAL_WTILE=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 \
      > gpurun_out/wt_bench_$w.json 2>&1
  FRACTAL_WTILE=$w timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
      --clock-control none --csv -k regex:escape -s 3 -c 3 --log-file gpurun_out/wt_ncu_$w.csv $CMD \
      > gpurun_out/wt_ncu_$w.log 2>&1
done
