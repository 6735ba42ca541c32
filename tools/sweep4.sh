#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for C in 0 1 2 4 6; do
  FRACTAL_SCHED=refill FRACTAL_REFILL_CTAS_PER_SM=$C timeout 300 python tools/perf_probe.py cfg2 cfg3 > gpurun_out/perf_${TAG}_c$C.log 2>&1
  FRACTAL_SCHED=refill FRACTAL_REFILL=16,4 FRACTAL_REFILL_CTAS_PER_SM=$C timeout 300 python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_c${C}_164.log 2>&1
done
