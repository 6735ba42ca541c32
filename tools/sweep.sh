#!/bin/bash
# Correctness under every scheduler + a scheduler/variant timing sweep.
TAG=${1:-sweep}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for S in auto static refill amort; do
  FRACTAL_SCHED=$S timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg5 and not cfg4_strict" > gpurun_out/pytest_${TAG}_$S.log 2>&1
  echo "rc=$?" >> gpurun_out/pytest_${TAG}_$S.log
done
for S in static refill amort; do
  FRACTAL_SCHED=$S timeout 300 python tools/perf_probe.py cfg2 cfg3 cfg5 > gpurun_out/perf_${TAG}_$S.log 2>&1
done
for V in 16,1 16,4 16,8 8,8; do
  FRACTAL_SCHED=refill FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_refill_$V.log 2>&1
done
