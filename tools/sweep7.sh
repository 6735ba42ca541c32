#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for S in refill auto; do
FRACTAL_SCHED=$S timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict" > gpurun_out/pytest_${TAG}_$S.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_$S.log
done
for V in 16,16 16,8 16,4 32,16 8,8; do
  FRACTAL_SCHED=refill FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_$V.log 2>&1
  FRACTAL_REFILL_CPC=0 FRACTAL_SCHED=refill FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_p_$V.log 2>&1
done
