#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_SCHED=refill timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg5 and not cfg4" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
for O in 1 0; do for V in 16,16 16,8 16,1 8,8; do
  FRACTAL_ORDER=$O FRACTAL_SCHED=refill FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg2 cfg3 > gpurun_out/perf_${TAG}_o${O}_$V.log 2>&1
done; done
