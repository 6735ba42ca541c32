#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for S in refill amort; do
FRACTAL_SCHED=$S timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4" > gpurun_out/pytest_${TAG}_$S.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_$S.log
done
for C in 0 4 8 16 32; do for V in 16,8 16,1; do
  FRACTAL_REFILL_CPC=$C FRACTAL_SCHED=refill FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg2 cfg3 > gpurun_out/perf_${TAG}_c${C}_$V.log 2>&1
done; done
for C in 0 16 64; do FRACTAL_REFILL_CPC=$C timeout 300 python tools/perf_probe.py cfg5 > gpurun_out/perf_${TAG}_cfg5_c$C.log 2>&1; done
