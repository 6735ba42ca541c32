#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_SCHED=refill timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict and not schedulers" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python tools/scale_probe.py > gpurun_out/scale_${TAG}.log 2>&1
for V in 16,8 16,16 16,24 8,8 32,16; do FRACTAL_REFILL=$V timeout 300 python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_$V.log 2>&1; done
FRACTAL_SCHED=refill timeout 300 python tools/perf_probe.py cfg2 > gpurun_out/perf_${TAG}_cfg2.log 2>&1
