#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_CONT=1 FRACTAL_SCHED=refill timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict and not schedulers" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 300 python tools/scale_probe.py > gpurun_out/scale_${TAG}_c0.log 2>&1
for C2 in 1 2 4 8; do FRACTAL_CONT=1 FRACTAL_CONT_CTAS=$C2 timeout 300 python tools/scale_probe.py > gpurun_out/scale_${TAG}_c1_$C2.log 2>&1; done
