#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_SCHED=refill timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict and not schedulers" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
for O in 1 0; do for C in 1 0; do FRACTAL_ORDER=$O FRACTAL_CONT=$C timeout 300 python tools/scale_probe.py > gpurun_out/scale_${TAG}_o${O}c$C.log 2>&1; done; done
