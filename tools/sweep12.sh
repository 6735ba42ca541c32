#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_STATIC_K=2 timeout 900 python -m pytest tests -m gpu -q -x -k "path or cfg4 or cardioid or cfg1 or cfg2" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
for KK in 4 2; do for F in 32 64; do FRACTAL_STATIC_K=$KK FRACTAL_FPC=$F timeout 300 python tools/perf_probe.py cfg4 > gpurun_out/perf_${TAG}_k${KK}_f$F.log 2>&1; done; done
