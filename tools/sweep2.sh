#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg5" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
FRACTAL_STATIC_K=2 timeout 900 python -m pytest tests -m gpu -q -x -k "path or cfg4 or cfg2 or cfg1" > gpurun_out/pytest_${TAG}_k2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_k2.log
timeout 300 python tools/perf_probe.py cfg2 cfg4 > gpurun_out/perf_${TAG}_k4.log 2>&1
FRACTAL_STATIC_K=2 timeout 300 python tools/perf_probe.py cfg2 cfg4 > gpurun_out/perf_${TAG}_k2.log 2>&1
