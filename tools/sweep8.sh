#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "not largest and not cfg5" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
for F in 8 16 32 64; do FRACTAL_FPC=$F timeout 300 python tools/perf_probe.py cfg4 > gpurun_out/perf_${TAG}_f$F.log 2>&1; done
timeout 300 python tools/perf_probe.py cfg2 > gpurun_out/perf_${TAG}_cfg2.log 2>&1
