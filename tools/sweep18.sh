#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for V in 128,4 64,8 64,4; do
  FRACTAL_AMORT=$V timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "strict_fuzz or cfg5" > gpurun_out/pytest_${TAG}_$V.log 2>&1 ; echo "rc=$?" >> gpurun_out/pytest_${TAG}_$V.log
  FRACTAL_AMORT=$V timeout 200 python tools/perf_probe.py cfg5 > gpurun_out/perf_${TAG}_$V.log 2>&1
done
