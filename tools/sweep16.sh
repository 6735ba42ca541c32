#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_SCHED=refill timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "strict_configs_full_frame" > gpurun_out/pytest_${TAG}_0.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_0.log
grep -q "rc=0" gpurun_out/pytest_${TAG}_0.log || exit 3
FRACTAL_SCHED=refill timeout 300 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict and not schedulers" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 120 python tools/refill_timeline.py 1 > gpurun_out/tl_${TAG}.log 2>&1
for T in 8 4 16 0; do FRACTAL_TAIL_CHUNKS_PER_WARP16=$T timeout 120 python tools/scale_probe.py > gpurun_out/scale_${TAG}_t$T.log 2>&1; done
