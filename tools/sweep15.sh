#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
FRACTAL_SCHED=refill timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "strict_configs_full_frame and cfg1" > gpurun_out/pytest_${TAG}_0.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_0.log
grep -q "rc=0" gpurun_out/pytest_${TAG}_0.log || exit 3
FRACTAL_SCHED=refill timeout 300 python -m pytest tests -m gpu -q -x -k "not largest and not cfg4_strict and not schedulers" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
grep -q "rc=0" gpurun_out/pytest_${TAG}.log || exit 4
FRACTAL_SCHED=refill FRACTAL_REFILL_CPC=16 timeout 300 python -m pytest tests -m gpu -q -x -k "strict_fuzz or bands or written or ragged" > gpurun_out/pytest_${TAG}_cpc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_cpc.log
for C in 1 0; do FRACTAL_COMPACT=$C timeout 120 python tools/scale_probe.py > gpurun_out/scale_${TAG}_c$C.log 2>&1; done
for V in 16,8 16,16 16,4; do timeout 120 env FRACTAL_REFILL=$V python tools/perf_probe.py cfg3 > gpurun_out/perf_${TAG}_$V.log 2>&1; done
