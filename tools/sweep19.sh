#!/bin/bash
TAG=${1:-s}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "not largest and not schedulers and not cfg5 and not cfg4_strict" > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
FRACTAL_SCHED=static timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fuzz or ragged or bands or written or fast_mode_tolerance_julia" > gpurun_out/pytest_${TAG}_st.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_st.log
for S2 in 1 0; do FRACTAL_S2=$S2 timeout 200 python tools/perf_probe.py cfg1 cfg2 > gpurun_out/perf_${TAG}_s2$S2.log 2>&1; done
timeout 300 python tools/interactive_tick.py gpurun_out/tick_${TAG}.json > gpurun_out/tick_${TAG}.log 2>&1
