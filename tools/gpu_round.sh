#!/bin/bash
# Standard GPU-box sequence: tests, bench, launch list, one full ncu capture.
# usage: tools/gpu_round.sh <tag> [pytest-args]
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs ${2:-} > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1"
timeout 300 $CMD > gpurun_out/bench_small_$TAG.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "ncu-launches rc=$?" >> gpurun_out/ncu_launches_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:escape -s 3 -c 1 \
    -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu-full rc=$?" >> gpurun_out/ncu_full_$TAG.log
