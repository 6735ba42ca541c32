#!/bin/bash
# GPU-box consolidation run: build, full -m gpu suite, smoke, bench (10 steps), the ncu
# launch list of the bench command, one --set full capture of the bench kernel, the
# interactive tick, the Fig. 1 sweep and the small-frame latency probe.
# usage: tools/gpu_profile.sh <tag>
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1"
timeout 300 $CMD > gpurun_out/bench_small_$TAG.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "ncu-launches rc=$?" >> gpurun_out/ncu_launches_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:escape -s 3 -c 1 \
    -o gpurun_out/prof_bench_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu-full rc=$?" >> gpurun_out/ncu_full_$TAG.log
timeout 300 python tools/interactive_tick.py > gpurun_out/tick_$TAG.json 2>&1
timeout 600 python tools/fig1_sweep.py gpurun_out/fig1_$TAG.json > gpurun_out/fig1_$TAG.log 2>&1
timeout 300 python tools/latency_probe.py > gpurun_out/latency_$TAG.txt 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
tail -c 1500 gpurun_out/bench_$TAG.json
