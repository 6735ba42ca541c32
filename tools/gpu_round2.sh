#!/bin/bash
# Round-2 GPU-box sequence: tests, smoke, bench, launch list of the bench command, one
# --set full capture of the bench kernel (SX), then a vote-block A/B of S2/P1.
# usage: tools/gpu_round2.sh <tag>
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
tools/ab_cfg_env.sh cfg2 2 "FRACTAL_VOTE_K=4" "FRACTAL_VOTE_K=2" > /dev/null 2>&1
cp gpurun_out/abce_summary.txt gpurun_out/ab_votek_cfg2_$TAG.txt
tools/ab_cfg_env.sh cfg3 2 "FRACTAL_VOTE_K=4" "FRACTAL_VOTE_K=2" > /dev/null 2>&1
cp gpurun_out/abce_summary.txt gpurun_out/ab_votek_cfg3_$TAG.txt
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -1 gpurun_out/smoke_$TAG.log
cat gpurun_out/ab_votek_cfg2_$TAG.txt gpurun_out/ab_votek_cfg3_$TAG.txt
