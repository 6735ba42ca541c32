set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export FRACTAL_REFILL=16,8
python tools/run_one.py cfg3 2 > gpurun_out/one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -s 1 -c 1 -o gpurun_out/prof_cfg3_r3 -f python tools/run_one.py cfg3 2 > gpurun_out/ncu_cfg3.log 2>&1
python tools/run_one.py cfg5 1 FP64_FAST 4096 > gpurun_out/one5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -c 1 -o gpurun_out/prof_cfg5_amort -f python tools/run_one.py cfg5 1 FP64_FAST 4096 > gpurun_out/ncu_cfg5.log 2>&1
echo done
