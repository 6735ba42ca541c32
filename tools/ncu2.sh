set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/run_one.py cfg3 2 > gpurun_out/one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -s 1 -c 1 -o gpurun_out/prof_cfg3_refill -f python tools/run_one.py cfg3 2 > gpurun_out/ncu_cfg3.log 2>&1
python tools/run_one.py cfg4 1 > gpurun_out/one4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -c 1 -o gpurun_out/prof_cfg4_static -f python tools/run_one.py cfg4 1 > gpurun_out/ncu_cfg4.log 2>&1
echo done
