set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/run_one.py cfg2 3 > gpurun_out/o2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -s 2 -c 1 -o gpurun_out/prof_cfg2 -f python tools/run_one.py cfg2 3 > gpurun_out/ncu_cfg2.log 2>&1
python tools/run_colorize.py > gpurun_out/oc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:colorize -s 2 -c 1 -o gpurun_out/prof_colorize -f python tools/run_colorize.py > gpurun_out/ncu_col.log 2>&1
python tools/run_one.py cfg3 2 > gpurun_out/o3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -s 1 -c 1 -o gpurun_out/prof_cfg3_final -f python tools/run_one.py cfg3 2 > gpurun_out/ncu_cfg3f.log 2>&1
echo done
