set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for S in 1 2; do
python tools/run_cfg3_scaled.py $S 2 > gpurun_out/one_s$S.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:escape -s 1 -c 1 -o gpurun_out/prof_cfg3_s$S -f python tools/run_cfg3_scaled.py $S 2 > gpurun_out/ncu_s$S.log 2>&1
done
echo done
