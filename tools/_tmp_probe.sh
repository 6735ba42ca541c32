python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for b in 64 96 128 160; do for o in 2 3; do FRACTAL_BUDGET=$b FRACTAL_P2_OCC=$o timeout 120 python tools/time_cfg.py cfg3 100 | sed "s/^/b=$b o=$o /"; done; done > gpurun_out/sw.txt 2>&1
for b in 64 96 128; do for o in 2 3; do FRACTAL_BUDGET=$b FRACTAL_P2_OCC=$o timeout 120 python tools/time_cfg.py cfg3 100 FP32_STRICT | sed "s/^/strict b=$b o=$o /"; done; done >> gpurun_out/sw.txt 2>&1
