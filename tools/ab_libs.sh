#!/bin/bash
# Same-box A/B of PRE-BUILT libraries under paper_1611_03079_b200/variants/ (no rebuild):
# R interleaved rounds of bench.py (--no-extra) and tools/time_cfg.py cfg2/cfg3.
# usage: tools/ab_libs.sh R name1 name2 ...   -> gpurun_out/abl_summary.txt
set -u
mkdir -p gpurun_out
R=$1; shift
V=paper_1611_03079_b200/variants
: > gpurun_out/abl_raw.txt
for r in $(seq 1 $R); do
  for name in "$@"; do
    export FRACTAL_LIB=$V/libfractal_$name.so
    b=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 2>/dev/null | tail -1)
    echo "$name bench $b" >> gpurun_out/abl_raw.txt
    for cfg in cfg2 cfg3; do
      t=$(timeout 120 python tools/time_cfg.py $cfg 200 2>/dev/null | tail -1)
      echo "$name $cfg $t" >> gpurun_out/abl_raw.txt
    done
    unset FRACTAL_LIB
  done
done
python - <<'PY' > gpurun_out/abl_summary.txt
import json, collections
res = collections.defaultdict(list)
for line in open("gpurun_out/abl_raw.txt"):
    parts = line.split(" ", 2)
    if len(parts) < 3 or not parts[2].strip():
        continue
    try:
        d = json.loads(parts[2])
    except Exception:
        continue
    res[(parts[0], parts[1])].append(round(d.get("ms_per_step", d.get("ms")), 4))
for k, v in sorted(res.items()):
    print(f"{k[0]:24s} {k[1]:6s} min={min(v):.4f} ms  all={v}")
PY
cat gpurun_out/abl_summary.txt
