#!/bin/bash
# Same-box A/B of compile-time variants on the bench workload and single-frame configs:
# builds libfractal with each -D set into paper_1611_03079_b200/variants/, then R
# interleaved rounds of bench.py (--no-extra) and tools/time_cfg.py cfg2/cfg3 per variant.
# usage: tools/ab_cfgs.sh R name1:DEF1,DEF2 name2: ...   -> gpurun_out/abc_summary.txt
set -u
mkdir -p gpurun_out
R=$1; shift
V=paper_1611_03079_b200/variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python - "$name" "$defs" <<'PY' > gpurun_out/abc_build_$name.log 2>&1
import sys
from paper_1611_03079_b200 import build
print(build.build_variant(sys.argv[1], [d for d in sys.argv[2].split(",") if d]))
PY
done
: > gpurun_out/abc_raw.txt
for r in $(seq 1 $R); do
  for spec in "$@"; do
    name=${spec%%:*}
    export FRACTAL_LIB=$V/libfractal_$name.so
    b=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 2>/dev/null | tail -1)
    echo "$name bench $b" >> gpurun_out/abc_raw.txt
    for cfg in cfg2 cfg3; do
      t=$(timeout 120 python tools/time_cfg.py $cfg 200 2>/dev/null | tail -1)
      echo "$name $cfg $t" >> gpurun_out/abc_raw.txt
    done
    unset FRACTAL_LIB
  done
done
python - <<'PY' > gpurun_out/abc_summary.txt
import json, collections
res = collections.defaultdict(list)
for line in open("gpurun_out/abc_raw.txt"):
    parts = line.split(" ", 2)
    if len(parts) < 3 or not parts[2].strip():
        continue
    try:
        d = json.loads(parts[2])
    except Exception:
        continue
    v = d.get("ms_per_step", d.get("ms"))
    res[(parts[0], parts[1])].append(round(v, 4))
for k, v in sorted(res.items()):
    print(f"{k[0]:24s} {k[1]:6s} min={min(v):.4f} ms  all={v}")
PY
cat gpurun_out/abc_summary.txt
