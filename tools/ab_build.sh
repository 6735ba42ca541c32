#!/bin/bash
# Same-box A/B of compile-time variants: builds libfractal with each -D set into
# paper_1611_03079_b200/variants/ and times bench.py (no extras) with FRACTAL_LIB, R rounds
# interleaved; also one ncu metric pass (time, instructions, DRAM bytes) per variant.
# usage: tools/ab_build.sh R name1:DEF1,DEF2 name2: ...   -> gpurun_out/abb_summary.txt
set -u
mkdir -p gpurun_out
R=$1; shift
V=paper_1611_03079_b200/variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python - "$name" "$defs" <<'PY' > gpurun_out/abb_build_$name.log 2>&1
import sys
from paper_1611_03079_b200 import build
print(build.build_variant(sys.argv[1], [d for d in sys.argv[2].split(",") if d]))
PY
done
for r in $(seq 1 $R); do
  for spec in "$@"; do
    name=${spec%%:*}
    FRACTAL_LIB=$V/libfractal_$name.so timeout 300 python bench.py --steps 10 --warmup 3 \
        --no-extra --cpu-seconds 1 > gpurun_out/abb_${name}_$r.json 2>/dev/null
  done
done
CMD="python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1"
for spec in "$@"; do
  name=${spec%%:*}
  FRACTAL_LIB=$V/libfractal_$name.so timeout 600 ncu --metrics \
      gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv -k regex:escape -s 3 -c 1 \
      --log-file gpurun_out/abb_ncu_$name.csv $CMD > /dev/null 2>&1
done
python - "$R" "$@" > gpurun_out/abb_summary.txt <<'PY'
import csv, json, sys
R, specs = int(sys.argv[1]), sys.argv[2:]
for spec in specs:
    name = spec.split(":")[0]
    v = []
    for r in range(1, R + 1):
        try:
            d = json.loads(open(f"gpurun_out/abb_{name}_{r}.json").read().strip().splitlines()[-1])
            v.append(round(d["ms_per_step"], 4))
        except Exception:
            v.append(None)
    m = {}
    try:
        lines = [l for l in open(f"gpurun_out/abb_ncu_{name}.csv") if l.startswith('"')]
        for row in csv.DictReader(lines):
            m[row["Metric Name"]] = row["Metric Value"]
    except Exception as e:
        m = {"err": str(e)}
    print(f"{spec:40s} ms={v} {m}")
PY
