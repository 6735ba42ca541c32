#!/bin/bash
# Same-box A/B of bench.py (no extras) under env settings, interleaved R rounds.
# usage: tools/ab_env.sh R "ENV=a" "ENV=b" ...   -> gpurun_out/ab_summary.txt (ms/step)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1
R=$1; shift
for r in $(seq 1 $R); do
  i=0
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-extra --cpu-seconds 1 \
        > gpurun_out/ab_${i}_$r.json 2>/dev/null
    i=$((i+1))
  done
done
python - "$R" "$@" > gpurun_out/ab_summary.txt <<'PY'
import json, sys
R, envs = int(sys.argv[1]), sys.argv[2:]
for i, e in enumerate(envs):
    v = []
    for r in range(1, R + 1):
        try:
            d = json.loads(open(f"gpurun_out/ab_{i}_{r}.json").read().strip().splitlines()[-1])
            v.append(round(d["ms_per_step"], 4))
        except Exception:
            v.append(None)
    print(f"{e:40s} {v}")
PY
