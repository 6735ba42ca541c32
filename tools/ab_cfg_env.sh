#!/bin/bash
# Same-box A/B of one single-frame config (tools/time_cfg.py) under env settings, R
# interleaved rounds.  usage: tools/ab_cfg_env.sh cfg3 R "ENV=a ENV2=b" "ENV=c" ...
#   -> gpurun_out/abce_summary.txt (min and all ms per call)
set -u
mkdir -p gpurun_out
CFG=$1; R=$2; shift 2
: > gpurun_out/abce_raw.txt
for r in $(seq 1 $R); do
  i=0
  for e in "$@"; do
    t=$(env $e timeout 120 python tools/time_cfg.py $CFG 200 2>/dev/null | tail -1)
    echo "$i|$e|$t" >> gpurun_out/abce_raw.txt
    i=$((i+1))
  done
done
python - <<'PY' > gpurun_out/abce_summary.txt
import json, collections
res, names = collections.defaultdict(list), {}
for line in open("gpurun_out/abce_raw.txt"):
    i, e, t = line.rstrip("\n").split("|", 2)
    names[i] = e
    try:
        res[i].append(round(json.loads(t)["ms"], 4))
    except Exception:
        res[i].append(None)
for i in sorted(res, key=int):
    v = [x for x in res[i] if x is not None]
    print(f"{names[i]:50s} min={min(v) if v else None} all={res[i]}")
PY
cat gpurun_out/abce_summary.txt
