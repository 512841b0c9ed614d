#!/bin/bash
# A/B timing of env-var variants through bench.py (L2 flushed per step).
# Usage: tools/ab.sh <workload> "<ENV=..>" "<ENV=..>" ...   (reps: AB_REPS, default 2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
wl=$1; shift
for rep in $(seq 1 ${AB_REPS:-2}); do
  for v in "$@"; do
    r=$(env $v timeout 300 python bench.py --config $wl --steps ${AB_STEPS:-300} --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null \
        | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("%.4e %.4f ms frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["frac"]))')
    echo "rep=$rep $wl [$v] $r"
  done
done
