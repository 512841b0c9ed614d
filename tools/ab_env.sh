#!/bin/bash
# Sweep one env var through bench.py. Usage: tools/ab_env.sh <workload> <steps> <VAR> values...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
wl=$1; steps=$2; var=$3; shift 3
for v in "$@"; do
  r=$(env $var=$v timeout 300 python bench.py --config $wl --steps $steps --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null \
      | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print("%.4e %.4f ms dom %.4f ms frac %.3f" % (d["value"], d["ms_per_step"], r["mean_launch_ms"], r["frac"]))')
  echo "$wl $var=$v $r"
done
