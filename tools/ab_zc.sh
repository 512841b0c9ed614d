#!/bin/bash
# z-chunk sweep of k_node_pair (EMRKC_PAIR_ZC) through bench.py. Usage: tools/ab_zc.sh <workload> <steps> zc...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
wl=$1; steps=$2; shift 2
for zc in "$@"; do
  r=$(EMRKC_PAIR_ZC=$zc timeout 300 python bench.py --config $wl --steps $steps --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null \
      | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print("%.4e %.4f ms node %.4f ms frac %.3f" % (d["value"], d["ms_per_step"], r["mean_launch_ms"], r["frac"]))')
  echo "$wl zc=$zc $r"
done
