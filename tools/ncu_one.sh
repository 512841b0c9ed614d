#!/bin/bash
# ncu --set full of one kernel launch of probe.py (after a plain run exits 0).
# Usage: tools/ncu_one.sh <out_name> <kernel_regex> <workload> [skip]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=$1; kre=$2; wl=$3; skip=${4:-5}
export EMRKC_PROBE_FAST_ONLY=1
python tools/probe.py $wl > gpurun_out/$out.plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/$out.plain.log; exit 1; }
tail -1 gpurun_out/$out.plain.log
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
  -o gpurun_out/$out python tools/probe.py $wl > gpurun_out/$out.ncu.log 2>&1
echo "ncu rc=$?"
