"""BASELINE config 5 (stiffness sweep) and the other workloads at 1 GPU:
s, m, rho and device node-steps/s per workload, same protocol as bench.py's
`value` (per-launch CUDA events, L2 flushed before every step).

    python tools/sweep.py [--steps 20] > profiles/<tag>_sweep.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2401_01745_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--names", nargs="*", default=[
    "hh3d_sweep_25", "hh3d_sweep_50", "hh3d_sweep_100", "hh3d_sweep_200",
    "hh2d_256x256", "hh3d_128x128x128", "hh3d_256x256x128", "hh3d_512x512x256"])
args = ap.parse_args()
peak, kind = bench.hbm_peak()
rows = []
for name in args.names:
    w = workloads.get(name)
    m = bench.measure_device(w, 0, 3, args.steps, with_e2e=False)
    tot = float(m["launch_ms"].sum())
    rf = bench.roofline_of(m, w, peak, kind)
    rows.append({"workload": name, "nodes": w.n_nodes, "h_mm": w.problem.dx[0], "s": m["s"],
                 "m": m["m"], "rho_F": m["rF"], "rho_S": m["rS"],
                 "node_steps_per_s": w.n_nodes * args.steps / (tot * 1e-3),
                 "ms_per_step": tot / args.steps, "step_frac_hbm": rf["step_frac"],
                 "dominant_kernel": rf["kernel"], "dominant_frac": rf["frac"],
                 "run": m["run"],
                 "note": w.note})
    m["op"].close()
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
print(json.dumps({"steps": args.steps, "hbm_peak_gbs": peak, "rows": rows}, indent=1))
