"""Generate tests/golden/runs.json from the REFERENCE ITSELF (oracle/_ref) on
BASELINE workloads too large to store whole: run_simulation's emRKC loop from
the workload's seeded initial state (paper_2401_01745_b200.workloads, numpy
PCG64: identical bytes on every machine) and keep the run record (s, m, rho,
counters, gate range, abort step / kind / stage), per-block L2 norms and sums
of the final state, and 512 seeded sample nodes per block.

Run here (where /root/reference exists):  python tests/golden/make_runs.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Reference  # noqa: E402
from paper_2401_01745_b200 import workloads  # noqa: E402

# (workload, steps): config 5 at N = 100 runs into the reference's own
# NumericalAbort at step 47 (HH at h = 0.1 mm, m = 2); N = 50 and config 2
# run clean over their full T.
RUNS = [("hh3d_sweep_100", 60), ("hh3d_sweep_50", 100), ("hh3d_128x128x128", 100),
        ("hh3d_sweep_200", 60)]
# The reference's own conditioning: the same run from y0 (1 + 1e-15 u),
# u ~ U(-1, 1) seeded, diverges from the unperturbed run by "sensitivity"
# (trapezoid rel-L2 per block, the reference's rel_l2_error).
NSAMP = 512


def main():
    ref = Reference()
    orc = Oracle()
    out = {}
    for name, n in RUNS:
        w = workloads.get(name)
        p = w.problem
        y0 = w.initial_state()
        rF, _ = ref.estimate_rho(p, 0, 0.0, y0)
        rS, _ = ref.estimate_rho(p, 1, 0.0, y0)
        y, res, wall = ref.run(p, y0, 0, n, w.dt, w.eps, rF.rho, rS.rho)
        nn = p.n_nodes
        y1 = y0 * (1.0 + 1e-15 * np.random.default_rng(5).uniform(-1.0, 1.0, y0.size))
        yp, resp, _ = ref.run(p, y1, 0, n, w.dt, w.eps, rF.rho, rS.rho)
        sens = [float(orc.rel_l2(p, yp[b * nn:(b + 1) * nn], y[b * nn:(b + 1) * nn]))
                for b in range(4)]
        idx = np.sort(np.random.default_rng(1234).choice(nn, NSAMP, replace=False))
        blocks = [y[b * nn:(b + 1) * nn] for b in range(4)]
        out[name] = {
            "steps": n, "dt": w.dt, "eps": w.eps,
            "rho_F": rF.rho, "rho_F_iterations": rF.iterations,
            "rho_S": rS.rho, "rho_S_iterations": rS.iterations,
            "record": {k: (float(v) if isinstance(v, float) else int(v))
                       for k, v in res.as_dict().items() if k != "device_ms"},
            "norm2": [float(np.linalg.norm(b)) for b in blocks],
            "sum": [float(np.sum(b)) for b in blocks],
            "sample_index": idx.tolist(),
            "sample": [b[idx].tolist() for b in blocks],
            "ref_wall_s": wall,
            "sensitivity": sens,
            "sensitivity_same_abort": bool(resp.abort_step == res.abort_step),
        }
        print(name, out[name]["record"], f"{wall:.1f} s", "sensitivity", sens, flush=True)
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
