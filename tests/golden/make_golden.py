"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the
reference sources under /root/reference/proj/src compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo; nothing at test time reads /root/reference.
Each case stores the problem, the seeded initial state, the reference's
rho_F / rho_S estimates (value, iterations, converged), the stage plan, the
final state after n steps of run_simulation's emRKC loop and its run record
(counters, gate range, abort step / kind / stage).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402
from paper_2401_01745_b200.monodomain import make_problem  # noqa: E402

SIG_DEF = 0.17 * 0.62 / 0.79


def cases():
    yield "g1d_201_dt0.05", make_problem(1, [201], [0.1], [SIG_DEF], 140.0, 0.01, 50.0, [0.0], [1.5], 0.0, 2.0), 0.05, 100, None, "rest"
    yield "g2d_24x20", make_problem(2, [24, 20], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0, [-0.125, -0.125], [1.875, 1.875], 0.0, 1.0), 0.05, 40, None, "vnoise"
    yield "g3d_12x10x8", make_problem(3, [12, 10, 8], [0.25] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, [-0.125] * 3, [0.875] * 3, 0.0, 1.0), 0.05, 30, None, "vnoise"
    yield "g2d_32x24_s3m2", make_problem(2, [32, 24], [0.05, 0.05], [0.2, 0.2], 140.0, 0.01, 70.0, [-0.025, -0.025], [0.375, 0.375], 0.0, 1.0), 0.05, 15, 200.0, "vnoise"
    yield "g3d_16x12x10_s2m2", make_problem(3, [16, 12, 10], [0.05] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, [-0.025] * 3, [0.175] * 3, 0.0, 1.0), 0.05, 12, 50.0, "mult"
    yield "g2d_abort", make_problem(2, [16, 12], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0, [-0.125, -0.125], [0.875, 0.875], 0.0, 1.0), 0.05, 5, None, "nan"
    yield "g2d_guard", make_problem(2, [16, 12], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0, [-0.125, -0.125], [0.875, 0.875], 0.0, 1.0), 0.05, 5, None, "huge"


def initial(ref, p, kind, seed):
    y = ref.initial_state(p)
    nn = p.n_nodes
    rng = np.random.default_rng(seed)
    if kind == "vnoise":
        y[:nn] += rng.normal(0.0, 0.1, nn)
    elif kind == "mult":
        y *= rng.uniform(0.99, 1.01, y.size)
    elif kind == "nan":
        y[:nn] += rng.normal(0.0, 0.1, nn)
        y[2 * nn + 7] = np.nan
    elif kind == "huge":
        y[:nn] += rng.normal(0.0, 0.1, nn)
        y[nn // 2] = 4e6
    return y


def main():
    ref = Reference()
    index = {}
    for seed, (name, p, dt, n, rS_forced, kind) in enumerate(cases()):
        y0 = initial(ref, p, kind, 100 + seed)
        ok = np.all(np.isfinite(y0))
        if ok:
            eF, _ = ref.estimate_rho(p, 0, 0.0, y0)
            eS, _ = ref.estimate_rho(p, 1, 0.0, y0)
            rF, rS = eF.rho, (rS_forced if rS_forced is not None else eS.rho)
        else:
            eF = eS = None
            rF, rS = 20.0, 0.7
        y, res, _ = ref.run(p, y0, 0, n, dt, 0.05, rF, rS)
        rec = {k: getattr(res, k) for k, _ in res._fields_}
        rec.pop("device_ms")
        meta = {
            "problem": p.describe(), "dt": dt, "eps": 0.05, "n_steps": n,
            "rho_F": rF, "rho_S": rS,
            "rho_F_est": None if eF is None else [eF.rho, eF.iterations, eF.converged],
            "rho_S_est": None if eS is None else [eS.rho, eS.iterations, eS.converged],
            "rho_S_forced": rS_forced, "run": rec,
        }
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), y0=y0, y=y)
        index[name] = meta
        print(name, "s,m =", res.s, res.m, "aborted", res.aborted, "kind", res.abort_kind)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
