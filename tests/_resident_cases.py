"""Cases shared by tests/test_gpu_resident.py and its EMRKC_RESIDENT=0
subprocess: python tests/_resident_cases.py <out.npz> runs every case and
saves final states and run records."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem, resting_state  # noqa: E402


def _state(p, seed, edit=None):
    V, z = resting_state()
    nn = p.n_nodes
    y = np.concatenate([np.full(nn, V)] + [np.full(nn, z[g]) for g in range(3)])
    y[:nn] += np.random.default_rng(seed).normal(0.0, 0.1, nn)
    if edit:
        edit(y, nn)
    return y


def _p2():
    return make_problem(2, [64, 48], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                        [-0.125, -0.125], [3.875, 3.875], 0.0, 1.0)


def _p3():
    return make_problem(3, [24, 20, 18], [0.25] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0,
                        [-0.125] * 3, [0.875] * 3, 0.0, 1.0)


def _far(y, nn):
    rng = np.random.default_rng(9)
    idx = rng.choice(nn, 12, replace=False)
    y[idx] = rng.choice([160.0, -170.0, 400.0, -300.0, 1200.0], 12)


def _nan(y, nn):
    y[nn + 5] = np.nan


def _guard(y, nn):
    y[100] = 5e6


# name -> (problem, state edit, step0, nsteps, rho_F, rho_S, method)
CASES = {
    "2d_clean": (_p2, None, 0, 30, 10.0, 0.7, "emrkc"),
    "3d_clean": (_p3, None, 0, 25, 12.0, 0.7, "emrkc"),
    "3d_far": (_p3, _far, 0, 5, 12.0, 0.7, "emrkc"),
    "2d_nan": (_p2, _nan, 0, 5, 10.0, 0.7, "emrkc"),
    "2d_guard": (_p2, _guard, 3, 4, 10.0, 0.7, "emrkc"),
    "2d_progressive": (_p2, None, 0, 20, 10.0, 0.7, "progressive"),
    "3d_exex": (_p3, None, 0, 40, 0.0, 0.0, "exex"),
}


def run_case(name):
    mk, edit, step0, n, rF, rS, method = CASES[name]
    p = mk()
    op = MonodomainOperator(p)
    op.set_state(_state(p, 4, edit))
    if method == "exex":
        res = op.exex_run(step0, n, 0.01)
    else:
        from paper_2401_01745_b200 import capi
        var = capi.EMRKC_VARIANT_PROGRESSIVE if method == "progressive" else capi.EMRKC_VARIANT_STANDARD
        res = op.run(step0, n, 0.05, rF, rS, variant=var)
    y = op.get_state()
    rec = res.as_dict()
    op.close()
    return y, rec


if __name__ == "__main__":
    out = {}
    for name in CASES:
        y, rec = run_case(name)
        out[name + "/y"] = y
        for k, v in rec.items():
            out[name + "/" + k] = np.asarray(v)
    np.savez(sys.argv[1], **out)
