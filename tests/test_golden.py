"""Golden vectors produced by the reference itself (tests/golden/make_golden.py
runs oracle/_ref = the reference sources compiled in place). The C oracle
must reproduce them bit for bit; the GPU path within the north_star bar."""
import json
import os

import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200.capi import Problem

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(HERE, "golden.json")) as _f:
    GOLDEN = json.load(_f)
NAMES = sorted(GOLDEN)


def load(name):
    meta = GOLDEN[name]
    d = np.load(os.path.join(HERE, f"{name}.npz"))
    return meta, Problem.from_dict(meta["problem"]), d["y0"], d["y"]


def check_record(res, run, exact=True):
    for k in ("n_steps", "steps_done", "aborted", "abort_kind", "abort_step", "abort_stage",
              "n_fF", "n_fS", "n_exp", "s", "m"):
        assert getattr(res, k) == run[k], (k, getattr(res, k), run[k])
    if exact:
        assert res.gate_min == run["gate_min"] and res.gate_max == run["gate_max"]
        assert res.eta == run["eta"]
    else:
        assert abs(res.gate_min - run["gate_min"]) <= 1e-9
        assert abs(res.gate_max - run["gate_max"]) <= 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_reference_golden(oracle, name):
    meta, p, y0, y_ref = load(name)
    if meta["rho_F_est"] is not None:
        for which, key in ((0, "rho_F_est"), (1, "rho_S_est")):
            est, _ = oracle.estimate_rho(p, which, 0.0, y0)
            assert [est.rho, est.iterations, est.converged] == meta[key]
    y, res, _ = oracle.run(p, y0, 0, meta["n_steps"], meta["dt"], meta["eps"], meta["rho_F"],
                           meta["rho_S"])
    check_record(res, meta["run"], exact=True)
    assert np.array_equal(y, y_ref, equal_nan=True)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(oracle, name):
    from paper_2401_01745_b200.monodomain import MonodomainOperator

    meta, p, y0, y_ref = load(name)
    op = MonodomainOperator(p)
    op.set_state(y0)
    if meta["rho_F_est"] is not None:
        for which, key in ((0, "rho_F_est"), (1, "rho_S_est")):
            est = op.estimate_spectral_radius(which, 0.0)
            ref = meta[key]
            assert est.iterations == ref[1] and est.converged == bool(ref[2])
            assert abs(est.rho - ref[0]) <= 1e-9 * ref[0]
    res = op.run(0, meta["n_steps"], meta["dt"], meta["rho_F"], meta["rho_S"], meta["eps"])
    check_record(res, meta["run"], exact=False)
    y = op.get_state()
    if meta["run"]["abort_kind"] == 1:
        assert np.array_equal(y, y_ref, equal_nan=True)  # state not assigned
    else:
        assert max(rel_l2_blocks(oracle, p, y, y_ref)) <= 1e-9
