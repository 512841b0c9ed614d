"""Temporally blocked inner stages (k_vin_tb: stages 2..m of an outer stage
in one HBM pass, north_star (1)): bitwise equal to the per-stage kernels and
within the parity bar of the CPU oracle, for m = 3, 4, 5 and s = 1, 2."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu

TOL = 1e-9


def problem(n, h):
    # iso sigma 0.1 mS/mm, chi 140/mm, C_m 0.01: rho_F ~ 0.9 / h^2
    return make_problem(3, n, [h] * 3, [0.1, 0.1, 0.1], 140.0, 0.01, 70.0,
                        [-0.5 * h] * 3, [3.5 * h] * 3, 0.0, 1.0)


def run(p, y0, rF, rS, nsteps, tb, monkeypatch):
    monkeypatch.setenv("EMRKC_TB", str(tb))
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(0, nsteps, 0.05, rF, rS)
    y = op.get_state()
    op.close()
    return y, res


@pytest.mark.parametrize("n,h,rho_S,want", [
    ((40, 36, 30), 0.06, None, (1, 3)),
    ((40, 36, 30), 0.045, None, (1, 4)),
    ((36, 34, 33), 0.035, None, (1, 5)),
    ((40, 36, 30), 0.035, 50.0, (2, 3)),
    ((34, 40, 36), 0.022, 50.0, (2, 4)),
])
def test_tb_matches_stagewise_and_oracle(oracle, monkeypatch, n, h, rho_S, want):
    p = problem(n, h)
    y0 = oracle.initial_state(p)
    y0[: p.n_nodes] += np.random.default_rng(7).normal(0.0, 0.1, p.n_nodes)
    rF = oracle.estimate_rho(p, 0, 0.0, y0)[0].rho
    rS = rho_S if rho_S is not None else oracle.estimate_rho(p, 1, 0.0, y0)[0].rho
    nsteps = 12
    y_tb, r_tb = run(p, y0, rF, rS, nsteps, 1, monkeypatch)
    y_st, r_st = run(p, y0, rF, rS, nsteps, 0, monkeypatch)
    assert (r_tb.s, r_tb.m) == want
    assert np.array_equal(y_tb, y_st)  # same arithmetic, same order
    yo, ro, _ = oracle.run(p, y0, 0, nsteps, 0.05, 0.05, rF, rS)
    assert (r_tb.s, r_tb.m) == (ro.s, ro.m)
    assert max(rel_l2_blocks(oracle, p, y_tb, yo)) <= TOL
    assert (r_tb.n_fF, r_tb.n_fS, r_tb.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    assert r_tb.aborted == ro.aborted == 0


def test_tb_nonfinite_inner_stage(oracle, monkeypatch):
    """A non-finite d_1 (from an infinite V far outside the fast range)
    reports the first failing stage in program order like the reference."""
    p = problem((40, 36, 30), 0.045)
    y0 = oracle.initial_state(p)
    y0[1234] = 1e300
    rF = 444.0
    y_tb, r_tb = run(p, y0, rF, 0.7, 3, 1, monkeypatch)
    y_st, r_st = run(p, y0, rF, 0.7, 3, 0, monkeypatch)
    _, ro, _ = oracle.run(p, y0, 0, 3, 0.05, 0.05, rF, 0.7)
    for r in (r_tb, r_st):
        assert r.aborted == ro.aborted
        assert (r.abort_kind, r.abort_step, r.abort_stage, r.abort_inner) == \
            (ro.abort_kind, ro.abort_step, ro.abort_stage, ro.abort_inner)
    assert np.array_equal(y_tb, y_st, equal_nan=True)
