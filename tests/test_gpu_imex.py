"""IMEX-RL with device CG (P/src/baselines.cpp:20-82,132-190) against the CPU
oracle (pinned bitwise to the reference in test_oracle_vs_ref)."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator, NumericalAbort

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.mark.parametrize("name,dt,nsteps,jacobi", [("p2d_128_s3m2", 0.02, 40, True),
                                                   ("p3d_48_s2m2", 0.05, 20, True),
                                                   ("hh2d_256x256", 0.05, 100, False),
                                                   ("hh3d_sweep_50", 0.05, 20, True)])
def test_imex_run_parity(oracle, name, dt, nsteps, jacobi):
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    res, it = op.imex_run(0, nsteps, dt, 1e-8, 0, jacobi)
    yg = op.get_state()
    op.close()
    yo, ro, io = oracle.run_imex(p, y0, 0, nsteps, dt, 1e-8, 0, jacobi)
    assert max(rel_l2_blocks(oracle, p, yg, yo)) <= TOL
    # CG iterations: reductions run in another order; a borderline stopping
    # test may move by one iteration in a step
    assert abs(it - io) <= max(1, nsteps // 20)
    assert res.n_fF - it == ro.n_fF - io == 2 * nsteps
    assert (res.n_fS, res.n_exp) == (ro.n_fS, ro.n_exp) == (nsteps, nsteps)
    assert res.aborted == ro.aborted == 0 and res.steps_done == nsteps
    assert abs(res.gate_min - ro.gate_min) <= 1e-9 and abs(res.gate_max - ro.gate_max) <= 1e-9


def test_imex_cg_failure_and_step(oracle):
    w = workloads.get("p2d_128_s3m2")
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    res, _ = op.imex_run(4, 3, 0.05, 1e-12, 2, True)
    _, ro, _ = oracle.run_imex(p, y0, 4, 3, 0.05, 1e-12, 2, True)
    assert res.aborted == ro.aborted == 1 and res.abort_step == ro.abort_step == 4
    assert res.abort_kind == ro.abort_kind == capi.EMRKC_ABORT_NONFINITE
    assert np.array_equal(op.get_state(), y0)  # not assigned
    with pytest.raises(NumericalAbort):
        op.imex_step(0.0, 0.05, 1e-12, 2)
    rep, it = op.imex_step(0.0, 0.05)
    yo, _, io = oracle.run_imex(p, y0, 0, 1, 0.05)
    assert max(rel_l2_blocks(oracle, p, op.get_state(), yo)) <= TOL and abs(it - io) <= 1
    op.close()
