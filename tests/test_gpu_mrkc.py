"""mRKC with the stiff-gate split (P/src/multirate.cpp:158-171,60-76;
P/src/simulate.cpp:132-150) on the device, against the CPU oracle (itself
pinned bitwise to the reference in test_oracle_vs_ref)."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import (MonodomainOperator, NumericalAbort,
                                              identify_stiff_gates)

pytestmark = pytest.mark.gpu

TOL = 1e-9
RHO_TOL = 1e-12


def test_gated_rhs_bit_exact(oracle):
    w = workloads.parity_3d()
    p = w.problem
    rng = np.random.default_rng(4)
    nn = p.n_nodes
    y = np.concatenate([rng.uniform(-90, 50, nn), rng.uniform(0, 1, 3 * nn)])
    op = MonodomainOperator(p)
    for stiff in (1, 3, 6):
        op.set_stiff_gates(stiff)
        for which, ow in ((capi.EMRKC_RHS_F_GATES, 0), (capi.EMRKC_RHS_S_GATES, 1)):
            got = op._rhs(which, 0.4, y)
            want = oracle.rhs_gates(p, ow, stiff, 0.4, y)
            # V rows: no transcendental, bit-exact; gate rows go through
            # libdevice exp vs the host libm: a few ulp of the rates (cancellation
            # in z - z_inf makes it absolute)
            assert np.array_equal(got[:nn], want[:nn]), (stiff, which)
            np.testing.assert_allclose(got[nn:], want[nn:], rtol=1e-12, atol=1e-13)
    op.close()


def test_identify_stiff_gates(oracle):
    V = np.linspace(-90.0, 40.0, 131)
    got = identify_stiff_gates(V)
    assert got == oracle.identify_stiff_gates(V) and got[0] == 0  # m is the stiffest


@pytest.mark.parametrize("name,nsteps", [("p2d_128_s3m2", 60), ("p3d_48_s2m2", 40),
                                         ("hh2d_256x256", 200), ("hh3d_sweep_100", 10)])
def test_mrkc_run_parity(oracle, name, nsteps):
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_stiff_gates(1)
    op.set_state(y0)
    rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F_GATES).rho
    rS = w.rho_S_forced if w.rho_S_forced is not None else \
        op.estimate_spectral_radius(capi.EMRKC_RHS_S_GATES).rho
    oF = oracle.estimate_rho_gates(p, oracle.RHS_F_GATES, 1, 0.0, y0)[0]
    assert abs(rF - oF.rho) <= RHO_TOL * oF.rho
    oS = w.rho_S_forced if w.rho_S_forced is not None else \
        oracle.estimate_rho_gates(p, oracle.RHS_S_GATES, 1, 0.0, y0)[0].rho
    res = op.mrkc_run(0, nsteps, w.dt, rF, rS, w.eps)
    yg = op.get_state()
    op.close()
    yo, ro, _ = oracle.run_mrkc(p, y0, 0, nsteps, w.dt, 1, w.eps, oF.rho, oS)
    assert (res.s, res.m) == (ro.s, ro.m)
    assert max(rel_l2_blocks(oracle, p, yg, yo)) <= TOL
    assert (res.n_fF, res.n_fS, res.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    assert res.n_exp == 0 and res.aborted == ro.aborted == 0
    assert abs(res.gate_min - ro.gate_min) <= 1e-9 and abs(res.gate_max - ro.gate_max) <= 1e-9


def test_mrkc_abort_and_guard(oracle):
    w = workloads.get("p3d_48_s2m2")
    p = w.problem
    y0 = w.initial_state()
    bad = y0.copy()
    bad[2 * p.n_nodes + 9] = np.nan  # h gate (slow part): inner stage 1 fails
    op = MonodomainOperator(p)
    op.set_state(bad)
    with pytest.raises(NumericalAbort) as ei:
        op.mrkc_step(0.0, w.dt, 388.0, 50.0, w.eps)
    assert ei.value.stage == 1 and ei.value.inner
    assert np.array_equal(op.get_state(), bad, equal_nan=True)
    res = op.mrkc_run(5, 3, w.dt, 388.0, 50.0, w.eps)
    _, ro, _ = oracle.run_mrkc(p, bad, 5, 3, w.dt, 1, w.eps, 388.0, 50.0)
    assert res.aborted == ro.aborted == 1 and res.abort_step == ro.abort_step == 5
    assert (res.abort_kind, res.abort_stage, res.abort_inner) == \
        (ro.abort_kind, ro.abort_stage, ro.abort_inner)
    assert (res.n_fF, res.n_fS, res.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    big = y0.copy()
    big[77] = 3e6
    op.set_state(big)
    res = op.mrkc_run(0, 3, w.dt, 388.0, 50.0, w.eps)
    yg = op.get_state()
    yo, ro, _ = oracle.run_mrkc(p, big, 0, 3, w.dt, 1, w.eps, 388.0, 50.0)
    assert res.abort_kind == ro.abort_kind and res.abort_step == ro.abort_step
    assert max(rel_l2_blocks(oracle, p, yg, yo)) <= TOL
    op.close()
