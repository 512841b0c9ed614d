"""GPU parity of the other stepping methods on the device path, against the
CPU oracle (itself pinned bitwise to the reference in test_oracle_vs_ref):

* emRKC progressive variant (P/src/multirate.cpp:106-115);
* EXEX-RL, the reference-solution stepper (P/src/baselines.cpp:192-210),
  inside run_simulation's loop (norm guard, gate range, counters).

Bars as in test_gpu_parity: s, m exact; rel-L2 <= 1e-9 per SoA block."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import CudaError, MonodomainOperator, exex_rl_step

pytestmark = pytest.mark.gpu

TOL = 1e-9
PROG = capi.EMRKC_VARIANT_PROGRESSIVE


@pytest.mark.parametrize("name,nsteps", [("p2d_128_s3m2", 60), ("p3d_48_s2m2", 40),
                                         ("hh2d_256x256", 200), ("hh3d_sweep_100", 10)])
def test_progressive_run_parity(oracle, name, nsteps):
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    rF = op.estimate_spectral_radius(0).rho
    rS = w.rho_S_forced if w.rho_S_forced is not None else op.estimate_spectral_radius(1).rho
    res = op.run(0, nsteps, w.dt, rF, rS, w.eps, variant=PROG)
    yg = op.get_state()
    op.close()
    oF = oracle.estimate_rho(p, 0, 0.0, y0)[0].rho
    oS = w.rho_S_forced if w.rho_S_forced is not None else oracle.estimate_rho(p, 1, 0.0, y0)[0].rho
    yo, ro, _ = oracle.run_method(p, y0, 0, nsteps, w.dt, oracle.EMRKC_PROGRESSIVE, w.eps, oF, oS)
    assert (res.s, res.m) == (ro.s, ro.m)
    errs = rel_l2_blocks(oracle, p, yg, yo)
    assert max(errs) <= TOL, errs
    assert (res.n_fF, res.n_fS, res.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    assert res.aborted == ro.aborted == 0
    assert abs(res.gate_min - ro.gate_min) <= 1e-9 and abs(res.gate_max - ro.gate_max) <= 1e-9


def test_progressive_step_api(oracle):
    w = workloads.get("p3d_48_s2m2")
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    rep = op.step(0.0, w.dt, 388.2, w.rho_S_forced, w.eps, variant=PROG)
    assert (rep.s, rep.m) == (2, 2)
    yo, ro, _ = oracle.run_method(p, y0, 0, 1, w.dt, oracle.EMRKC_PROGRESSIVE, w.eps, 388.2,
                                  w.rho_S_forced)
    assert max(rel_l2_blocks(oracle, p, op.get_state(), yo)) <= TOL
    op.close()


def test_progressive_needs_fast_kernels(monkeypatch):
    monkeypatch.setenv("EMRKC_FAST", "0")
    w = workloads.get("p3d_48_s2m2")
    op = MonodomainOperator(w.problem)
    op.set_state(w.initial_state())
    with pytest.raises(ValueError):
        op.run(0, 1, w.dt, 388.2, w.rho_S_forced, w.eps, variant=PROG)
    op.close()


@pytest.mark.parametrize("name,dt,nsteps", [("p2d_128_s3m2", 0.002, 300),
                                            ("p3d_48_s2m2", 0.002, 100),
                                            ("hh2d_256x256", 0.01, 400),
                                            ("hh3d_sweep_50", 0.005, 100)])
def test_exex_run_parity(oracle, name, dt, nsteps):
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.exex_run(0, nsteps, dt)
    yg = op.get_state()
    op.close()
    yo, ro, _ = oracle.run_method(p, y0, 0, nsteps, dt, oracle.EXEX_RL)
    errs = rel_l2_blocks(oracle, p, yg, yo)
    assert max(errs) <= TOL, errs
    assert res.n_fF == res.n_fS == res.n_exp == ro.n_fF == nsteps
    assert res.aborted == ro.aborted == 0 and res.steps_done == nsteps
    assert abs(res.gate_min - ro.gate_min) <= 1e-9 and abs(res.gate_max - ro.gate_max) <= 1e-9


def test_exex_nonfinite_gate_guard(oracle):
    """A NaN gate is no NumericalAbort under EXEX-RL: V turns NaN in the same
    step (reaction at the new gates) and the norm guard stops the run with
    the state assigned."""
    w = workloads.get("p2d_128_s3m2")
    p = w.problem
    y0 = w.initial_state()
    y0[p.n_nodes + 7] = np.nan
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.exex_run(2, 5, 0.002)
    yg = op.get_state()
    op.close()
    yo, ro, _ = oracle.run_method(p, y0, 2, 5, 0.002, oracle.EXEX_RL)
    assert res.aborted and ro.aborted
    assert res.abort_kind == ro.abort_kind == capi.EMRKC_ABORT_NORM_GUARD
    assert res.abort_step == ro.abort_step == 2 and res.steps_done == ro.steps_done == 1
    assert np.array_equal(np.isnan(yg), np.isnan(yo))
    fin = ~np.isnan(yo)
    np.testing.assert_allclose(yg[fin], yo[fin], rtol=1e-9, atol=1e-12)


def test_exex_step_dropin(oracle):
    w = workloads.get("p3d_48_s2m2")
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    y1 = exex_rl_step(0.0, y0, 0.002, op)
    yo, _, _ = oracle.run_method(p, y0, 0, 1, 0.002, oracle.EXEX_RL)
    assert max(rel_l2_blocks(oracle, p, y1, yo)) <= TOL
    with pytest.raises((ValueError, CudaError)):
        op.exex_step(0.0, -1.0)
    op.close()


@pytest.mark.parametrize("name", ["hh3d_128x128x128", "hh2d_256x256", "hh3d_sweep_100",
                                  "hh3d_sweep_200"])
def test_step_host_pipelined_matches_device_step(oracle, name):
    """emrkc_step_host streams s = 1 steps in z-chunks, stencil level k
    lagging the copy-in by k planes (m = 1, 2 and 4 here; copies overlap the
    step); results equal the device-resident step bit for bit."""
    import ctypes as C
    import torch

    from paper_2401_01745_b200.capi import StepReport, dptr
    from paper_2401_01745_b200.monodomain import _lib

    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    rF = op.estimate_spectral_radius(0).rho
    rS = op.estimate_spectral_radius(1).rho
    ref = op
    ref.step(0.0, w.dt, rF, rS, w.eps)
    ref.step(w.dt, w.dt, rF, rS, w.eps)
    y_dev = ref.get_state()
    hin = torch.from_numpy(y0.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    h2 = MonodomainOperator(p)
    rep = StepReport()
    for k in range(2):
        rc = _lib().emrkc_step_host(h2.handle, k * w.dt, C.cast(hin.data_ptr(), C.POINTER(C.c_double)),
                                    C.cast(hout.data_ptr(), C.POINTER(C.c_double)), hin.numel(),
                                    w.dt, w.eps, capi.EMRKC_VARIANT_STANDARD, rF, rS, C.byref(rep))
        assert rc == 0
        assert rep.s == 1 and rep.n_fF == rep.m and (rep.n_fS, rep.n_exp) == (1, 1)
        hin.copy_(hout)
    assert np.array_equal(hout.numpy(), y_dev)
    assert np.array_equal(h2.get_state(), y_dev)
    # aliasing y_out = y_in
    hin.copy_(torch.from_numpy(y0))
    for k in range(2):
        assert _lib().emrkc_step_host(h2.handle, k * w.dt, C.cast(hin.data_ptr(), C.POINTER(C.c_double)),
                                      C.cast(hin.data_ptr(), C.POINTER(C.c_double)), hin.numel(),
                                      w.dt, w.eps, 0, rF, rS, C.byref(rep)) == 0
    assert np.array_equal(hin.numpy(), y_dev)
    # NumericalAbort: device state stays y_in
    bad = y0.copy()
    bad[p.n_nodes + 3] = np.nan
    hin.copy_(torch.from_numpy(bad))
    rc = _lib().emrkc_step_host(h2.handle, 0.0, C.cast(hin.data_ptr(), C.POINTER(C.c_double)),
                                C.cast(hout.data_ptr(), C.POINTER(C.c_double)), hin.numel(),
                                w.dt, w.eps, 0, rF, rS, C.byref(rep))
    assert rc == capi.EMRKC_ENONFINITE and rep.abort_stage == 1
    assert np.array_equal(h2.get_state(), bad, equal_nan=True)
    h2.close()
    ref.close()
