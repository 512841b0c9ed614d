"""Run-loop events on grids that take several waves of blocks (and, for the
host step, several z-chunk launches): a norm guard or NumericalAbort raised
by early blocks must not stop later blocks of the same level
(kernels.h level_floor). The guard step's state is assigned in full
(P/src/simulate.cpp:222-227), so it must equal the oracle's everywhere, and
the per-call host step treats the guard as no event (it belongs to the run
loop) and returns the full step."""
import ctypes as C

import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _spiked(node_z):
    w = workloads.get("hh3d_128x128x128")
    p = w.problem
    y0 = w.initial_state()
    plane = int(p.n[0]) * int(p.n[1])
    y0[node_z * plane + 37 * int(p.n[0]) + 61] = 5e6  # V spike: |V| > 1e6 after the step
    return w, p, y0


@pytest.mark.parametrize("z", [0, 70])
@pytest.mark.parametrize("rho_S", [0.7, 30.0])  # s = 1 / s = 2 (the guard follows the last stage)
def test_norm_guard_multiwave(oracle, z, rho_S):
    w, p, y0 = _spiked(z)
    rF = 15.48
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(0, 3, w.dt, rF, rho_S, w.eps)
    yg = op.get_state()
    op.close()
    yo, ro, _ = oracle.run(p, y0, 0, 3, w.dt, w.eps, rF, rho_S)
    assert res.aborted and ro.aborted
    assert res.abort_kind == ro.abort_kind == capi.EMRKC_ABORT_NORM_GUARD
    assert (res.abort_step, res.steps_done, res.s, res.m) == \
        (ro.abort_step, ro.steps_done, ro.s, ro.m)
    assert (res.n_fF, res.n_fS, res.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    errs = rel_l2_blocks(oracle, p, yg, yo)
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("z", [0, 127])
def test_step_host_guard_chunks(oracle, z):
    """emrkc_step_host (pipelined over 8 z-chunk launches at 128^3, s = m = 1)
    with |V| > 1e6 in the first / last chunk: OK and the whole step."""
    import torch

    w, p, y0 = _spiked(z)
    lib = capi.load()
    rF, rS = 15.48, 0.7
    op = MonodomainOperator(p)
    n = y0.size
    hin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hin.numpy()[:] = y0
    rep = capi.StepReport()
    rc = lib.emrkc_step_host(op.handle, 0.0, C.cast(hin.data_ptr(), capi.DP),
                             C.cast(hout.data_ptr(), capi.DP), n, w.dt, w.eps, 0, rF, rS,
                             C.byref(rep))
    assert rc == capi.EMRKC_OK, lib.emrkc_last_error(op.handle).decode()
    yg = hout.numpy().copy()
    dev = op.get_state()
    op.close()
    yo, orep, orc = oracle.emrkc_step(p, 0.0, y0, w.dt, w.eps, rF, rS)
    assert orc == 0 and (rep.s, rep.m) == (orep.s, orep.m) == (1, 1)
    assert np.abs(yo[:p.n_nodes]).max() > 1e6  # the run loop's guard would fire
    assert max(rel_l2_blocks(oracle, p, yg, yo)) <= TOL
    np.testing.assert_array_equal(dev, yg)  # device state = the returned step


def test_step_host_aliasing_abort_keeps_input(oracle):
    """y_out == y_in and a NumericalAbort: the input survives (the reference
    throws before assigning y)."""
    import torch

    w = workloads.get("hh3d_128x128x128")
    p = w.problem
    y0 = w.initial_state()
    y0[p.n_nodes + 12345] = np.nan  # a gate: inner stage 1 fails
    lib = capi.load()
    op = MonodomainOperator(p)
    buf = torch.empty(y0.size, dtype=torch.float64, pin_memory=True)
    buf.numpy()[:] = y0
    ptr = C.cast(buf.data_ptr(), capi.DP)
    rep = capi.StepReport()
    rc = lib.emrkc_step_host(op.handle, 0.0, ptr, ptr, y0.size, w.dt, w.eps, 0, 15.48, 0.7,
                             C.byref(rep))
    op.close()
    assert rc == capi.EMRKC_ENONFINITE and rep.abort_stage == 1
    np.testing.assert_array_equal(buf.numpy(), y0)
