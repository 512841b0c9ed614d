"""The z-pipelined step (EMRKC_ZPIPE=K: node-kernel z-chunks on the
handle's stream, the inner-stage chunks on a second stream behind them)
against the unpipelined step: bitwise equal states and identical run
records, for m = 2 and m = 4, with the stimulus, a norm guard and a
NumericalAbort, through emrkc_run, emrkc_step and the bench's timed form."""
import numpy as np
import pytest

from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu


def grid(nx, ny, nz, h=0.1):
    lo = [(i - 0.5) * h for i in (10, 12, 3)]
    hi = [(i + 0.5) * h for i in (17, 19, 8)]
    return make_problem(3, [nx, ny, nz], [h] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0, lo, hi,
                        0.0, 1.0)


def state(oracle, p, seed=0):
    y = oracle.initial_state(p)
    y[: p.n_nodes] += np.random.default_rng(seed).normal(0.0, 0.1, p.n_nodes)
    return y


def run(p, y0, n, K, monkeypatch, rF, rS=0.7, step_after=True):
    monkeypatch.setenv("EMRKC_ZPIPE", str(K))
    monkeypatch.setenv("EMRKC_TB", "0")  # the z-pipelined step chains per-stage inner kernels
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(0, n, 0.05, rF, rS).as_dict()
    mode = capi.load().emrkc_fused_active(op.handle)
    y = op.get_state()
    y2 = None
    if step_after:  # emrkc_step after the run
        op.step(n * 0.05, 0.05, rF, rS)
        y2 = op.get_state()
    op.close()
    res.pop("device_ms")
    return y, y2, res, mode


@pytest.mark.parametrize("rF,m", [(60.0, 2), (500.0, 4)])
def test_zpipe_bitwise(oracle, rF, m, monkeypatch):
    p = grid(96, 80, 72)
    y0 = state(oracle, p)
    yz, yz2, rz, mz = run(p, y0, 25, 8, monkeypatch, rF)
    yu, yu2, ru, mu = run(p, y0, 25, 0, monkeypatch, rF)
    assert (mz, mu) == (2, 0) and rz["m"] == m
    assert rz == ru
    assert np.array_equal(yz, yu) and np.array_equal(yz2, yu2)


def test_zpipe_events(oracle, monkeypatch):
    p = grid(96, 80, 72)
    plane = 96 * 80
    y0 = state(oracle, p, 2)
    yg = y0.copy()
    yg[plane * 40 + 96 * 30 + 50] = 5e6  # norm guard in a middle chunk
    a = run(p, yg, 4, 8, monkeypatch, 60.0, step_after=False)
    b = run(p, yg, 4, 0, monkeypatch, 60.0, step_after=False)
    assert a[2]["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD and a[2] == b[2]
    assert np.array_equal(a[0], b[0])
    yn = y0.copy()
    yn[p.n_nodes + plane * 70 + 5] = np.nan  # NumericalAbort in the last chunk
    a = run(p, yn, 4, 8, monkeypatch, 60.0, step_after=False)
    b = run(p, yn, 4, 0, monkeypatch, 60.0, step_after=False)
    assert a[2]["abort_kind"] == capi.EMRKC_ABORT_NONFINITE and a[2] == b[2]
    assert np.array_equal(a[0], b[0], equal_nan=True)


def test_zpipe_timed_form(monkeypatch):
    """emrkc_run_timed (the bench's timed loop) with the z-pipelined step:
    the same final state as emrkc_run."""
    import ctypes as C

    from paper_2401_01745_b200.capi import RunResult, dptr

    w = workloads.get("hh3d_sweep_100")  # m = 2, s = 1
    y0 = w.initial_state()
    monkeypatch.setenv("EMRKC_ZPIPE", "8")
    lib = capi.load()
    op = MonodomainOperator(w.problem)
    op.set_state(y0)
    rF, rS = 96.74305633668402, 0.7113972689294705
    ms = np.zeros(2 * 10)
    res = RunResult()
    assert lib.emrkc_run_timed(op.handle, 0, 10, w.dt, w.eps, 0, rF, rS, 0, dptr(ms), ms.size,
                               C.byref(res)) == 0
    assert lib.emrkc_fused_active(op.handle) == 2
    y_t = op.get_state()
    assert np.all(ms[0::2] > 0) and np.all(ms[1::2] < 0.05 * ms[0::2])
    op.set_state(y0)
    op.run(0, 10, w.dt, rF, rS, w.eps)
    assert np.array_equal(op.get_state(), y_t)
    op.close()
