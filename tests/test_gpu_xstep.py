"""Cross-step fusion (k_step_x, EMRKC_XSTEP=1: inner stage 2 of step n and
the node update of step n + 1 in one launch) against the two-kernel step:
bitwise equal states and identical run records on grids that are no multiple
of the tile, with a stimulus box that splits pairs, nodes outside the fast
window, a norm guard and NumericalAborts in either half, through emrkc_run
and the bench's timed form. EMRKC_PAIR=2 forces the pair kernels on these
small grids."""
import ctypes as C

import numpy as np
import pytest

from paper_2401_01745_b200 import capi
from paper_2401_01745_b200.capi import RunResult, dptr
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu


def grid(n, h, stim_lo=(3, 2, 1), stim_hi=(9, 7, 6)):
    lo = [(i - 0.5) * h for i in stim_lo]
    hi = [(i + 0.5) * h for i in stim_hi]
    return make_problem(3, list(n), [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)


def state(oracle, p, seed=0, slow=True):
    y = oracle.initial_state(p)
    rng = np.random.default_rng(seed)
    y[: p.n_nodes] += rng.normal(0.0, 0.1, p.n_nodes)
    if slow:
        idx = rng.choice(p.n_nodes, 9, replace=False)
        y[idx] = -260.0
    return y


def run(p, y0, n, xs, monkeypatch, rF, rS, follow=0):
    monkeypatch.setenv("EMRKC_XSTEP", str(xs))
    monkeypatch.setenv("EMRKC_PAIR", "2")
    monkeypatch.setenv("EMRKC_PAIR_TX", "64")  # k_step_x works on 64 x 4 tiles
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(0, n, 0.05, rF, rS).as_dict()
    mode = capi.load().emrkc_fused_active(op.handle)
    res.pop("device_ms")
    y = op.get_state()
    y2 = None
    if follow:  # a second run continues from the first one's state
        op.run(n, follow, 0.05, rF, rS)
        y2 = op.get_state()
    op.close()
    return y, res, mode, y2


CASES = {"a": ((72, 18, 21), 0.1, 100.0, 0.7), "b": ((130, 10, 9), 0.1, 100.0, 0.7),
         "c": ((64, 8, 50), 0.1, 100.0, 0.7)}


@pytest.mark.parametrize("case", list(CASES))
def test_xstep_bitwise(oracle, case, monkeypatch):
    n, h, rF, rS = CASES[case]
    p = grid(n, h)
    y0 = state(oracle, p, 3)
    ya, ra, ma, ya2 = run(p, y0, 9, 1, monkeypatch, rF, rS, follow=2)
    yb, rb, mb, yb2 = run(p, y0, 9, 0, monkeypatch, rF, rS, follow=2)
    assert (ma, mb) == (3, 0) and ra["m"] == 2 and ra["s"] == 1
    assert ra == rb and ra["steps_done"] == 9
    assert np.array_equal(ya, yb)
    assert np.array_equal(ya2, yb2)


def test_xstep_events(oracle, monkeypatch):
    n, h, rF, rS = CASES["a"]
    p = grid(n, h)
    nn, plane = p.n_nodes, n[0] * n[1]
    y0 = state(oracle, p, 7, slow=False)
    yg = y0.copy()
    yg[plane * 9 + n[0] * 11 + 21] = 5e6  # norm guard (step 0, after its inner stage 2)
    a = run(p, yg, 5, 1, monkeypatch, rF, rS)
    b = run(p, yg, 5, 0, monkeypatch, rF, rS)
    assert a[1]["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD and a[1] == b[1]
    assert np.array_equal(a[0], b[0])
    yn = y0.copy()
    yn[2 * nn + plane * 15 + 5] = np.nan  # NumericalAbort in step 0's node level
    a = run(p, yn, 5, 1, monkeypatch, rF, rS)
    b = run(p, yn, 5, 0, monkeypatch, rF, rS)
    assert a[1]["abort_kind"] == capi.EMRKC_ABORT_NONFINITE and a[1] == b[1]
    assert np.array_equal(a[0], b[0], equal_nan=True)
    yl = y0.copy()
    yl[nn + plane * 4 + n[0] * 3 + 40] = 40.0  # a gate far out of range: blows up a few steps in
    a = run(p, yl, 12, 1, monkeypatch, rF, rS)
    b = run(p, yl, 12, 0, monkeypatch, rF, rS)
    assert a[1] == b[1]
    assert np.array_equal(a[0], b[0], equal_nan=True)


def test_xstep_timed_form(oracle, monkeypatch):
    """emrkc_run_timed (the bench's loop) with the fused launches: the same
    final state as emrkc_run, one non-zero entry per step after the first."""
    n, h, rF, rS = CASES["c"]
    p = grid(n, h)
    y0 = state(oracle, p, 5)
    monkeypatch.setenv("EMRKC_XSTEP", "1")
    monkeypatch.setenv("EMRKC_PAIR", "2")
    monkeypatch.setenv("EMRKC_PAIR_TX", "64")
    lib = capi.load()
    op = MonodomainOperator(p)
    op.set_state(y0)
    ms = np.zeros(2 * 7)
    res = RunResult()
    rc = lib.emrkc_run_timed(op.handle, 0, 7, 0.05, 0.05, 0, rF, rS, 1 << 20, dptr(ms), ms.size,
                             C.byref(res))
    assert rc == 0 and lib.emrkc_fused_active(op.handle) == 3
    yt = op.get_state()
    op.close()
    yr, rr, _, _ = run(p, y0, 7, 0, monkeypatch, rF, rS)
    assert np.array_equal(yt, yr)
    assert res.steps_done == rr["steps_done"] == 7
    assert ms[0] > 0 and (ms[1::2] > 0).all() and (ms[2::2] < 0.01).all()
