"""k_node_pair (pair-per-thread node kernel, the default on large 3-D whole
grids) against k_node_tma: bitwise equal states and identical run records on
grids whose sizes are not multiples of the 64 x 4 tile, with a stimulus box
that splits pairs, nodes outside the fast ionic window (reference-order
path), m = 1 / m = 2 / forced s = 2, a norm guard and a NumericalAbort.
EMRKC_PAIR=2 forces the kernel on these small grids."""
import numpy as np
import pytest

from paper_2401_01745_b200 import capi
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
    if slow:  # a few nodes below the fast window (about -208 mV at eta 0.05)
        idx = rng.choice(p.n_nodes, 9, replace=False)
        y[idx] = -260.0
    return y


def run(p, y0, n, pair, monkeypatch, rF, rS, per_step=False):
    monkeypatch.setenv("EMRKC_PAIR", str(pair))
    monkeypatch.setenv("EMRKC_RESIDENT", "0")
    op = MonodomainOperator(p)
    op.set_state(y0)
    if per_step:
        for k in range(n):
            op.step(k * 0.05, 0.05, rF, rS)
        res = None
    else:
        res = op.run(0, n, 0.05, rF, rS).as_dict()
        res.pop("device_ms")
    y = op.get_state()
    op.close()
    return y, res


CASES = {
    # name: (n, h, rho_F, rho_S, steps)
    "m1": ((40, 22, 18), 0.25, 16.0, 0.7, 10),
    "m2": ((72, 18, 21), 0.1, 100.0, 0.7, 8),
    "s2m2": ((66, 12, 17), 0.05, 390.0, 50.0, 6),
    "m4_tb": ((130, 20, 24), 0.05, 390.0, 0.7, 6),
}


@pytest.mark.parametrize("case", list(CASES))
def test_pair_bitwise(oracle, case, monkeypatch):
    n, h, rF, rS, steps = CASES[case]
    p = grid(n, h)
    y0 = state(oracle, p, 3)
    ya, ra = run(p, y0, steps, 2, monkeypatch, rF, rS)
    yb, rb = run(p, y0, steps, 0, monkeypatch, rF, rS)
    assert ra == rb and ra["steps_done"] == steps
    assert np.array_equal(ya, yb)
    ya, _ = run(p, y0, 3, 2, monkeypatch, rF, rS, per_step=True)
    yb, _ = run(p, y0, 3, 0, monkeypatch, rF, rS, per_step=True)
    assert np.array_equal(ya, yb)


def test_pair_against_oracle(oracle, monkeypatch):
    n, h, rF, rS, steps = CASES["m2"]
    p = grid(n, h)
    y0 = state(oracle, p, 5, slow=False)
    y, r = run(p, y0, steps, 2, monkeypatch, rF, rS)
    yo, ro, _ = oracle.run(p, y0, 0, steps, 0.05, 0.05, rF, rS)
    assert (r["s"], r["m"]) == (ro.s, ro.m)
    nn = p.n_nodes
    for b in range(4):
        assert oracle.rel_l2(p, y[b * nn:(b + 1) * nn], yo[b * nn:(b + 1) * nn]) <= 1e-9


def test_pair_events(oracle, monkeypatch):
    n, h, rF, rS, _ = CASES["m1"]
    p = grid(n, h)
    plane = n[0] * n[1]
    y0 = state(oracle, p, 7, slow=False)
    yg = y0.copy()
    yg[plane * 9 + n[0] * 11 + 21] = 5e6  # norm guard
    a = run(p, yg, 4, 2, monkeypatch, rF, rS)
    b = run(p, yg, 4, 0, monkeypatch, rF, rS)
    assert a[1]["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD and a[1] == b[1]
    assert np.array_equal(a[0], b[0])
    yn = y0.copy()
    yn[2 * p.n_nodes + plane * 15 + 5] = np.nan  # NumericalAbort (gate h)
    a = run(p, yn, 4, 2, monkeypatch, rF, rS)
    b = run(p, yn, 4, 0, monkeypatch, rF, rS)
    assert a[1]["abort_kind"] == capi.EMRKC_ABORT_NONFINITE and a[1] == b[1]
    assert np.array_equal(a[0], b[0], equal_nan=True)


def test_pair_gate_range_irregular(oracle, monkeypatch):
    """Gate range with values outside (0, 1): a negative gate in the initial
    state disables the high-word prefilter (the earlier range is not
    positive); a gate that turns negative during the run must reach the
    exact path. Records (gate_min / gate_max) bitwise k_node_tma's, and the
    oracle's to rounding level."""
    n, h, rF, rS, _ = CASES["m1"]
    p = grid(n, h)
    nn, plane = p.n_nodes, n[0] * n[1]
    for tweak in ("neg_initial", "neg_later", "big_later"):
        y0 = state(oracle, p, 9, slow=False)
        if tweak == "neg_initial":
            y0[nn + plane * 3 + 17] = -0.02
        elif tweak == "neg_later":
            y0[3 * nn + plane * 8 + n[0] * 5 + 9] = 1e-7  # n gate: relaxes through tiny values
            y0[plane * 8 + n[0] * 5 + 9] = -95.0
        else:
            y0[2 * nn + plane * 12 + n[0] * 3 + 30] = 1.5
        a = run(p, y0, 6, 2, monkeypatch, rF, rS)
        b = run(p, y0, 6, 0, monkeypatch, rF, rS)
        assert a[1] == b[1], tweak
        assert np.array_equal(a[0], b[0])
        _, ro, _ = oracle.run(p, y0, 0, 6, 0.05, 0.05, rF, rS)
        # against the oracle: rounding-level differences of the fast path only
        assert a[1]["gate_min"] == pytest.approx(ro.gate_min, rel=1e-9, abs=1e-12), tweak
        assert a[1]["gate_max"] == pytest.approx(ro.gate_max, rel=1e-9, abs=1e-12), tweak
