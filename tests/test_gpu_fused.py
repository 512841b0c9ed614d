"""The fused s = 1, m = 2 step (k_fused2: node update, inner stage 2 and the
outer update in one persistent pass, d_1 tile edges exchanged between
co-resident blocks through L2) against the two-kernel step
(EMRKC_FUSED=0: k_node_tma + k_vin_tma_r, itself parity-tested against the
oracle): bitwise equal states and identical run records (abort step /
kind / stage, counters, gate range), on tile plans with one and several
z-chunks, with the stimulus window, nodes outside the fast ionic window,
a norm guard and a NumericalAbort; plus the oracle directly."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu

H = 0.1


@pytest.fixture(scope="module", autouse=True)
def _needs_k_fused2():
    """k_fused2 is measured slower than the two-kernel step and compiled only
    with -DEMRKC_EXPERIMENTAL=1 (tools/build_variant.sh exp
    -DEMRKC_EXPERIMENTAL=1; EMRKC_LIB=build_var/lib_exp.so): skip without it."""
    import os

    old = os.environ.get("EMRKC_FUSED")
    os.environ["EMRKC_FUSED"] = "1"
    try:
        lo, hi = [-0.05] * 3, [0.75] * 3
        p = make_problem(3, [256, 192, 40], [H] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0, lo, hi,
                         0.0, 1.0)
        op = MonodomainOperator(p)
        op.set_state(op.initial_state())
        op.run(0, 1, 0.05, 60.0, 0.7)
        active = capi.load().emrkc_fused_active(op.handle)
        op.close()
    finally:
        if old is None:
            os.environ.pop("EMRKC_FUSED", None)
        else:
            os.environ["EMRKC_FUSED"] = old
    if active != 1:
        pytest.skip("k_fused2 not built (-DEMRKC_EXPERIMENTAL=1)")


def grid(nx, ny, nz, sigma=(0.3, 0.1, 0.1), stim_lo=(10, 12, 3), stim_hi=(17, 19, 8)):
    lo = [(i - 0.5) * H for i in stim_lo]
    hi = [(i + 0.5) * H for i in stim_hi]
    return make_problem(3, [nx, ny, nz], [H] * 3, list(sigma), 140.0, 0.01, 70.0, lo, hi, 0.0, 1.0)


def state(oracle, p, seed=0):
    y = oracle.initial_state(p)
    y[: p.n_nodes] += np.random.default_rng(seed).normal(0.0, 0.1, p.n_nodes)
    return y


def run(p, y0, nsteps, fused, monkeypatch, rF=60.0, rS=0.7, step0=0):
    monkeypatch.setenv("EMRKC_FUSED", "1" if fused else "0")
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(step0, nsteps, 0.05, rF, rS)
    active = capi.load().emrkc_fused_active(op.handle)
    y = op.get_state()
    op.close()
    return y, res.as_dict(), active


SHAPES = [(256, 192, 40), (128, 96, 64), (192, 160, 33)]


@pytest.mark.parametrize("shape", SHAPES)
def test_fused_bitwise_vs_two_kernels(oracle, shape, monkeypatch):
    p = grid(*shape)
    y0 = state(oracle, p)
    yf, rf, af = run(p, y0, 30, True, monkeypatch)
    yu, ru, au = run(p, y0, 30, False, monkeypatch)
    assert (af, au) == (1, 0)
    assert (rf["s"], rf["m"]) == (1, 2)
    rf.pop("device_ms")
    ru.pop("device_ms")
    assert rf == ru
    assert np.array_equal(yf, yu)


def test_fused_vs_oracle(oracle, monkeypatch):
    p = grid(128, 96, 64)
    y0 = state(oracle, p, 3)
    yf, rf, af = run(p, y0, 12, True, monkeypatch)
    yo, ro, _ = oracle.run(p, y0, 0, 12, 0.05, 0.05, 60.0, 0.7)
    assert af == 1 and (rf["s"], rf["m"]) == (ro.s, ro.m) == (1, 2)
    assert max(rel_l2_blocks(oracle, p, yf, yo)) <= 1e-9


def test_fused_slow_window_and_events(oracle, monkeypatch):
    p = grid(256, 192, 40)
    nn = p.n_nodes
    plane = 256 * 192
    y0 = state(oracle, p, 1)
    # nodes outside the fast ionic window (V < ~-208 mV at eta 0.05)
    for k, i in enumerate([5, 64 * 3 + 17, plane * 7 + 255, plane * 39 + 256 * 191 + 3]):
        y0[i] = -250.0 - 10.0 * k
    yf, rf, _ = run(p, y0, 6, True, monkeypatch)
    yu, ru, _ = run(p, y0, 6, False, monkeypatch)
    rf.pop("device_ms")
    ru.pop("device_ms")
    assert rf == ru and np.array_equal(yf, yu)
    # norm guard: |V| > 1e6 after the step, state assigned
    yg = y0.copy()
    yg[plane * 20 + 256 * 100 + 128] = 5e6
    yf, rf, _ = run(p, yg, 4, True, monkeypatch)
    yu, ru, _ = run(p, yg, 4, False, monkeypatch)
    assert rf["aborted"] and rf["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD
    rf.pop("device_ms")
    ru.pop("device_ms")
    assert rf == ru and np.array_equal(yf, yu)
    # NumericalAbort in inner stage 1 (a NaN gate), the pre-step state kept
    yn = y0.copy()
    yn[nn + plane * 30 + 77] = np.nan
    yf, rf, _ = run(p, yn, 4, True, monkeypatch)
    yu, ru, _ = run(p, yn, 4, False, monkeypatch)
    assert rf["aborted"] and rf["abort_kind"] == capi.EMRKC_ABORT_NONFINITE
    rf.pop("device_ms")
    ru.pop("device_ms")
    assert rf == ru
    assert np.array_equal(yf, yu, equal_nan=True)


@pytest.mark.slow
def test_fused_config4_grid(monkeypatch):
    """Config 4's grid (512 x 512 x 256, the bench headline), 8 steps."""
    from paper_2401_01745_b200 import workloads

    w = workloads.get("hh3d_512x512x256")
    y0 = w.initial_state()
    yf, rf, af = run(w.problem, y0, 8, True, monkeypatch, 139.0046116240814, 0.711397268929107)
    yu, ru, _ = run(w.problem, y0, 8, False, monkeypatch, 139.0046116240814, 0.711397268929107)
    assert af == 1
    rf.pop("device_ms")
    ru.pop("device_ms")
    assert rf == ru and np.array_equal(yf, yu)
