"""The SYNTHETIC width stand-in (EMRKC_MODEL_HH_AUX, include/emrkc.h: HH plus
n_aux passive auxiliary variables, the CRN / TTP state widths N = 21 / 19 of
configs 3 / 4; SURVEY §8(c) option 2, no physiology claim) on the device
against the plain-C oracle, whose restatement of the model is pinned bit for
bit against the reference's own generic machinery running the same model
(tests/test_oracle_vs_ref.py::test_synthetic_width_bitwise), and against
the reference's run record on config 3's grid at width 21."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-9


def prob(dim, n_aux):
    h = 0.25  # rho_F ~ 23 (3-D), ~18 (2-D)
    if dim == 3:
        return make_problem(3, [40, 24, 18], [h] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0,
                            [-0.125] * 3, [0.875] * 3, 0.0, 1.0, n_aux=n_aux)
    return make_problem(2, [136, 40], [h] * 2, [0.2, 0.2], 140.0, 0.01, 70.0,
                        [-0.125] * 2, [1.875] * 2, 0.0, 1.0, n_aux=n_aux)


def noisy(oracle, p, seed=0):
    y = oracle.initial_state(p)
    return y * np.random.default_rng(seed).uniform(0.99, 1.01, y.size)


@pytest.mark.parametrize("n_aux", [15, 17])
def test_operator_and_rho_bitwise(oracle, n_aux):
    p = prob(3, n_aux)
    y = noisy(oracle, p)
    op = MonodomainOperator(p)
    assert op.len == p.state_len() == (4 + n_aux) * p.n_nodes
    np.testing.assert_array_equal(op.initial_state(), oracle.initial_state(p))
    for which in (0, 1):
        assert np.array_equal(op.f_F(0.5, y) if which == 0 else op.f_S(0.5, y),
                              oracle.rhs(p, which, 0.5, y))
    lam, yinf = op.exp_part(y)
    rl, ri = oracle.exp_part(p, y)
    np.testing.assert_allclose(lam, rl, rtol=1e-14, atol=0)
    np.testing.assert_allclose(yinf, ri, rtol=1e-14, atol=1e-300)
    op.set_state(y)
    for which in (0, 1):
        got = op.estimate_spectral_radius(which, 0.0)
        ref, _ = oracle.estimate_rho(p, which, 0.0, y)
        assert (got.rho, got.iterations) == (ref.rho, ref.iterations)
    op.close()


@pytest.mark.parametrize("dim,n_aux,rF,rS,n", [(3, 15, 25.0, 0.7, 12), (3, 17, 100.0, 0.7, 8),
                                               (3, 15, 390.0, 50.0, 6), (2, 17, 20.0, 0.7, 10)])
def test_runs_against_oracle(oracle, dim, n_aux, rF, rS, n):
    """s = 1 / m = 1, s = 1 / m = 2 (node kernel + inner stage), forced
    s = 2 / m = 2 (outer stages j >= 2), 2-D; emrkc_run and emrkc_step."""
    p = prob(dim, n_aux)
    y0 = noisy(oracle, p, 1)
    op = MonodomainOperator(p)
    op.set_state(y0)
    res = op.run(0, n, 0.05, rF, rS)
    y = op.get_state()
    op.set_state(y0)
    for k in range(n):
        op.step(k * 0.05, 0.05, rF, rS)
    y_step = op.get_state()
    op.close()
    yo, ro, _ = oracle.run(p, y0, 0, n, 0.05, 0.05, rF, rS)
    assert (res.s, res.m, res.aborted) == (ro.s, ro.m, ro.aborted) and not ro.aborted
    assert (res.n_fF, res.n_fS, res.n_exp) == (ro.n_fF, ro.n_fS, ro.n_exp)
    assert abs(res.gate_min - ro.gate_min) <= TOL and abs(res.gate_max - ro.gate_max) <= TOL
    errs = rel_l2_blocks(oracle, p, y, yo)
    assert len(errs) == 4 + n_aux and max(errs) <= TOL, errs
    assert np.array_equal(y, y_step)


def test_step_host_and_slabs(oracle, monkeypatch):
    """The pipelined host step moves every field; z-slab groups are bitwise
    the whole grid with the aux fields."""
    import ctypes as C

    import torch

    from paper_2401_01745_b200.capi import Partition, RunResult, load

    p = make_problem(3, [64, 40, 48], [0.1] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0,
                     [-0.05] * 3, [0.75] * 3, 0.0, 1.0, n_aux=15)
    y0 = noisy(oracle, p, 2)
    lib = load()
    whole = MonodomainOperator(p)
    whole.set_state(y0)
    whole.step(0.0, 0.05, 145.0, 0.7)  # rho_F ~ 143 at h = 0.1: m = 2
    yw = whole.get_state()
    hin = torch.from_numpy(y0.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    rep = capi.StepReport()
    assert lib.emrkc_step_host(whole.handle, 0.0, C.cast(hin.data_ptr(), capi.DP),
                               C.cast(hout.data_ptr(), capi.DP), hin.numel(), 0.05, 0.05, 0,
                               145.0, 0.7, C.byref(rep)) == 0
    assert rep.m == 2 and np.array_equal(hout.numpy(), yw)
    whole.set_state(y0)
    rw = whole.run(0, 6, 0.05, 145.0, 0.7)
    yw = whole.get_state()
    whole.close()
    nn, plane, nf = p.n_nodes, 64 * 40, p.n_fields
    ops, hs = [], []
    for z0, z1 in [(0, 17), (17, 30), (30, 48)]:
        part = Partition(z0, z1)
        o = MonodomainOperator(p, 0, part)
        o.set_state(np.concatenate([y0[b * nn + z0 * plane: b * nn + z1 * plane]
                                    for b in range(nf)]))
        ops.append((o, z0, z1))
        hs.append(o.handle)
    grp = C.c_void_p()
    arr = (C.c_void_p * 3)(*hs)
    assert lib.emrkc_group_create(arr, 3, C.byref(grp)) == 0
    res = RunResult()
    assert lib.emrkc_group_run(grp, 0, 6, 0.05, 0.05, 0, 145.0, 0.7, C.byref(res)) == 0
    lib.emrkc_group_destroy(grp)
    full = np.empty_like(yw)
    for o, z0, z1 in ops:
        ys = o.get_state()
        m = (z1 - z0) * plane
        for b in range(nf):
            full[b * nn + z0 * plane: b * nn + z1 * plane] = ys[b * m:(b + 1) * m]
        o.close()
    assert (res.s, res.m, res.n_fF) == (rw.s, rw.m, rw.n_fF)
    assert np.array_equal(full, yw)


def test_unsupported_methods_fail_loudly(oracle):
    p = prob(3, 15)
    op = MonodomainOperator(p)
    op.set_state(oracle.initial_state(p))
    with pytest.raises(ValueError):
        op.exex_step(0.0, 0.01)
    op.close()
