"""The reference's known-answer tests run THROUGH THE PRODUCT: the generic
integrator layer of include/emrkc.h (rkc_iteration, exponential Euler,
averaged forces, emrkc_step / mrkc_step over a SplitRhs, the power
iteration) on the device, with the reference's scalar surrogate problems
(P/tests/test_multirate.cpp:54-66) as callbacks. Constants and tolerances
are the reference tests' own (file:line below); where oracle/_ref is built,
results are also compared with the reference's own functions.

Plus the grid problem through the same generic layer (emrkc_bind_split_rhs:
the handle's f_F / f_S / exp_part as device callbacks) against the oracle
and against the fused emrkc_step kernels."""
import math

import numpy as np
import pytest

from paper_2401_01745_b200 import capi
from paper_2401_01745_b200 import integrators as I
from paper_2401_01745_b200.monodomain import MonodomainOperator, NumericalAbort, make_problem

pytestmark = pytest.mark.gpu


def phi(z):  # P/src/multirate.cpp:42-47
    if abs(z) < 1e-5:
        return 1.0 + z * (0.5 + z * (1.0 / 6.0 + z / 24.0))
    return math.expm1(z) / z


def scalar_split(lF, lS, lE=0.0, yinf=0.0, with_exp=True):
    """P/tests/test_multirate.cpp:54-66"""
    return I.GenericSplitRhs(lambda t, y: lF * y, lambda t, y: lS * y,
                             (lambda y: (np.array([lE]), np.array([yinf]))) if with_exp else None,
                             abs(lF), abs(lS))


def R(s, eps, z):
    return I.stability_poly(s, eps, z)


def stability_phi(s, eps, z):  # P/src/cheb.cpp:120-131
    if abs(z) < 1e-8:
        h = 1e-5
        rpp = (R(s, eps, h) - 2.0 + R(s, eps, -h)) / (h * h)
        return 1.0 + 0.5 * rpp * z
    return (R(s, eps, z) - 1.0) / z


# ---- cheb (P/tests/test_cheb.cpp) -------------------------------------------

def test_rkc_iteration_kats():
    y = np.array([1.5, -2.0, 0.25])
    for s in (1, 3, 9):  # :111-117
        out = I.rkc_iteration(0.0, y, 0.7, lambda t, u: np.zeros_like(u), s, 0.05)
        np.testing.assert_allclose(out, y, rtol=1e-14)
    ev = [0]

    def counted(lam):
        def f(t, u):
            ev[0] += 1
            return lam * u
        return f

    out = I.rkc_iteration(0.0, [2.0], 0.3, counted(-4.0), 1, 0.05)  # :118-124
    assert out[0] == pytest.approx(2.0 * (1.0 - 1.2), rel=1e-14) and ev[0] == 1
    ev[0] = 0
    out = I.rkc_iteration(0.0, [1.0], 1.0, counted(-1.0), 2, 0.0)  # :125-131
    assert out[0] == pytest.approx(0.125, rel=1e-14) and ev[0] == 2
    for s in (1, 2, 5, 17):  # :132-138
        ev[0] = 0
        I.rkc_iteration(0.0, [1.0], 1e-3, counted(-1.0), s, 0.05)
        assert ev[0] == s
    with pytest.raises(NumericalAbort) as ei:  # :139-149
        I.rkc_iteration(0.0, [1.0], 1.0, lambda t, u: np.full_like(u, np.inf), 3, 0.05)
    assert "stage 1" in str(ei.value) and ei.value.stage == 1
    times = []  # :150-160

    def probe(t, u):
        times.append(t)
        return np.zeros_like(u)

    I.rkc_iteration(10.0, [1.0], 2.0, probe, 4, 0.05)
    from paper_2401_01745_b200.monodomain import rkc_coeffs

    c = rkc_coeffs(4, 0.05).c
    assert len(times) == 4
    for j in range(4):
        assert times[j] == pytest.approx(10.0 + c[j] * 2.0, rel=1e-15)


def test_stability_polynomial():
    """R_s(0) = 1; R_2 with eps = 0 is 1 + z + z^2/8; |R_s| <= 1 on the
    damped interval; R_s(z) = T_s(w0 + w1 z) / T_s(w0) (the closed form of
    the damped RKC polynomial) to 1e-14 (P/tests/test_cheb.cpp:168-223)."""
    from paper_2401_01745_b200.monodomain import rkc_coeffs

    for s in (1, 2, 7, 23, 50):  # :169-172
        assert abs(R(s, 0.05, 0.0) - 1.0) < 1e-12
    for z in (-0.5, -2.0, -7.9):
        assert R(2, 0.0, z) == pytest.approx(1 + z + z * z / 8, rel=1e-14, abs=1e-14)
    rng = np.random.default_rng(3)
    for _ in range(40):
        s = int(rng.integers(1, 30))
        k = rkc_coeffs(s, 0.05)
        beta = 2 - 4 * 0.05 / 3
        z = -beta * s * s * rng.random()
        T = np.polynomial.chebyshev.Chebyshev.basis(s)
        closed = T(k.omega0 + k.omega1 * z) / T(k.omega0)
        got = R(s, 0.05, z)
        assert abs(got) <= 1.0 + 1e-12
        assert got == pytest.approx(closed, rel=1e-12, abs=1e-14)


def test_rkc_iteration_matches_reference(reference):
    rng = np.random.default_rng(7)
    for _ in range(60):  # P/tests/test_cheb.cpp:206-223 style, bitwise to the reference
        s = int(rng.integers(1, 21))
        beta = 2 - 4 * 0.05 / 3
        z = -beta * s * s * rng.random()
        dt = 0.25 + rng.random()
        lam = z / dt
        y0 = 1.0 + rng.random()
        a = reference.rkc_iteration_scalar(0.0, y0, dt, lam, s, 0.05)
        b = I.rkc_iteration(0.0, [y0], dt, lambda t, y: lam * y, s, 0.05)
        assert a == b[0]


# ---- multirate (P/tests/test_multirate.cpp) ---------------------------------

def test_exponential_euler():
    out = I.exponential_euler_step([1.0], 0.5, [-2.0], [0.25])  # :28-32
    assert out[0] == pytest.approx(0.25 + 0.75 * math.exp(-1.0), rel=1e-15)
    y = np.array([0.3, -1.2, 7.0])
    assert np.array_equal(I.exponential_euler_step(y, 0.5, [0, 0, 0], [0, 0, 0]), y)
    y = np.array([0.6, 0.2])
    assert np.array_equal(I.exponential_euler_step(y, 3.0, [-5.0, -1.0], y), y)
    rng = np.random.default_rng(5)  # :37-49: gates stay in [0, 1]
    n = 200
    y, zi, lam = rng.random(n), rng.random(n), -50.0 * rng.random(n)
    out = I.exponential_euler_step(y, 2.0 * rng.random(), lam, zi)
    assert np.all(out >= 0.0) and np.all(out <= 1.0)


def test_averaged_force_mrkc_kats():
    rhs = scalar_split(-10.0, -1.0, with_exp=False)
    f = I.averaged_force_mrkc(0.0, [1.0], 0.1, rhs, 1, 0.05)  # :70-74
    assert f[0] == pytest.approx(-11.0, rel=1e-13)
    f = I.averaged_force_mrkc(0.0, [2.0], 0.1, scalar_split(0.0, 0.0, with_exp=False), 3, 0.05)
    assert abs(f[0]) < 1e-13  # :75-79
    f = I.averaged_force_mrkc(0.0, [1.0], 0.1, rhs, 2, 0.05)  # :80-85
    assert f[0] == pytest.approx(stability_phi(2, 0.05, -1.0) * -11.0, rel=1e-13)
    rhs = scalar_split(-10.0, -1.0, with_exp=False)  # :86-93
    I.averaged_force_mrkc(0.0, [1.0], 0.1, rhs, 5, 0.05)
    assert rhs.counters["n_fS"] == 1 and rhs.counters["n_fF"] == 5


def test_averaged_force_emrkc_kats(reference):
    rhs = scalar_split(-10.0, -1.0, -5.0)  # :97-106
    f = I.averaged_force_emrkc(0.0, [1.0], 0.1, rhs, 1)[0]
    assert f == pytest.approx(-11.0 * math.exp(-0.5) + phi(-0.5) * -5.0, rel=1e-13)
    assert f == pytest.approx(-10.60653, rel=1e-6)
    assert f == pytest.approx(reference.averaged_force_emrkc(-10.0, -1.0, -5.0, 0.0, 1.0, 0.1, 1),
                              rel=1e-15)
    f = I.averaged_force_emrkc(0.0, [1.0], 0.1, scalar_split(0.0, 0.0, -5.0), 1)[0]  # :124-131
    assert f == pytest.approx(phi(-0.5) * -5.0, rel=1e-13)
    assert f == pytest.approx(-3.934693, rel=1e-6)
    rng = np.random.default_rng(11)  # :107-123: lambda_E = 0 reduces to mRKC
    for _ in range(25):
        rhs = scalar_split(-20.0 * rng.random(), -2.0 * rng.random(), 0.0, rng.random())
        m = 1 + int(rng.integers(0, 4))
        y = [1.0 + rng.random()]
        a = I.averaged_force_emrkc(0.0, y, 0.05, rhs, m)[0]
        b = I.averaged_force_mrkc(0.0, y, 0.05, rhs, m)[0]
        assert a == pytest.approx(b, rel=1e-14)
    rhs = scalar_split(-8.0, -0.5, 0.0, 0.7)  # :132-140
    a = I.averaged_force_emrkc(0.0, [1.3], 0.1, rhs, 2, capi.EMRKC_VARIANT_STANDARD)[0]
    b = I.averaged_force_emrkc(0.0, [1.3], 0.1, rhs, 2, capi.EMRKC_VARIANT_PROGRESSIVE)[0]
    assert a == pytest.approx(b, rel=1e-15)
    rhs = scalar_split(-10.0, -1.0, -2.0)  # :141-150
    I.averaged_force_emrkc(0.0, [1.0], 0.1, rhs, 3)
    assert rhs.counters == {"n_fF": 3, "n_fS": 1, "n_exp_steps": 1}
    with pytest.raises(ValueError):  # m >= 1, exp_part required
        I.averaged_force_emrkc(0.0, [1.0], 0.1, scalar_split(-1.0, -1.0), 0)
    with pytest.raises(ValueError):
        I.averaged_force_emrkc(0.0, [1.0], 0.1, scalar_split(-1.0, -1.0, with_exp=False), 1)


def test_mrkc_step_kats():
    out, rep = I.mrkc_step(0.0, [3.0], 1.0, scalar_split(0.0, 0.0, with_exp=False))  # :154-161
    assert out[0] == 3.0 and (rep.s, rep.m) == (1, 1)
    rng = np.random.default_rng(13)  # :162-177
    for _ in range(40):
        lF = -10 ** (4 * rng.random())
        lS = -10 ** (1.5 * rng.random())
        dt = 10 ** (-2 + 3 * rng.random())
        out, rep = I.mrkc_step(0.0, [1.0], dt, scalar_split(lF, lS, with_exp=False))
        inner = stability_phi(rep.m, 0.05, rep.eta * lF) * (lF + lS)
        assert out[0] == pytest.approx(R(rep.s, 0.05, dt * inner), rel=1e-12, abs=1e-300)
    rhs = scalar_split(-500.0, -3.0, with_exp=False)  # :178-188
    out, rep = I.mrkc_step(0.0, [1.0], 0.5, rhs)
    assert rep.eta == pytest.approx(2 * 0.5 / rep.ell_s, rel=1e-14)
    assert rep.eta * rhs.rho_F <= rep.ell_m + 1e-12
    assert rhs.counters["n_fS"] == rep.s and rhs.counters["n_fF"] == rep.s * rep.m
    assert rep.n_fS == rep.s and rep.n_fF == rep.s * rep.m


def test_emrkc_step_kats(reference):
    out, _ = I.emrkc_step(0.0, [3.0], 1.0, scalar_split(0.0, 0.0, 0.0))  # :192-196
    assert out[0] == 3.0
    rng = np.random.default_rng(17)  # :197-214
    for _ in range(40):
        lF = -10 ** (4 * rng.random())
        lS = -10 ** (1.5 * rng.random())
        lE = -10 ** (3 * rng.random())
        dt = 10 ** (-2 + 3 * rng.random())
        out, rep = I.emrkc_step(0.0, [1.0], dt, scalar_split(lF, lS, lE))
        inner = (stability_phi(rep.m, 0.05, rep.eta * lF) * (lF + lS) * math.exp(rep.eta * lE)
                 + phi(rep.eta * lE) * lE)
        assert out[0] == pytest.approx(R(rep.s, 0.05, dt * inner), rel=1e-12, abs=1e-300)
        ref, s, m, eta = reference.emrkc_step_scalar(lF, lS, lE, 0.0, 1.0, dt)
        assert (rep.s, rep.m, rep.eta) == (s, m, eta)
        assert out[0] == pytest.approx(ref, rel=1e-13, abs=1e-300)
    out, rep = I.emrkc_step(0.0, [1.0], 0.8, scalar_split(0.0, 0.0, -4.0, 0.25), 0.0)  # :215-228
    assert (rep.s, rep.m) == (1, 1)
    assert out[0] == pytest.approx(0.25 + 0.75 * math.exp(0.8 * -4.0), rel=1e-12)
    with pytest.raises(ValueError):  # :229-233
        I.emrkc_step(0.0, [1.0], 0.1, scalar_split(-1.0, -1.0, with_exp=False))
    with pytest.raises(ValueError):
        I.emrkc_step(0.0, [1.0], 0.0, scalar_split(-1.0, -1.0))


# ---- spectral (P/tests/test_spectral.cpp) ------------------------------------

def test_spectral_kats():
    r = I.estimate_spectral_radius(0.0, [1.0, 2.0], lambda t, y: np.zeros_like(y))  # :13-19
    assert r.rho == 0.0
    r = I.estimate_spectral_radius(0.0, [0.5, 0.5], lambda t, y: np.array([-3 * y[0], -7 * y[1]]),
                                   v0=[1.0, 1.0])  # :21-29
    assert r.converged and r.rho / r.safety == pytest.approx(7.0, rel=0.01)
    r = I.estimate_spectral_radius(0.0, [0.0, 0.0], lambda t, y: np.array([2 * y[1], 0.5 * y[0]]),
                                   v0=[1.0, 0.0])  # :106-116
    assert not r.converged and r.iterations == 50
    with pytest.raises(ValueError):
        I.estimate_spectral_radius(0.0, [1.0], lambda t, y: y.copy(), v0=[0.0])
    n = 201  # :31-47
    w = (0.17 * 0.62 / 0.79) / (140.0 * 0.01 * 0.1 * 0.1)

    def lap(t, y):
        vm = np.concatenate([[y[1]], y[:-1]])
        vp = np.concatenate([y[1:], [y[-2]]])
        return w * (vp - 2.0 * y + vm)

    r = I.estimate_spectral_radius(0.0, np.full(n, -65.0), lap)
    sn = math.sin((n - 1) * math.pi / (2.0 * n))
    assert r.rho / r.safety == pytest.approx(4 * w * sn * sn, rel=0.05)


def test_spectral_matches_reference(reference):
    """Same iteration count and rho as the reference's own power iteration
    on the 1-D Laplacian from its seeded direction."""
    n = 201
    w = (0.17 * 0.62 / 0.79) / (140.0 * 0.01 * 0.1 * 0.1)

    def lap(t, y):
        vm = np.concatenate([[y[1]], y[:-1]])
        vp = np.concatenate([y[1:], [y[-2]]])
        return w * (vp - 2.0 * y + vm)

    y = np.full(n, -65.0)
    a = I.estimate_spectral_radius(0.0, y, lap)
    b, _ = reference.estimate_rho_fn(lap, y)
    assert a.iterations == b.iterations and abs(a.rho - b.rho) <= 1e-12 * b.rho


# ---- the grid problem through the generic layer -------------------------------

@pytest.mark.parametrize("rho_F,rho_S", [(60.0, 0.7), (300.0, 60.0)])  # s = 1 / 2, m = 2
def test_generic_grid_step_matches_fused_and_oracle(oracle, rho_F, rho_S):
    h = 0.25
    p = make_problem(3, [20, 16, 12], [h] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0,
                     [-0.125] * 3, [0.875] * 3, 0.0, 1.0)
    y0 = oracle.initial_state(p)
    y0[: p.n_nodes] += np.random.default_rng(4).normal(0.0, 0.1, p.n_nodes)
    op = MonodomainOperator(p)
    rhs = I.bind(op)
    rhs.rho_F, rhs.rho_S = rho_F, rho_S
    y_gen, rep = I.emrkc_step(0.1, y0, 0.05, rhs)
    # the power iteration through the generic layer on the operator's f_F
    # equals the handle's own (both sum norms in the reference's order)
    fF = I.estimate_spectral_radius(0.0, y0, (rhs.f_F, rhs.f_F_ctx))
    op.set_state(y0)
    rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F, 0.0)
    op.step(0.1, 0.05, rho_F, rho_S)
    y_fused = op.get_state()
    op.close()
    y_ref, orep, rc = oracle.emrkc_step(p, 0.1, y0, 0.05, 0.05, rho_F, rho_S)
    assert rc == 0 and (rep.s, rep.m) == (orep.s, orep.m) and rep.m == 2
    nn = p.n_nodes
    for b in range(4):
        sl = slice(b * nn, (b + 1) * nn)
        assert oracle.rel_l2(p, y_gen[sl], y_ref[sl]) <= 1e-13
        assert oracle.rel_l2(p, y_fused[sl], y_gen[sl]) <= 1e-12
    assert fF.iterations == rF.iterations and fF.rho == rF.rho


def test_callback_exception_propagates():
    """A right-hand side that raises aborts the device iteration and its own
    exception reaches the caller (as the cause of EMRKC_ECALLBACK)."""
    def bad(t, y):
        raise KeyError("boom")

    with pytest.raises(RuntimeError) as ei:
        I.rkc_iteration(0.0, [1.0], 0.1, bad, 3, 0.05)
    assert isinstance(ei.value.__cause__, KeyError)
    rhs = scalar_split(-1.0, -1.0, -1.0)
    rhs.f_S = bad
    with pytest.raises(RuntimeError) as ei:
        I.emrkc_step(0.0, [1.0], 0.1, rhs)
    assert isinstance(ei.value.__cause__, KeyError)
    # the context is usable afterwards
    out = I.rkc_iteration(0.0, [2.0], 0.3, lambda t, y: -4.0 * y, 1, 0.05)
    assert out[0] == pytest.approx(2.0 * (1.0 - 1.2), rel=1e-14)


# ---- the reference's nonlinear-system checks (P/tests/test_multirate.cpp:236-389)

def _test_system(lE=-3.0):
    """y0' = -5 y0 (fast), y1' = -y1 y0 (slow), y2' = lE (y2 - 0.5) (exp)."""
    def fF(t, y):
        out = np.zeros_like(y)
        out[0] = -5.0 * y[0]
        return out

    def fS(t, y):
        out = np.zeros_like(y)
        out[1] = -y[1] * y[0]
        return out

    def ex(y):
        lam = np.zeros_like(y)
        yinf = np.zeros_like(y)
        lam[2], yinf[2] = lE, 0.5
        return lam, yinf

    def exact(t, y0):
        return np.array([y0[0] * math.exp(-5.0 * t),
                         y0[1] * math.exp((math.exp(-5.0 * t) - 1.0) / 5.0 * y0[0]),
                         0.5 + (y0[2] - 0.5) * math.exp(lE * t)])

    return (lambda: I.GenericSplitRhs(fF, fS, ex, 5.0, 1.5)), exact


def _slope(xs, ys):
    x, y = np.log(xs), np.log(ys)
    n = len(x)
    return (n * (x * y).sum() - x.sum() * y.sum()) / (n * (x * x).sum() - x.sum() ** 2)


def test_emrkc_lambda_zero_equals_mrkc_nonlinear():
    """:287-314, 30 random nonlinear systems, 1e-13."""
    rng = np.random.default_rng(23)
    for _ in range(30):
        n = 2 + int(rng.integers(0, 9))

        def fF(t, y):
            out = -30.0 * y
            out[1:] += 2.0 * y[:-1]
            return out

        rhs = I.GenericSplitRhs(fF, lambda t, y: -0.5 * y * y + 0.1 * np.sin(y),
                                lambda y: (np.zeros_like(y), np.full_like(y, 0.3)), 35.0, 2.0)
        y = rng.random(n)
        dt = 0.05 + 0.2 * rng.random()
        a, _ = I.mrkc_step(0.0, y, dt, rhs)
        b, _ = I.emrkc_step(0.0, y, dt, rhs)
        assert np.abs(a - b).max() < 1e-13


@pytest.mark.parametrize("variant", [capi.EMRKC_VARIANT_STANDARD, capi.EMRKC_VARIANT_PROGRESSIVE])
def test_local_error_order_two(variant):
    """:316-342: one-step error slope 2 +- 0.15 over dt = 2^-4 .. 2^-10."""
    mk, exact = _test_system()
    y0 = np.array([1.0, 1.0, 0.9])
    hs, errs = [], []
    for k in range(4, 11):
        dt = 2.0 ** -k
        out, _ = I.emrkc_step(0.0, y0, dt, mk(), 0.05, variant)
        hs.append(dt)
        errs.append(np.abs(out - exact(dt, y0)).max())
    assert abs(_slope(hs, errs) - 2.0) <= 0.15


def test_global_first_order():
    """:344-389: global error slope 1 +- 0.1 for emRKC and for mRKC with the
    exponential part folded into f_S, dt = 2^-3 .. 2^-8 to T = 1."""
    mk, exact = _test_system()
    y0 = np.array([1.0, 1.0, 0.9])

    def em(t, y, dt):
        return I.emrkc_step(t, y, dt, mk())[0]

    def mr(t, y, dt):
        r = mk()
        base = r.f_S

        def fS(t2, y2):
            out = base(t2, y2)
            out[2] += -3.0 * (y2[2] - 0.5)
            return out

        return I.mrkc_step(t, y, dt, I.GenericSplitRhs(r.f_F, fS, None, 5.0, 4.0))[0]

    for stepper in (em, mr):
        hs, errs = [], []
        for k in range(3, 9):
            dt = 2.0 ** -k
            y = y0.copy()
            for i in range(round(1.0 / dt)):
                y = stepper(i * dt, y, dt)
            hs.append(dt)
            errs.append(np.abs(y - exact(1.0, y0)).max())
        assert abs(_slope(hs, errs) - 1.0) <= 0.1
