"""Pin the CPU oracle (oracle/emrkc_oracle.c) against the reference's own
known-answer constants (the doctest suites under
P/tests/ cannot be built here, so their constants are restated) and, where
oracle/_ref is built, run the same checks through the compiled reference."""
import math

import numpy as np
import pytest

from paper_2401_01745_b200.monodomain import make_problem


@pytest.fixture(params=["oracle", "reference"])
def impl(request, oracle):
    if request.param == "oracle":
        return oracle
    from oracle.oracle import Reference, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref not built")
    return Reference()


# ---- cheb (P/tests/test_cheb.cpp) -------------------------------------------

def test_get_stages(impl):
    s, ell, beta = impl.get_stages(0.1, 193.3333, 0.05)  # :42-47
    assert s == 4 and abs(ell - 30.93333) <= 1e-5 * 30.93333
    s, ell, _ = impl.get_stages(1.0, 0.0, 0.05)  # :48-52
    assert s == 1 and abs(ell - 1.933333) <= 1e-6 * 1.933333
    assert impl.get_stages(1.0, 1.933333, 0.05)[0] == 1  # :53-56
    for bad in [(0.0, 1.0, 0.05), (1.0, -1.0, 0.05), (1.0, math.nan, 0.05), (1.0, 1.0, 1.5)]:
        with pytest.raises(ValueError):
            impl.get_stages(*bad)


def test_rkc_coeffs_known(impl):
    k = impl.rkc_coeffs(1, 0.05)  # :65-71
    assert abs(k["omega0"] - 1.05) <= 1e-15 and k["mu"][1] == pytest.approx(1.0, rel=1e-15)
    assert k["c"][1] == pytest.approx(1.0, rel=1e-15)
    k = impl.rkc_coeffs(2, 0.0)  # :72-79
    assert k["mu"][1] == pytest.approx(0.25, rel=1e-15)
    assert k["mu"][2] == pytest.approx(0.5, rel=1e-15)
    assert k["nu"][2] == pytest.approx(2.0, rel=1e-15)
    assert k["kappa"][2] == pytest.approx(-1.0, rel=1e-15)
    assert k["c"][2] == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(ValueError):
        impl.rkc_coeffs(0, 0.05)


def test_rkc_coeffs_invariants(impl):
    for s in range(1, 51):  # :82-97
        k = impl.rkc_coeffs(s, 0.05)
        assert k["c"][0] == 0.0 and abs(k["c"][s] - 1.0) < 1e-12
        for j in range(2, s + 1):
            assert abs(k["nu"][j] + k["kappa"][j] - 1.0) < 1e-12
        assert np.all(k["c"] >= -1e-12) and np.all(k["c"] <= 1 + 1e-12)


def test_rkc_iteration_scalar(oracle):
    # s=1 damped Euler on y' = -4y from 2 over 0.3: 2(1 - 1.2)  (:118-124)
    out, rc, _ = oracle.rkc_iteration(lambda t, y: -4.0 * y, np.array([2.0]), 0.3, 1, 0.05)
    assert rc == 0 and out[0] == pytest.approx(2.0 * (1.0 - 1.2), rel=1e-14)
    # s=2, eps=0: R_2(-1) = 1 - 1 + 1/8 (:125-131)
    out, rc, _ = oracle.rkc_iteration(lambda t, y: -1.0 * y, np.array([1.0]), 1.0, 2, 0.0)
    assert out[0] == pytest.approx(0.125, rel=1e-14)
    # zero rhs keeps y (:111-117)
    y = np.array([1.5, -2.0, 0.25])
    for s in (1, 3, 9):
        out, _, _ = oracle.rkc_iteration(lambda t, u: np.zeros_like(u), y, 0.7, s, 0.05)
        np.testing.assert_allclose(out, y, rtol=1e-14)
    # exactly s evaluations, stage times t + c_j dt (:132-166)
    times = []

    def probe(t, u):
        times.append(t)
        return np.zeros_like(u)

    oracle.rkc_iteration(probe, np.array([1.0]), 2.0, 4, 0.05, t=10.0)
    c = oracle.rkc_coeffs(4, 0.05)["c"]
    assert len(times) == 4
    for j in range(4):
        assert times[j] == pytest.approx(10.0 + c[j] * 2.0, rel=1e-15)
    # non-finite stage aborts naming stage 1 (:143-153)
    out, rc, st = oracle.rkc_iteration(lambda t, u: np.full_like(u, np.inf), np.array([1.0]), 1.0, 3, 0.05)
    assert rc == 2 and st == 1


def test_rkc_iteration_matches_reference(reference, oracle):
    rng = np.random.default_rng(7)
    for _ in range(100):  # P/tests/test_cheb.cpp:206-223 style
        s = int(rng.integers(1, 21))
        beta = 2 - 4 * 0.05 / 3
        z = -beta * s * s * rng.random()
        dt = 0.25 + rng.random()
        lam = z / dt
        y0 = 1.0 + rng.random()
        a = reference.rkc_iteration_scalar(0.0, y0, dt, lam, s, 0.05)
        b, rc, _ = oracle.rkc_iteration(lambda t, y: lam * y, np.array([y0]), dt, s, 0.05)
        assert rc == 0 and a == b[0]


# ---- multirate (P/tests/test_multirate.cpp) -----------------------------------

def test_phi(impl):
    assert impl.phi(0.0) == 1.0
    assert impl.phi(-1.0) == pytest.approx(1 - math.exp(-1), rel=1e-15)
    assert impl.phi(1e-6) == pytest.approx(1 + 0.5e-6, rel=1e-12)


def test_exponential_euler(oracle):
    out = oracle.exponential_euler_step([1.0], 0.5, [-2.0], [0.25])  # :28-32
    assert out[0] == pytest.approx(0.25 + 0.75 * math.exp(-1.0), rel=1e-15)
    y = np.array([0.3, -1.2, 7.0])
    assert np.array_equal(oracle.exponential_euler_step(y, 0.5, [0, 0, 0], [0, 0, 0]), y)
    y = np.array([0.6, 0.2])
    assert np.array_equal(oracle.exponential_euler_step(y, 3.0, [-5.0, -1.0], y), y)


def test_averaged_force_emrkc_closed_forms(impl):
    # m=1: (lF+lS) e^{eta lE} + phi(eta lE) lE  (:97-106)
    f = impl.averaged_force_emrkc(-10.0, -1.0, -5.0, 0.0, 1.0, 0.1, 1)
    assert f == pytest.approx(-11.0 * math.exp(-0.5) + impl.phi(-0.5) * -5.0, rel=1e-13)
    assert f == pytest.approx(-10.60653, rel=1e-6)
    # pure exponential part (:124-131)
    f = impl.averaged_force_emrkc(0.0, 0.0, -5.0, 0.0, 1.0, 0.1, 1)
    assert f == pytest.approx(-3.934693, rel=1e-6)


def _stab_poly(impl_rkc, s, eps, z):
    return impl_rkc(s, eps, z)


def test_emrkc_step_scalar_closed_form(oracle):
    """P/tests/test_multirate.cpp:189-214: emrkc_step equals
    P_s(dt [Phi_m(eta lF)(lF+lS) e^{eta lE} + phi(eta lE) lE])."""
    def R(s, eps, z):
        out, _, _ = oracle.rkc_iteration(lambda t, y: z * y, np.array([1.0]), 1.0, s, eps)
        return out[0]

    def Phi(s, eps, z):
        if abs(z) < 1e-8:
            h = 1e-5
            rpp = (R(s, eps, h) - 2.0 + R(s, eps, -h)) / (h * h)
            return 1.0 + 0.5 * rpp * z
        return (R(s, eps, z) - 1.0) / z

    rng = np.random.default_rng(17)
    for _ in range(60):
        lF = -10 ** (4 * rng.random())
        lS = -10 ** (1.5 * rng.random())
        lE = -10 ** (3 * rng.random())
        dt = 10 ** (-2 + 3 * rng.random())
        out, s, m, eta = oracle.emrkc_step_scalar(lF, lS, lE, 0.0, 1.0, dt)
        inner = Phi(m, 0.05, eta * lF) * (lF + lS) * math.exp(eta * lE) + oracle.phi(eta * lE) * lE
        expected = R(s, 0.05, dt * inner)
        assert out == pytest.approx(expected, rel=1e-12, abs=1e-300)


def test_emrkc_gating_only_exact(impl):
    # eps=0, s=m=1: exact frozen-Lambda solution (:215-228)
    out, s, m, _ = impl.emrkc_step_scalar(0.0, 0.0, -4.0, 0.25, 1.0, 0.8, 0.0)
    assert (s, m) == (1, 1)
    assert out == pytest.approx(0.25 + 0.75 * math.exp(0.8 * -4.0), rel=1e-12)


def test_emrkc_zero_problem_fixed_point(impl):
    out, s, m, _ = impl.emrkc_step_scalar(0.0, 0.0, 0.0, 0.0, 3.0, 1.0)
    assert out == 3.0


# ---- spectral (P/tests/test_spectral.cpp) ------------------------------------

def test_spectral_known(impl):
    res, _ = impl.estimate_rho_fn(lambda t, y: np.zeros_like(y), np.array([1.0, 2.0]))
    assert res.rho == 0.0  # :13-19
    res, _ = impl.estimate_rho_fn(lambda t, y: np.array([-3 * y[0], -7 * y[1]]), np.array([0.5, 0.5]),
                                  v0=np.array([1.0, 1.0]))
    assert res.converged and res.rho / res.safety == pytest.approx(7.0, rel=0.01)  # :21-29
    # cycling operator hits the iteration cap (:106-116)
    res, _ = impl.estimate_rho_fn(lambda t, y: np.array([2 * y[1], 0.5 * y[0]]), np.array([0.0, 0.0]),
                                  v0=np.array([1.0, 0.0]))
    assert not res.converged and res.iterations == 50
    with pytest.raises(ValueError):
        impl.estimate_rho_fn(lambda t, y: y.copy(), np.array([1.0]), v0=np.array([0.0]))


def test_spectral_1d_laplacian(impl):
    n = 201  # :31-47
    sigma = 0.17 * 0.62 / 0.79
    w = sigma / (140.0 * 0.01 * 0.1 * 0.1)

    def lap(t, y):
        out = np.empty_like(y)
        vm = np.concatenate([[y[1]], y[:-1]])
        vp = np.concatenate([y[1:], [y[-2]]])
        out[:] = w * (vp - 2.0 * y + vm)
        return out

    res, _ = impl.estimate_rho_fn(lap, np.full(n, -65.0))
    sn = math.sin((n - 1) * math.pi / (2.0 * n))
    assert res.rho / res.safety == pytest.approx(4 * w * sn * sn, rel=0.05)


def test_seeded_direction_is_libstdcxx(oracle, reference):
    a = oracle.uniform_direction(0x9E3779B97F4A7C15, 5000)
    b = reference.uniform_direction(0x9E3779B97F4A7C15, 5000)
    assert np.array_equal(a, b)


# ---- monodomain + HH (P/tests/test_monodomain.cpp, test_ionic.cpp) ------------

def _p1d(stim=50.0):
    sig = 0.17 * 0.62 / 0.79
    return make_problem(1, [201], [0.1], [sig], 140.0, 0.01, stim, [0.0], [1.5], 0.0, 2.0)


def test_diffusion_unit_bump(oracle):
    p = _p1d()
    w = p.sigma[0] / (140.0 * 0.01 * 0.1 * 0.1)
    assert w == pytest.approx(9.52984, rel=1e-5)  # :94-97
    y = np.zeros(4 * 201)
    y[100] = 1.0
    out = oracle.rhs(p, 0, 0.0, y)
    assert out[99] == pytest.approx(w, rel=1e-14) and out[101] == pytest.approx(w, rel=1e-14)
    assert out[100] == pytest.approx(-2 * w, rel=1e-14) and out[98] == 0.0
    y[:201] = -63.7
    assert np.all(oracle.rhs(p, 0, 0.0, y)[:201] == 0.0)  # constant -> 0 (:80-88)


def test_stimulus_box(impl):
    p = _p1d()
    assert impl.stimulus_rate(p, 1.0, 0) == pytest.approx(50.0 / 1.4, rel=1e-15)  # :274-279
    assert impl.stimulus_rate(p, 1.0, 15) > 0.0
    assert impl.stimulus_rate(p, 1.0, 16) == 0.0
    assert impl.stimulus_rate(p, 2.5, 0) == 0.0


def test_hh_rates_and_rest(impl):
    a, b = impl.rates(-40.0)
    assert a[0] == 1.0  # P/tests/test_ionic.cpp:12-18
    a, b = impl.rates(-55.0)
    assert a[2] == 0.1
    V, z = impl.resting_state()
    assert V == -64.99637933119206  # SURVEY §3.1 [measured]
    assert abs(impl.ionic_current(V, z)) < 1e-10
    for Vs in np.arange(-100.0, 60.0, 0.7):
        lam, zi = impl.gate_coeffs(Vs)
        assert np.all(lam <= 0) and np.all(zi >= 0) and np.all(zi <= 1)


def test_rest_is_fixed_point(oracle):
    """Resting run stays at V_rest within 0.01 mV (P/tests/test_harness.cpp:117-135)."""
    p = _p1d(stim=0.0)
    y0 = oracle.initial_state(p)
    y, res, _ = oracle.run(p, y0, 0, 100, 0.1, 0.05, 40.0, 0.7)
    assert not res.aborted
    assert np.max(np.abs(y[:201] - y0[0])) < 0.01


def test_rel_l2(oracle):
    p = make_problem(1, [9], [0.25], [0.1])
    a = np.full(9, 1.01)
    b = np.full(9, 1.0)
    assert oracle.rel_l2(p, a, b) == pytest.approx(0.01, rel=1e-12)
    assert oracle.rel_l2(p, b, b) == 0.0
