"""Pin the C restatement against the reference compiled from its own sources
(oracle/_ref) on BASELINE workloads: bit-identical rho estimates, plans,
run records and states."""
import numpy as np
import pytest

from paper_2401_01745_b200 import workloads


@pytest.mark.parametrize("name,nsteps", [("hh2d_256x256", 20), ("p2d_128_s3m2", 10),
                                         ("p3d_48_s2m2", 4), ("hh3d_sweep_25", 10)])
def test_bitwise_on_workloads(oracle, reference, name, nsteps):
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    ests = []
    for impl in (oracle, reference):
        eF, vF = impl.estimate_rho(p, 0, 0.0, y0)
        eS, vS = impl.estimate_rho(p, 1, 0.0, y0)
        ests.append((eF.rho, eF.iterations, eS.rho, eS.iterations, vF, vS))
    a, b = ests
    assert a[:4] == b[:4]
    assert np.array_equal(a[4], b[4]) and np.array_equal(a[5], b[5])
    rS = w.rho_S_forced if w.rho_S_forced is not None else a[2]
    ya, ra, _ = oracle.run(p, y0, 0, nsteps, w.dt, w.eps, a[0], rS)
    yb, rb, _ = reference.run(p, y0, 0, nsteps, w.dt, w.eps, a[0], rS)
    assert np.array_equal(ya, yb)
    for k, _ in ra._fields_:
        if k != "device_ms":
            assert getattr(ra, k) == getattr(rb, k), k


def test_operator_pieces_bitwise(oracle, reference):
    w = workloads.parity_3d()
    p = w.problem
    rng = np.random.default_rng(5)
    nn = p.n_nodes
    y = np.concatenate([rng.uniform(-90, 50, nn), rng.uniform(0, 1, 3 * nn)])
    for which in (0, 1):
        for t in (0.0, 0.5, 3.0):
            assert np.array_equal(oracle.rhs(p, which, t, y), reference.rhs(p, which, t, y))
    la, ia = oracle.exp_part(p, y)
    lb, ib = reference.exp_part(p, y)
    assert np.array_equal(la, lb) and np.array_equal(ia, ib)
    for V in np.linspace(-100, 60, 321):
        assert np.array_equal(oracle.rates(V)[0], reference.rates(V)[0])
    assert oracle.analytic_rho_F(p) == reference.analytic_rho_F(p)


def test_single_step_abort_records(oracle, reference):
    w = workloads.hh2d_256()
    p = w.problem
    y0 = w.initial_state()
    y0[p.n_nodes * 3 + 11] = np.inf
    oa, ra, rca = oracle.emrkc_step(p, 0.0, y0, 0.05, 0.05, 10.0, 0.7)
    ob, rb, rcb = reference.emrkc_step(p, 0.0, y0, 0.05, 0.05, 10.0, 0.7)
    assert rca == rcb == 2
    assert ra.abort_stage == rb.abort_stage == 1
    assert (ra.n_fF, ra.n_fS, ra.n_exp) == (rb.n_fF, rb.n_fS, rb.n_exp)


def _same_records(ra, rb):
    for k, _ in ra._fields_:
        if k != "device_ms":
            va, vb = getattr(ra, k), getattr(rb, k)
            assert va == vb or (va != va and vb != vb), k


@pytest.mark.parametrize("name,nsteps", [("p2d_128_s3m2", 10), ("p3d_48_s2m2", 4),
                                         ("hh2d_256x256", 20)])
def test_progressive_variant_bitwise(oracle, reference, name, nsteps):
    """emRKC progressive (P/src/multirate.cpp:106-115): restatement vs reference."""
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    eF, _ = reference.estimate_rho(p, 0, 0.0, y0)
    rS = w.rho_S_forced if w.rho_S_forced is not None else reference.estimate_rho(p, 1, 0.0, y0)[0].rho
    ya, ra, _ = oracle.run_method(p, y0, 0, nsteps, w.dt, oracle.EMRKC_PROGRESSIVE, w.eps, eF.rho, rS)
    yb, rb, _ = reference.run_method(p, y0, 0, nsteps, w.dt, reference.EMRKC_PROGRESSIVE, w.eps,
                                     eF.rho, rS)
    assert np.array_equal(ya, yb)
    _same_records(ra, rb)
    # for HH (no aux) the V rows equal the standard variant's; gates differ
    # only by rounding (constant forcing on gate rows)
    ys, _, _ = oracle.run_method(p, y0, 0, nsteps, w.dt, oracle.EMRKC, w.eps, eF.rho, rS)
    for b in range(4):
        assert oracle.rel_l2(p, ya[b * p.n_nodes:(b + 1) * p.n_nodes],
                             ys[b * p.n_nodes:(b + 1) * p.n_nodes]) < 1e-12


@pytest.mark.parametrize("dim", [2, 3])
def test_exex_rl_bitwise(oracle, reference, dim):
    """EXEX-RL (P/src/baselines.cpp:192-210) inside run_simulation's loop."""
    w = workloads.get("p2d_128_s3m2" if dim == 2 else "p3d_48_s2m2")
    p = w.problem
    y0 = w.initial_state()
    ya, ra, _ = oracle.run_method(p, y0, 0, 60, 0.002, oracle.EXEX_RL)
    yb, rb, _ = reference.run_method(p, y0, 0, 60, 0.002, reference.EXEX_RL)
    assert np.array_equal(ya, yb)
    _same_records(ra, rb)
    assert ra.n_fF == ra.n_fS == ra.n_exp == 60 and not ra.aborted


def test_exex_rl_nonfinite_gate(oracle, reference):
    """exex_rl_step never throws: a NaN gate reaches V a step later and the
    norm guard (max_abs_v -> inf) stops the run with the state assigned."""
    w = workloads.get("p2d_128_s3m2")
    p = w.problem
    y0 = w.initial_state()
    y0[p.n_nodes + 7] = np.nan
    ya, ra, _ = oracle.run_method(p, y0, 2, 5, 0.002, oracle.EXEX_RL)
    yb, rb, _ = reference.run_method(p, y0, 2, 5, 0.002, reference.EXEX_RL)
    assert np.array_equal(ya, yb, equal_nan=True)
    _same_records(ra, rb)
    assert ra.aborted and ra.abort_kind == 2 and ra.abort_step == 2 and ra.steps_done == 1


def test_mrkc_pieces_bitwise(oracle, reference):
    """Stiff-gate split (P/src/monodomain.cpp:223-236,287-304) and
    identify_stiff_gates (P/src/ionic.cpp:130-146)."""
    w = workloads.parity_3d()
    p = w.problem
    rng = np.random.default_rng(9)
    nn = p.n_nodes
    y = np.concatenate([rng.uniform(-90, 50, nn), rng.uniform(0, 1, 3 * nn)])
    for stiff in (1, 2, 5, 7):
        for which in (0, 1):
            assert np.array_equal(oracle.rhs_gates(p, which, stiff, 0.3, y),
                                  reference.rhs_gates(p, which, stiff, 0.3, y))
    V = np.linspace(-90, 40, 200)
    assert oracle.identify_stiff_gates(V) == reference.identify_stiff_gates(V)
    assert oracle.identify_stiff_gates(V)[0] == 0  # m is the stiffest HH gate
    for which in (oracle.RHS_F_GATES, oracle.RHS_S_GATES):
        a, va = oracle.estimate_rho_gates(p, which, 1, 0.0, w.initial_state())
        b, vb = reference.estimate_rho(p, which | (1 << 4), 0.0, w.initial_state())
        assert (a.rho, a.iterations) == (b.rho, b.iterations) and np.array_equal(va, vb)


@pytest.mark.parametrize("name,nsteps", [("p2d_128_s3m2", 10), ("p3d_48_s2m2", 4),
                                         ("hh2d_256x256", 20)])
def test_mrkc_bitwise(oracle, reference, name, nsteps):
    """mrkc_step (P/src/multirate.cpp:158-171) with the m gate in the fast part."""
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    rF = reference.estimate_rho(p, 2 | (1 << 4), 0.0, y0)[0].rho
    rS = w.rho_S_forced if w.rho_S_forced is not None else \
        reference.estimate_rho(p, 3 | (1 << 4), 0.0, y0)[0].rho
    ya, ra, _ = oracle.run_mrkc(p, y0, 0, nsteps, w.dt, 1, w.eps, rF, rS)
    yb, rb, _ = reference.run_mrkc(p, y0, 0, nsteps, w.dt, 1, w.eps, rF, rS)
    assert np.array_equal(ya, yb)
    _same_records(ra, rb)
    assert ra.n_exp == 0 and ra.n_fF == nsteps * ra.s * ra.m and ra.n_fS == nsteps * ra.s


@pytest.mark.parametrize("name,dt,nsteps,jacobi", [("p2d_128_s3m2", 0.02, 8, True),
                                                   ("p3d_48_s2m2", 0.05, 3, True),
                                                   ("hh2d_256x256", 0.05, 10, False)])
def test_imex_rl_bitwise(oracle, reference, name, dt, nsteps, jacobi):
    """imex_rl_step with cg_solve (P/src/baselines.cpp:20-82,132-190)."""
    w = workloads.get(name)
    p = w.problem
    y0 = w.initial_state()
    ya, ra, ia = oracle.run_imex(p, y0, 0, nsteps, dt, 1e-8, 0, jacobi)
    yb, rb, ib = reference.run_imex(p, y0, 0, nsteps, dt, 1e-8, 0, jacobi)
    assert np.array_equal(ya, yb)
    _same_records(ra, rb)
    assert ia == ib > 0 and ra.n_fF == ia + 2 * nsteps


def test_imex_rl_cg_failure(oracle, reference):
    """max_iters too small: NumericalAbort, state not assigned."""
    w = workloads.get("p2d_128_s3m2")
    p = w.problem
    y0 = w.initial_state()
    ya, ra, _ = oracle.run_imex(p, y0, 4, 3, 0.05, 1e-12, 2, True)
    yb, rb, _ = reference.run_imex(p, y0, 4, 3, 0.05, 1e-12, 2, True)
    _same_records(ra, rb)
    assert ra.aborted and ra.abort_step == 4 and ra.steps_done == 0
    assert np.array_equal(ya, y0) and np.array_equal(yb, y0)


@pytest.mark.parametrize("n_aux,rS,nsteps", [(15, 0.7, 6), (17, 60.0, 4)])
def test_synthetic_width_bitwise(oracle, reference, n_aux, rS, nsteps):
    """EMRKC_MODEL_HH_AUX (the SYNTHETIC width stand-in, include/emrkc.h): the
    C restatement against the reference's own generic machinery (StateLayout
    with n_aux, f_S aux rows, exponential Euler passing aux through) running
    the harness's HHAux IonicModel: bit-identical operator pieces, rho and
    runs (s = 1 and forced s = 2, m = 2)."""
    from paper_2401_01745_b200.monodomain import make_problem

    h = 0.1
    p = make_problem(3, [12, 10, 9], [h] * 3, [0.3, 0.1, 0.1], 140.0, 0.01, 70.0,
                     [-0.05] * 3, [0.35] * 3, 0.0, 1.0, n_aux=n_aux)
    assert p.state_len() == (4 + n_aux) * p.n_nodes
    y0 = oracle.initial_state(p)
    assert np.array_equal(y0, reference.initial_state(p))
    rng = np.random.default_rng(9)
    y = y0 * rng.uniform(0.99, 1.01, y0.size)
    for which in (0, 1):
        assert np.array_equal(oracle.rhs(p, which, 0.5, y), reference.rhs(p, which, 0.5, y))
    la, ia = oracle.exp_part(p, y)
    lb, ib = reference.exp_part(p, y)
    assert np.array_equal(la, lb) and np.array_equal(ia, ib)
    eF, _ = oracle.estimate_rho(p, 0, 0.0, y)
    fF, _ = reference.estimate_rho(p, 0, 0.0, y)
    eS, _ = oracle.estimate_rho(p, 1, 0.0, y)
    fS, _ = reference.estimate_rho(p, 1, 0.0, y)
    assert (eF.rho, eF.iterations, eS.rho, eS.iterations) == \
        (fF.rho, fF.iterations, fS.rho, fS.iterations)
    ya, ra, _ = oracle.run(p, y, 0, nsteps, 0.05, 0.05, 250.0, rS)
    yb, rb, _ = reference.run(p, y, 0, nsteps, 0.05, 0.05, 250.0, rS)
    assert np.array_equal(ya, yb) and (ra.s, ra.m) == (rb.s, rb.m)
    for k, _ in ra._fields_:
        if k != "device_ms":
            assert getattr(ra, k) == getattr(rb, k), k
