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
