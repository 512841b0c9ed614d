"""Device convergence harness: EXEX-RL reference (MREF0001-cached), device
rel_l2_error, observed orders; checked against the CPU oracle."""
import math

import numpy as np
import pytest

from paper_2401_01745_b200 import convergence as cv
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu


def small():
    p = make_problem(2, [64, 48], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                     [-0.125, -0.125], [3.875, 3.875], 0.0, 1.0)
    return p


def test_device_rel_l2_matches_oracle(oracle):
    p = small()
    rng = np.random.default_rng(3)
    y = oracle.initial_state(p)
    y[: p.n_nodes] += rng.normal(0.0, 5.0, p.n_nodes)
    op = MonodomainOperator(p)
    op.set_state(y)
    nn = p.n_nodes
    for b in range(4):
        ref = y[b * nn:(b + 1) * nn] * (1.0 + 1e-3 * rng.normal(size=nn))
        got = op.rel_l2_error(ref, b)
        want = oracle.rel_l2(p, y[b * nn:(b + 1) * nn], ref)
        assert abs(got - want) <= 1e-12 * want
    with pytest.raises(ValueError):
        op.rel_l2_error(np.zeros(nn), 0)
    op.close()


def test_convergence_table(oracle, tmp_path):
    p = small()
    y0 = oracle.initial_state(p)
    y0[: p.n_nodes] += np.random.default_rng(1).normal(0.0, 0.1, p.n_nodes)
    t_end, dt_ref = 0.5, 1e-4   # asymptotic regime: observed order ~1 (emRKC is first order)
    dts = [0.05, 0.025, 0.0125]
    tab = cv.run_convergence(p, y0, t_end, dts, "emrkc", dt_ref=dt_ref, cache_dir=str(tmp_path))
    assert [r.dt for r in tab.rows] == dts and all(r.stable for r in tab.rows)
    errs = [r.err for r in tab.rows]
    assert errs[0] > errs[1] > errs[2] > 0
    assert math.isnan(tab.rows[0].order) and all(0.8 < r.order < 1.2 for r in tab.rows[1:])
    # the device EXEX-RL reference against the oracle's
    ref, path = cv.reference_solution(p, y0, t_end, dt_ref, str(tmp_path))
    assert path and cv.load_reference(path, y0.size) is not None
    yo, ro, _ = oracle.run_method(p, y0, 0, cv.step_count(t_end, dt_ref), dt_ref, oracle.EXEX_RL)
    nn = p.n_nodes
    for b in range(4):
        assert oracle.rel_l2(p, ref[b * nn:(b + 1) * nn], yo[b * nn:(b + 1) * nn]) <= 1e-9
    # each row's error against the oracle's own error on its own runs
    for r in tab.rows:
        n = cv.step_count(t_end, r.dt)
        eF = oracle.estimate_rho(p, 0, 0.0, y0)[0].rho
        eS = oracle.estimate_rho(p, 1, 0.0, y0)[0].rho
        ya, _, _ = oracle.run(p, y0, 0, n, r.dt, 0.05, eF, eS)
        e_or = oracle.rel_l2(p, ya[:nn], yo[:nn])
        assert abs(r.err - e_or) <= 1e-6 * e_or
    out = tmp_path / "conv.csv"
    cv.write_convergence_csv(str(out), tab)
    assert out.read_text().count("\n") == 4
    # second call hits the cache
    tab2 = cv.run_convergence(p, y0, t_end, dts[:1], "emrkc", dt_ref=dt_ref, cache_dir=str(tmp_path))
    assert tab2.rows[0].err == errs[0]
