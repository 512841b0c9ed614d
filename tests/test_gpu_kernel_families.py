"""Every selectable fast-kernel family against the oracle: EMRKC_PIPE = 3
(TMA-staged, default), 1 (cp.async-staged), 2 (persistent cp.async node
kernel when built with -DEMRKC_EXPERIMENTAL=1, measured slower; the
cp.async kernels otherwise), 0 (plain loads, z-march), on 3-D and 2-D grids with s = 1 / m = 1
and forced s = 2 / m = 2 (outer stages j >= 2 and V-only inner stages).
Runs use emrkc_step per step (the resident whole-run kernel would bypass
the families on small grids)."""
import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-9


def cases():
    p3 = make_problem(3, [40, 20, 18], [0.25] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0,
                      [-0.125] * 3, [0.875] * 3, 0.0, 1.0)
    p2 = make_problem(2, [136, 40], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                      [-0.125, -0.125], [1.875, 1.875], 0.0, 1.0)
    q3 = make_problem(3, [32, 24, 20], [0.05] * 3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0,
                      [-0.025] * 3, [0.175] * 3, 0.0, 1.0)
    # (name, problem, rho_F, rho_S, steps)
    return [("3d_s1m1", p3, 16.0, 0.7, 8), ("2d_s1m1", p2, 9.1, 0.7, 8),
            ("3d_s2m2", q3, 390.0, 50.0, 6)]


@pytest.mark.parametrize("pipe", ["3", "1", "2", "0"])
@pytest.mark.parametrize("case", [c[0] for c in cases()])
def test_family_against_oracle(oracle, monkeypatch, pipe, case):
    monkeypatch.setenv("EMRKC_PIPE", pipe)
    name, p, rF, rS, n = next(c for c in cases() if c[0] == case)
    y0 = oracle.initial_state(p)
    y0[: p.n_nodes] += np.random.default_rng(11).normal(0.0, 0.1, p.n_nodes)
    op = MonodomainOperator(p)
    op.set_state(y0)
    for k in range(n):
        rep = op.step(k * 0.05, 0.05, rF, rS)
    y = op.get_state()
    op.close()
    yo, ro, _ = oracle.run(p, y0, 0, n, 0.05, 0.05, rF, rS)
    assert (rep.s, rep.m) == (ro.s, ro.m)
    errs = rel_l2_blocks(oracle, p, y, yo)
    assert max(errs) <= TOL, errs
