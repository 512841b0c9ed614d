"""BASELINE's large grids run on the GPU against the reference's own records
(tests/golden/big_<workload>.npz, made by tests/golden/make_big_runs.py from
oracle/_ref = the unmodified reference sources): config 4's grid
(512x512x256, HH standing in for TTP: s = 1, m = 2) run into the
reference's own abort at step 65; config 3's grid (256x256x128, HH standing
in for CRN) over 20 steps (reference self-divergence 1e-16: the 1e-9 bar),
60 steps (self-divergence ~2e-9: 4x that) and its full 400 steps (the
reference diverges from itself by 0.05-0.5 there: record and rho only);
config 5 at N = 50 over its full T (three sensitivity seeds).

Exact: s, m, rho iteration counts, abort step / kind / stage, counters.
Within the bar: rho (RHO_TOL), gate range, and per block the per-plane sums
and sums of squares (a whole-field fingerprint, one entry per z-plane), the
block norm and sum, and rel-L2 over 65,536 seeded sample nodes. The bar is
north_star's 1e-9 unless the fixture's measured self-sensitivity of the
reference (its divergence from itself under a 1e-15 relative perturbation
of the initial state) says the problem is worse conditioned than that.

Plus the whole-field check of config 2 (128^3, 100 steps): the plain-C
oracle (bit-identical to the reference, tests/test_oracle_vs_ref.py) runs
the same simulation on the GPU box's host and the whole final state is
compared by the reference's trapezoid rel_l2_error per block."""
import glob
import json
import os

import numpy as np
import pytest

from conftest import rel_l2_blocks
from paper_2401_01745_b200 import capi, workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "big_*.npz")))
TOL = 1e-9
RHO_TOL = 1e-12
EXACT = ["n_steps", "steps_done", "aborted", "abort_kind", "abort_step", "abort_stage",
         "n_fF", "n_fS", "n_exp", "s", "m"]


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(f)[4:-4] for f in FIXTURES])
def test_big_run_against_reference(path):
    g = np.load(path)
    meta = json.loads(bytes(g["meta"]))
    w = workloads.get(meta["workload"])
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F)
    rS = op.estimate_spectral_radius(capi.EMRKC_RHS_S)
    assert (rF.iterations, rS.iterations) == (meta["rho_F_iterations"], meta["rho_S_iterations"])
    assert abs(rF.rho - meta["rho_F"]) <= RHO_TOL * meta["rho_F"], (rF.rho, meta["rho_F"])
    assert abs(rS.rho - meta["rho_S"]) <= RHO_TOL * meta["rho_S"], (rS.rho, meta["rho_S"])
    # the run continues from the reference's own rho (as make_big_runs did)
    res = op.run(0, meta["steps"], meta["dt"], meta["rho_F"], meta["rho_S"], meta["eps"]).as_dict()
    y = op.get_state()
    op.close()
    rec = meta["record"]
    for k in EXACT:
        assert res[k] == rec[k], (k, res[k], rec[k])
    assert abs(res["eta"] - rec["eta"]) <= 1e-15
    nf = p.n_fields
    sens = [max(s["rel_l2"][b] for s in meta["sensitivity"]) if meta["sensitivity"] else 0.0
            for b in range(nf)]
    bars = [max(TOL, 4.0 * sv) for sv in sens]
    # A run whose reference diverges from ITSELF by more than 1e-3 under a
    # 1e-15 input perturbation (config 3's grid over its full T: 0.05-0.5)
    # has no reproducible field to compare: the record (s, m, counters, no
    # abort) and rho are asserted above, the field differences are printed.
    chaotic = max(sens) > 1e-3
    if not chaotic:
        assert abs(res["gate_min"] - rec["gate_min"]) <= max(bars[1:4])
        assert abs(res["gate_max"] - rec["gate_max"]) <= max(bars[1:4])
    nn = p.n_nodes
    n_planes = int(p.n[p.dim - 1])
    idx = g["sample_index"]
    for b in range(nf):
        blk = y[b * nn:(b + 1) * nn]
        pl = blk.reshape(n_planes, -1)
        errs = {
            "plane_sum": _rel(pl.sum(axis=1), g[f"plane_sum_{b}"]),
            "plane_sq": _rel(np.einsum("ij,ij->i", pl, pl), g[f"plane_sq_{b}"]),
            "norm2": abs(float(np.linalg.norm(blk)) - float(g[f"norm2_{b}"])) / float(g[f"norm2_{b}"]),
            "sample": _rel(blk[idx], g["sample"][b]),
        }
        print(meta["workload"], meta["steps"], "block", b, errs, "bar", bars[b],
              "(ill-conditioned: not asserted)" if chaotic else "")
        if not chaotic:
            assert max(errs.values()) <= bars[b], (b, errs, bars[b])


@pytest.mark.slow
def test_config2_whole_field_vs_oracle(oracle):
    """Config 2 (128^3, 100 steps = T): the whole final field against the
    plain-C oracle run on this host (~70 s), trapezoid rel_l2 per block."""
    w = workloads.get("hh3d_128x128x128")
    p = w.problem
    y0 = w.initial_state()
    op = MonodomainOperator(p)
    op.set_state(y0)
    rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F).rho
    rS = op.estimate_spectral_radius(capi.EMRKC_RHS_S).rho
    res = op.run(0, w.n_steps, w.dt, rF, rS, w.eps)
    yg = op.get_state()
    op.close()
    oF, _ = oracle.estimate_rho(p, 0, 0.0, y0)
    oS, _ = oracle.estimate_rho(p, 1, 0.0, y0)
    assert abs(rF - oF.rho) <= RHO_TOL * oF.rho and abs(rS - oS.rho) <= RHO_TOL * oS.rho
    yo, ro, _ = oracle.run(p, y0, 0, w.n_steps, w.dt, w.eps, oF.rho, oS.rho)
    assert (res.s, res.m, res.steps_done, res.aborted) == (ro.s, ro.m, ro.steps_done, ro.aborted)
    errs = rel_l2_blocks(oracle, p, yg, yo)
    print("config 2 whole-field rel-L2 per block", errs)
    assert max(errs) <= TOL, errs
