"""Host side of the convergence harness (paper_2401_01745_b200/convergence.py):
dt snapping, the MREF0001 cache format, the CSV layout (CPU only)."""
import math

import numpy as np
import pytest

from paper_2401_01745_b200 import convergence as cv


def test_snap_and_step_count():
    assert cv.snap_dt(5.0, 0.05) == 0.05 and cv.step_count(5.0, 0.05) == 100
    assert cv.snap_dt(5.0, 0.03) == 5.0 / 167  # lround(166.67) = 167
    assert cv.snap_dt(1.0, 7.0) == 1.0          # at least one step
    with pytest.raises(ValueError):
        cv.step_count(5.0, 0.03)
    assert cv.default_reference_dt(5.0, 0.05, [0.1, 0.025]) == cv.snap_dt(5.0, 1e-4)
    assert cv.default_reference_dt(1.0, 0.001, []) == cv.snap_dt(1.0, 0.001 / 20)


def test_fnv1a_is_the_reference_constant_set():
    # experiments.cpp:45-52 (its offset constant, as written there)
    assert cv.fnv1a("") == 1469598103934665603
    h = 1469598103934665603
    for c in b"ab":
        h = ((h ^ c) * 1099511628211) % (1 << 64)
    assert cv.fnv1a("ab") == h


def test_mref_roundtrip(tmp_path):
    y = np.random.default_rng(0).normal(size=1000)
    path = str(tmp_path / "sub" / "ref_x.bin")
    cv.store_reference(path, y)
    raw = open(path, "rb").read()
    assert raw[:8] == b"MREF0001" and int.from_bytes(raw[8:16], "little") == 1000
    assert len(raw) == 16 + 8000
    assert np.array_equal(cv.load_reference(path, 1000), y)
    assert cv.load_reference(path, 999) is None          # size mismatch
    open(path, "r+b").write(b"MREF0002")
    assert cv.load_reference(path, 1000) is None         # bad magic
    assert cv.load_reference(str(tmp_path / "none.bin"), 1000) is None


def test_csv_layout(tmp_path):
    t = cv.ConvergenceTable("emrkc", 1e-4, [
        cv.ConvergenceRow(0.1, 0.02, math.nan, 1, 1, {"n_fF": 10, "n_fS": 10, "n_exp": 10,
                                                      "wall_s": 0.5}, True),
        cv.ConvergenceRow(0.05, math.inf, math.nan, 1, 2, {"n_fF": 40, "n_fS": 20, "n_exp": 20,
                                                           "wall_s": 1.0}, False)])
    path = str(tmp_path / "conv.csv")
    cv.write_convergence_csv(path, t)
    lines = open(path).read().splitlines()
    assert lines[0] == ("method,dt,rel_l2_err,order,s,m,stable,n_fF,n_fS,n_exp,n_linsolves,"
                        "cg_iters,wall_s,t_fF_s,t_fS_s,t_exp_s,t_other_s")
    assert lines[1] == "emrkc,0.1,0.02,nan,1,1,1,10,10,10,0,0,0.5,0,0,0,0.5"
    assert lines[2] == "emrkc,0.05,inf,nan,1,2,0,40,20,20,0,0,1,0,0,0,1"
