"""The C++ host shim (include/emrkc.hpp): compiles with g++ against the C ABI
here; on a GPU the demo (tests/cpp/shim_demo.cpp) runs the reference's
run_simulation flow and matches the CPU oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2401_01745_b200")


def build(tmp_path, name="shim_demo"):
    exe = str(tmp_path / name)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", LIBDIR,
                    "-lemrkc_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))
    assert os.path.exists(build(tmp_path, "shim_kats"))


@pytest.mark.gpu
def test_shim_kats(tmp_path):
    """The reference's scalar KATs through the C++ shim's generic layer
    (device recurrences) and the HH IonicModel adapter."""
    import math

    exe = build(tmp_path, "shim_kats")
    r = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    phi = math.expm1(-0.5) / -0.5
    assert r["af_m1"] == pytest.approx(-11.0 * math.exp(-0.5) + phi * -5.0, rel=1e-13)
    assert r["af_m1"] == pytest.approx(-10.60653, rel=1e-6)
    assert r["af_exp"] == pytest.approx(-3.934693, rel=1e-6)
    assert r["afm_m1"] == pytest.approx(-11.0, rel=1e-13)
    assert (r["n_fF"], r["n_fS"], r["n_exp"]) == (3, 1, 1)
    assert r["rkc_s1"] == pytest.approx(2.0 * (1.0 - 1.2), rel=1e-14)
    assert r["R2"] == pytest.approx(0.125, rel=1e-14)
    assert r["abort_stage"] == 1 and r["rejected"] == 1
    assert (r["gating_s"], r["gating_m"]) == (1, 1)
    assert r["gating"] == pytest.approx(0.25 + 0.75 * math.exp(-3.2), rel=1e-12)
    assert r["rho_diag"] == pytest.approx(7.0, rel=0.01)
    assert r["alpha_m_m40"] == 1.0 and r["alpha_n_m55"] == 0.1
    assert r["V_rest"] == -64.99637933119206 and abs(r["I_rest"]) < 1e-10


@pytest.mark.gpu
def test_shim_matches_oracle(tmp_path, oracle):
    from paper_2401_01745_b200.monodomain import make_problem

    exe = build(tmp_path)
    state = str(tmp_path / "state.bin")
    out = subprocess.run([exe, "40", state], capture_output=True, text=True, check=True).stdout
    r = json.loads(out)
    assert r["s4"] == 4 and r["einval"] == 1 and r["steps"] == 40 and not r["aborted"]
    p = make_problem(2, [64, 48], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                     [-0.125, -0.125], [1.875, 1.875], 0.0, 1.0)
    y0 = oracle.initial_state(p)
    eF, _ = oracle.estimate_rho(p, 0, 0.0, y0)
    eS, _ = oracle.estimate_rho(p, 1, 0.0, y0)
    assert abs(r["rho_F"] - eF.rho) <= 1e-9 * eF.rho
    yo, ro, _ = oracle.run(p, y0, 0, 40, 0.05, 0.05, eF.rho, eS.rho)
    assert (r["s"], r["m"]) == (ro.s, ro.m)
    yg = np.fromfile(state, dtype=np.float64)
    nn = p.n_nodes
    errs = [oracle.rel_l2(p, yg[b * nn:(b + 1) * nn], yo[b * nn:(b + 1) * nn]) for b in range(4)]
    assert max(errs) <= 1e-9, errs
