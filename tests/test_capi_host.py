"""The C-ABI library loads, exports every entry point include/emrkc.h
declares, and its host-side numerics (no device needed) are bit-identical to
the oracle (which is itself pinned to the reference)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2401_01745_b200 import capi
from paper_2401_01745_b200 import monodomain as md
from paper_2401_01745_b200 import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "emrkc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(emrkc_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    lib = capi.load()
    names = header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(capi.PROTOTYPES), set(names) ^ set(capi.PROTOTYPES)


def test_version():
    assert b"sm_100a" in capi.load().emrkc_version()


def test_get_stages_matches_oracle(oracle):
    rng = np.random.default_rng(0)
    for _ in range(500):
        dt = 10 ** rng.uniform(-3, 1)
        rho = 10 ** rng.uniform(-2, 4)
        eps = rng.uniform(0, 1.4)
        p = md.get_stages(dt, rho, eps)
        assert (p.s, p.ell, p.beta) == oracle.get_stages(dt, rho, eps)
    for bad in [(0.0, 1.0, 0.05), (1.0, -1.0, 0.05), (1.0, math.nan, 0.05), (1.0, 1.0, 1.5)]:
        with pytest.raises(ValueError):
            md.get_stages(*bad)


def test_rkc_coeffs_bitwise(oracle):
    for s in [1, 2, 3, 7, 20, 50, 200]:
        for eps in [0.0, 0.05, 0.5]:
            a = md.rkc_coeffs(s, eps)
            b = oracle.rkc_coeffs(s, eps)
            assert a.omega0 == b["omega0"] and a.omega1 == b["omega1"]
            for k in ("b", "mu", "nu", "kappa", "c"):
                assert np.array_equal(getattr(a, k), b[k]), (s, eps, k)
    with pytest.raises(ValueError):
        md.rkc_coeffs(0, 0.05)


def test_plan_step_matches_oracle(oracle):
    # forced-rho parity cases of SURVEY §8(d) and the BASELINE settings
    for dt, rF, rS, s, m in [(0.05, 453.3732502254644, 200.0, 3, 2),
                             (0.05, 388.2325741578916, 50.0, 2, 2),
                             (0.05, 9.064, 0.7114, 1, 1),
                             (0.05, 139.0046, 0.7114, 1, 2),
                             (0.05, 386.6, 0.7114, 1, 4)]:
        rep = md.plan_step(dt, rF, rS, 0.05)
        assert (rep.s, rep.m) == (s, m)
        assert (rep.n_fF, rep.n_fS, rep.n_exp) == (s * m, s, s)
        so, ell_s, _ = oracle.get_stages(dt, rS, 0.05)
        assert rep.eta == 2.0 * dt / ell_s


def test_resting_state_bitwise(oracle):
    V, z = md.resting_state()
    Vo, zo = oracle.resting_state()
    assert V == Vo and np.array_equal(z, zo)
    assert V == -64.99637933119206


@pytest.mark.parametrize("n_z,nranks", [(256, 8), (25, 8), (50, 3), (100, 7), (8, 8), (128, 1)])
def test_partition_slab(n_z, nranks):
    lib = capi.load()
    parts = []
    for r in range(nranks):
        pt = capi.Partition()
        assert lib.emrkc_partition_slab(n_z, nranks, r, C.byref(pt)) == 0
        parts.append((pt.z_begin, pt.z_end))
    assert parts[0][0] == 0 and parts[-1][1] == n_z
    for a, b in zip(parts, parts[1:]):
        assert a[1] == b[0]
    sizes = [e - b for b, e in parts]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    pt = capi.Partition()
    assert lib.emrkc_partition_slab(4, 8, 0, C.byref(pt)) == capi.EMRKC_EINVAL


def test_state_len():
    lib = capi.load()
    w = workloads.hh3d_128()
    assert lib.emrkc_state_len(C.byref(w.problem), None) == 4 * 128 ** 3
    pt = capi.Partition(10, 42)
    assert lib.emrkc_state_len(C.byref(w.problem), C.byref(pt)) == 4 * 128 * 128 * 32


def test_create_validates_problem():
    lib = capi.load()
    p = md.make_problem(2, [1, 10], [0.1, 0.1], [0.1, 0.1])
    h = C.c_void_p()
    assert lib.emrkc_create(C.byref(p), 0, None, C.byref(h)) == capi.EMRKC_EINVAL
    assert b"grid" in lib.emrkc_global_error()


def test_no_device_fails_loudly():
    """On a machine without a GPU the product path refuses (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(md.CudaError, match="no CUDA device"):
        md.MonodomainOperator(workloads.hh2d_256().problem)


def test_workloads_match_baseline_configs():
    w1 = workloads.hh2d_256()
    assert w1.n_nodes == 65536 and w1.n_steps == 200
    w2 = workloads.hh3d_128()
    assert w2.n_nodes == 2097152 and w2.n_steps == 100
    w4 = workloads.hh3d_512x512x256()
    assert w4.n_nodes == 67108864 and w4.n_steps == 200
    w3 = workloads.hh3d_256x256x128()
    assert w3.n_nodes == 8388608 and w3.n_steps == 400
    for N in (25, 50, 100, 200):
        assert workloads.hh3d_sweep(N).n_nodes == N ** 3


def test_stimulus_boxes_select_the_named_nodes(oracle):
    """Half-cell margins pick exactly the BASELINE node boxes."""
    w = workloads.hh2d_256()
    p = w.problem
    inside = [oracle.stimulus_rate(p, 0.5, i + 256 * j) > 0 for j in range(20) for i in range(20)]
    inside = np.array(inside).reshape(20, 20)
    assert inside[:16, :16].all() and not inside[16:, :].any() and not inside[:, 16:].any()
    assert oracle.stimulus_rate(p, 1.0, 0) > 0 and oracle.stimulus_rate(p, 1.0 + 1e-9, 0) == 0


def test_generic_layer_no_device_fails_loudly():
    """The generic integrator layer has no CPU fallback either."""
    import ctypes as C

    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    h = C.c_void_p()
    assert capi.load().emrkc_vctx_create(0, C.byref(h)) == capi.EMRKC_ECUDA


def test_model_formulas_bit_identical(oracle):
    """IonicModel adapter entry points (emrkc_model_rates / _ionic_current)
    against the oracle's restatement of P/src/ionic.cpp:98-116."""
    import ctypes as C

    lib = capi.load()
    a = np.zeros(3)
    b = np.zeros(3)
    cur = C.c_double()
    for V in np.linspace(-120.0, 80.0, 401):
        assert lib.emrkc_model_rates(0, V, capi.dptr(a), capi.dptr(b)) == 0
        ra, rb = oracle.rates(V)
        assert np.array_equal(a, ra) and np.array_equal(b, rb)
        z = np.array([0.05, 0.6, 0.3])
        assert lib.emrkc_model_ionic_current(0, V, capi.dptr(z), C.byref(cur)) == 0
        assert cur.value == oracle.ionic_current(V, z)
    assert lib.emrkc_model_rates(7, 0.0, capi.dptr(a), capi.dptr(b)) == capi.EMRKC_EINVAL
