"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU checkers.

* ``Oracle``   : our plain-C restatement (oracle/liboracle.so, built from
                 oracle/emrkc_oracle.c).
* ``Reference``: the reference's own sources compiled in place
                 (oracle/_ref/libmrkc_ref.so, built by oracle/Makefile from
                 /root/reference/proj/src + oracle/ref_driver.cpp).

Both expose the same Python surface so tests can run a case through either.
Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2401_01745_b200.capi import (
    DP,
    I32P,
    Problem,
    RhoResult,
    RunResult,
    StepReport,
    dptr,
)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmrkc_ref.so")

RHS_CB = C.CFUNCTYPE(None, C.c_double, DP, DP, C.c_int64, C.c_void_p)
OC_RHS_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_double, DP, DP, C.c_int64)

PP = C.POINTER(Problem)


def _sigs(pre: str):
    s = {
        "resting_state": (C.c_int, [DP, DP]),
        "hh_rates": (None, [C.c_double, DP, DP]),
        "gate_coeffs": (None, [C.c_double, DP, DP]),
        "ionic_current": (C.c_double, [C.c_double, DP]),
        "initial_state": (C.c_int, [PP, DP]),
        "exp_part": (None, [PP, DP, DP, DP]),
        "stimulus_rate": (C.c_double, [PP, C.c_double, C.c_int64]),
        "estimate_rho": (C.c_int, [PP, C.c_int32, C.c_double, DP, DP, C.c_double, C.POINTER(RhoResult), DP]),
        "run": (C.c_int, [PP, DP, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(RunResult), DP]),
        "run_method": (C.c_int, [PP, DP, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_double, C.c_double, C.POINTER(RunResult), DP]),
        "rel_l2_error": (C.c_double, [PP, DP, DP]),
        "identify_stiff_gates": (C.c_int, [DP, C.c_int64, I32P]),
        "run_imex": (C.c_int, [PP, DP, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_int32, C.POINTER(RunResult), C.POINTER(C.c_int64)]),
        "analytic_rho_F": (C.c_double, [PP]),
        "get_stages": (C.c_int, [C.c_double, C.c_double, C.c_double, I32P, DP, DP]),
        "rkc_coeffs": (C.c_int, [C.c_int32, C.c_double, DP, DP, DP, DP, DP, DP, DP]),
        "phi": (C.c_double, [C.c_double]),
        "last_error": (C.c_char_p, []),
    }
    if pre == "ref_":
        s["hh_rates"] = (C.c_int, [C.c_double, DP, DP])
        s["gate_coeffs"] = (C.c_int, [C.c_double, DP, DP])
        s["exp_part"] = (C.c_int, [PP, DP, DP, DP])
        s["rhs"] = (C.c_int, [PP, C.c_int, C.c_double, DP, DP])
        s["emrkc_step"] = (C.c_int, [PP, C.c_double, DP, C.c_double, C.c_double, C.c_double, C.c_double, DP, C.POINTER(StepReport)])
        s["estimate_rho_cb"] = (C.c_int, [RHS_CB, C.c_void_p, C.c_int64, C.c_double, DP, DP, C.c_double, C.POINTER(RhoResult), DP])
        s["bench"] = (C.c_int, [PP, DP, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32, DP])
        s["rkc_iteration_scalar"] = (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_double, DP])
        s["averaged_force_emrkc_scalar"] = (C.c_int, [C.c_double] * 6 + [C.c_int32, C.c_double, DP])
        s["emrkc_step_scalar"] = (C.c_int, [C.c_double] * 7 + [DP, I32P, I32P, DP])
        s["exponential_euler_step"] = (C.c_int, [DP, C.c_double, DP, DP, C.c_int64, DP])
        s["std_uniform_direction"] = (None, [C.c_uint64, C.c_int64, DP])
        s["std_normal"] = (None, [C.c_uint64, C.c_double, C.c_double, C.c_int64, DP])
        s["state_len"] = (C.c_int64, [PP])
        s["rhs_gates"] = (C.c_int, [PP, C.c_int, C.c_int, C.c_double, DP, DP])
    else:
        s["hh_rates"] = (None, [C.c_double, DP, DP])
        s["f_F"] = (None, [PP, C.c_double, DP, DP])
        s["f_S"] = (None, [PP, C.c_double, DP, DP])
        s["emrkc_step_grid"] = (C.c_int, [PP, C.c_double, DP, C.c_double, C.c_double, C.c_double, C.c_double, DP, C.POINTER(StepReport)])
        s["estimate_rho_cb"] = (C.c_int, [OC_RHS_CB, C.c_void_p, C.c_int64, C.c_double, DP, DP, C.c_double, C.POINTER(RhoResult), DP])
        s["rkc_iteration"] = (C.c_int, [C.c_double, DP, C.c_int64, C.c_double, OC_RHS_CB, C.c_void_p, C.c_int32, C.c_double, DP, I32P])
        s["exponential_euler_step"] = (None, [DP, C.c_double, DP, DP, C.c_int64, DP])
        s["mt19937_64_uniform"] = (None, [C.c_uint64, C.c_int64, DP])
        s["state_len"] = (C.c_int64, [PP])
        s["diffusion_apply"] = (None, [PP, DP, DP])
        s["hh_gate_coeffs"] = (None, [C.c_double, DP, DP])
        s["hh_ionic_current"] = (C.c_double, [C.c_double, DP])
        s["hh_resting_state"] = (C.c_int, [DP, DP])
        s["scalar_averaged_force"] = (C.c_int, [C.c_double] * 6 + [C.c_int32, C.c_double, DP])
        s["scalar_emrkc_step"] = (C.c_int, [C.c_double] * 7 + [DP, I32P, I32P, DP])
        s["exex_rl_step"] = (C.c_int, [PP, C.c_double, DP, C.c_double, DP])
        s["f_F_gates"] = (None, [PP, C.c_int32, C.c_double, DP, DP])
        s["f_S_gates"] = (None, [PP, C.c_int32, C.c_double, DP, DP])
        s.pop("gate_coeffs")
        s.pop("ionic_current")
        s.pop("resting_state")
    return s


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} missing (run make -C oracle)")
        self.lib = C.CDLL(self.path)
        for name, (res, args) in _sigs(self.prefix).items():
            fn = getattr(self.lib, self.prefix + name)
            fn.restype = res
            fn.argtypes = args

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def err(self) -> str:
        return self.fn("last_error")().decode()

    # ---- grid-level API (same for both libraries) ----
    def initial_state(self, p: Problem) -> np.ndarray:
        y = np.empty(p.state_len())
        rc = self.fn("initial_state")(C.byref(p), dptr(y))
        assert rc == 0, self.err()
        return y

    def exp_part(self, p: Problem, y: np.ndarray):
        lam = np.empty_like(y)
        yinf = np.empty_like(y)
        self.fn("exp_part")(C.byref(p), dptr(y), dptr(lam), dptr(yinf))
        return lam, yinf

    def stimulus_rate(self, p: Problem, t: float, node: int) -> float:
        return self.fn("stimulus_rate")(C.byref(p), t, node)

    def estimate_rho(self, p: Problem, which: int, t: float, y: np.ndarray, v0=None, rho0=0.0):
        res = RhoResult()
        v = np.empty_like(y)
        rc = self.fn("estimate_rho")(C.byref(p), which, t, dptr(y), dptr(v0), rho0, C.byref(res), dptr(v))
        if rc:
            raise ValueError(self.err())
        return res, v

    def run(self, p: Problem, y: np.ndarray, step0: int, nsteps: int, dt: float, eps: float,
            rho_F: float, rho_S: float):
        y = np.ascontiguousarray(y, dtype=np.float64).copy()
        res = RunResult()
        wall = C.c_double(0.0)
        rc = self.fn("run")(C.byref(p), dptr(y), step0, nsteps, dt, eps, rho_F, rho_S, C.byref(res), C.byref(wall))
        if rc:
            raise ValueError(self.err())
        return y, res, wall.value

    # Method codes of run_method (P/include/mrkc/config.hpp:17); MRKC takes
    # the stiff gate mask in bits 4..6
    EMRKC, EMRKC_PROGRESSIVE, EXEX_RL, MRKC = 0, 1, 2, 3
    # estimate_rho / rhs selectors for the mRKC split: f_F / f_S with gate rows
    RHS_F_GATES, RHS_S_GATES = 2, 3

    def run_mrkc(self, p: Problem, y: np.ndarray, step0: int, nsteps: int, dt: float,
                 stiff: int, eps: float = 0.05, rho_F: float = 0.0, rho_S: float = 0.0):
        """run_simulation's mrkc loop (P/src/simulate.cpp:191-195) with the
        stiff-gate split (gate mask ``stiff``)."""
        return self.run_method(p, y, step0, nsteps, dt, self.MRKC | (stiff << 4), eps, rho_F,
                               rho_S)

    def estimate_rho_gates(self, p: Problem, which: int, stiff: int, t: float, y: np.ndarray):
        """power iteration on f_F_with_gates (which 2) / f_S_with_gates (3)."""
        return self.estimate_rho(p, which | (stiff << 4), t, y)

    def run_imex(self, p: Problem, y: np.ndarray, step0: int, nsteps: int, dt: float,
                 rel_tol: float = 1e-8, max_iters: int = 0, jacobi: bool = True):
        """run_simulation's imex_rl loop; returns (state, RunResult, cg_iters_total)."""
        y = np.ascontiguousarray(y, dtype=np.float64).copy()
        res = RunResult()
        it = C.c_int64(0)
        rc = self.fn("run_imex")(C.byref(p), dptr(y), step0, nsteps, dt, rel_tol, max_iters,
                                 int(jacobi), C.byref(res), C.byref(it))
        if rc:
            raise ValueError(self.err())
        return y, res, it.value

    def identify_stiff_gates(self, V: np.ndarray):
        V = np.ascontiguousarray(V, dtype=np.float64)
        out = (C.c_int32 * 3)()
        rc = self.fn("identify_stiff_gates")(dptr(V), V.size, out)
        if rc:
            raise ValueError(self.err())
        return list(out)

    def run_method(self, p: Problem, y: np.ndarray, step0: int, nsteps: int, dt: float,
                   method: int, eps: float = 0.05, rho_F: float = 0.0, rho_S: float = 0.0):
        """run_simulation's loop for emrkc (0), emrkc_progressive (1), exex_rl (2)."""
        y = np.ascontiguousarray(y, dtype=np.float64).copy()
        res = RunResult()
        wall = C.c_double(0.0)
        rc = self.fn("run_method")(C.byref(p), dptr(y), step0, nsteps, dt, eps, method, rho_F,
                                   rho_S, C.byref(res), C.byref(wall))
        if rc:
            raise ValueError(self.err())
        return y, res, wall.value

    def rel_l2(self, p: Problem, a: np.ndarray, b: np.ndarray) -> float:
        return self.fn("rel_l2_error")(C.byref(p), dptr(np.ascontiguousarray(a)), dptr(np.ascontiguousarray(b)))

    def analytic_rho_F(self, p: Problem) -> float:
        return self.fn("analytic_rho_F")(C.byref(p))

    def get_stages(self, dt, rho, eps):
        s = C.c_int32()
        ell = C.c_double()
        beta = C.c_double()
        rc = self.fn("get_stages")(dt, rho, eps, C.byref(s), C.byref(ell), C.byref(beta))
        if rc:
            raise ValueError(self.err())
        return s.value, ell.value, beta.value

    def rkc_coeffs(self, s: int, eps: float) -> dict:
        arrs = {k: np.zeros(s + 1) for k in ("b", "mu", "nu", "kappa", "c")}
        w0 = C.c_double()
        w1 = C.c_double()
        rc = self.fn("rkc_coeffs")(s, eps, C.byref(w0), C.byref(w1), *(dptr(arrs[k]) for k in ("b", "mu", "nu", "kappa", "c")))
        if rc:
            raise ValueError(self.err())
        arrs["omega0"] = w0.value
        arrs["omega1"] = w1.value
        return arrs

    def phi(self, z: float) -> float:
        return self.fn("phi")(z)


class _Scalar:
    """Scalar-surrogate split of the reference tests
    (P/tests/test_multirate.cpp:54-66)."""

    _af = "scalar_averaged_force"
    _st = "scalar_emrkc_step"

    def averaged_force_emrkc(self, lF, lS, lE, yinf, y, eta, m, eps=0.05):
        out = C.c_double()
        rc = self.fn(self._af)(lF, lS, lE, yinf, y, eta, m, eps, C.byref(out))
        if rc:
            raise ValueError(self.err())
        return out.value

    def emrkc_step_scalar(self, lF, lS, lE, yinf, y, dt, eps=0.05):
        out = C.c_double()
        s = C.c_int32()
        m = C.c_int32()
        eta = C.c_double()
        rc = self.fn(self._st)(lF, lS, lE, yinf, y, dt, eps, C.byref(out), C.byref(s), C.byref(m), C.byref(eta))
        if rc:
            raise ValueError(self.err())
        return out.value, s.value, m.value, eta.value


class Oracle(_Scalar, _Lib):
    """Plain-C restatement (oracle/emrkc_oracle.c)."""

    prefix = "oc_"
    path = ORACLE_LIB

    def resting_state(self):
        V = C.c_double()
        z = np.zeros(3)
        rc = self.fn("hh_resting_state")(C.byref(V), dptr(z))
        assert rc == 0
        return V.value, z

    def rates(self, V):
        a = np.zeros(3)
        b = np.zeros(3)
        self.fn("hh_rates")(V, dptr(a), dptr(b))
        return a, b

    def gate_coeffs(self, V):
        lam = np.zeros(3)
        zi = np.zeros(3)
        self.fn("hh_gate_coeffs")(V, dptr(lam), dptr(zi))
        return lam, zi

    def ionic_current(self, V, z):
        return self.fn("hh_ionic_current")(V, dptr(np.ascontiguousarray(z, dtype=np.float64)))

    def rhs(self, p: Problem, which: int, t: float, y: np.ndarray) -> np.ndarray:
        out = np.empty_like(y)
        self.fn("f_F" if which == 0 else "f_S")(C.byref(p), t, dptr(y), dptr(out))
        return out

    def rhs_gates(self, p: Problem, which: int, stiff: int, t: float, y: np.ndarray):
        """f_F_with_gates (which 0) / f_S_with_gates (1), P/src/monodomain.cpp:287-304."""
        out = np.empty_like(y)
        self.fn("f_F_gates" if which == 0 else "f_S_gates")(C.byref(p), stiff, t, dptr(y),
                                                            dptr(out))
        return out

    def emrkc_step(self, p, t, y, dt, eps, rho_F, rho_S):
        out = np.empty_like(y)
        rep = StepReport()
        rc = self.fn("emrkc_step_grid")(C.byref(p), t, dptr(y), dt, eps, rho_F, rho_S, dptr(out), C.byref(rep))
        return out, rep, rc

    def uniform_direction(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.fn("mt19937_64_uniform")(seed, n, dptr(out))
        return out

    def estimate_rho_fn(self, f, y, v0=None, rho0=0.0, t=0.0):
        n = len(y)

        @OC_RHS_CB
        def cb(ctx, tt, yp, outp, nn):
            yy = np.ctypeslib.as_array(yp, shape=(nn,))
            oo = np.ctypeslib.as_array(outp, shape=(nn,))
            oo[:] = f(tt, yy.copy())

        res = RhoResult()
        v = np.empty(n)
        y = np.ascontiguousarray(y, dtype=np.float64)
        rc = self.fn("estimate_rho_cb")(cb, None, n, t, dptr(y), dptr(None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)), rho0, C.byref(res), dptr(v))
        if rc:
            raise ValueError(self.err())
        return res, v

    def rkc_iteration(self, f, y, dt, s, eps, t=0.0):
        n = len(y)

        @OC_RHS_CB
        def cb(ctx, tt, yp, outp, nn):
            yy = np.ctypeslib.as_array(yp, shape=(nn,))
            oo = np.ctypeslib.as_array(outp, shape=(nn,))
            oo[:] = f(tt, yy.copy())

        out = np.empty(n)
        st = C.c_int32(0)
        y = np.ascontiguousarray(y, dtype=np.float64)
        rc = self.fn("rkc_iteration")(t, dptr(y), n, dt, cb, None, s, eps, dptr(out), C.byref(st))
        return out, rc, st.value

    def exponential_euler_step(self, y, eta, lam, yinf):
        y, lam, yinf = (np.ascontiguousarray(a, dtype=np.float64) for a in (y, lam, yinf))
        out = np.empty_like(y)
        self.fn("exponential_euler_step")(dptr(y), eta, dptr(lam), dptr(yinf), len(y), dptr(out))
        return out


class Reference(_Scalar, _Lib):
    """The reference's own sources, compiled in place (oracle/_ref)."""

    prefix = "ref_"
    path = REF_LIB
    _af = "averaged_force_emrkc_scalar"
    _st = "emrkc_step_scalar"

    def rkc_iteration_scalar(self, t, y0, dt, lam, s, eps):
        out = C.c_double()
        rc = self.fn("rkc_iteration_scalar")(t, y0, dt, lam, s, eps, C.byref(out))
        if rc:
            raise ValueError(self.err())
        return out.value

    def resting_state(self):
        V = C.c_double()
        z = np.zeros(3)
        rc = self.fn("resting_state")(C.byref(V), dptr(z))
        assert rc == 0
        return V.value, z

    def rates(self, V):
        a = np.zeros(3)
        b = np.zeros(3)
        self.fn("hh_rates")(V, dptr(a), dptr(b))
        return a, b

    def gate_coeffs(self, V):
        lam = np.zeros(3)
        zi = np.zeros(3)
        self.fn("gate_coeffs")(V, dptr(lam), dptr(zi))
        return lam, zi

    def ionic_current(self, V, z):
        return self.fn("ionic_current")(V, dptr(np.ascontiguousarray(z, dtype=np.float64)))

    def rhs(self, p: Problem, which: int, t: float, y: np.ndarray) -> np.ndarray:
        out = np.empty_like(y)
        rc = self.fn("rhs")(C.byref(p), which, t, dptr(y), dptr(out))
        assert rc == 0, self.err()
        return out

    def rhs_gates(self, p: Problem, which: int, stiff: int, t: float, y: np.ndarray):
        out = np.empty_like(y)
        rc = self.fn("rhs_gates")(C.byref(p), which, stiff, t, dptr(y), dptr(out))
        assert rc == 0, self.err()
        return out

    def emrkc_step(self, p, t, y, dt, eps, rho_F, rho_S):
        out = np.empty_like(y)
        rep = StepReport()
        rc = self.fn("emrkc_step")(C.byref(p), t, dptr(y), dt, eps, rho_F, rho_S, dptr(out), C.byref(rep))
        return out, rep, rc

    def uniform_direction(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.fn("std_uniform_direction")(seed, n, dptr(out))
        return out

    def estimate_rho_fn(self, f, y, v0=None, rho0=0.0, t=0.0):
        n = len(y)

        @RHS_CB
        def cb(tt, yp, outp, nn, ctx):
            yy = np.ctypeslib.as_array(yp, shape=(nn,))
            oo = np.ctypeslib.as_array(outp, shape=(nn,))
            oo[:] = f(tt, yy.copy())

        res = RhoResult()
        v = np.empty(n)
        y = np.ascontiguousarray(y, dtype=np.float64)
        rc = self.fn("estimate_rho_cb")(cb, None, n, t, dptr(y), dptr(None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)), rho0, C.byref(res), dptr(v))
        if rc:
            raise ValueError(self.err())
        return res, v

    def bench(self, p, y0, nsteps, dt, eps, rho_F, rho_S, nthreads):
        secs = np.zeros(nthreads)
        rc = self.fn("bench")(C.byref(p), dptr(np.ascontiguousarray(y0)), nsteps, dt, eps, rho_F, rho_S, nthreads, dptr(secs))
        if rc:
            raise ValueError(self.err())
        return secs


def have_reference() -> bool:
    return os.path.exists(REF_LIB)


def have_oracle() -> bool:
    return os.path.exists(ORACLE_LIB)
