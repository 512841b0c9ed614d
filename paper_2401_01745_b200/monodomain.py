"""Python mirror of the reference's interface for the emRKC path.

Names, argument meaning and error behaviour follow the reference's C++ API
(P/ = /root/reference/proj/):

* ``get_stages`` / ``rkc_coeffs``      — P/include/mrkc/cheb.hpp:53-63
* ``MonodomainOperator``              — P/include/mrkc/monodomain.hpp:119-176
  (``f_F``, ``f_S``, ``exp_part``, ``initial_state``, ``layout``)
* ``SplitRhs`` + ``emrkc_step``        — P/include/mrkc/multirate.hpp:25-81
* ``estimate_spectral_radius``         — P/include/mrkc/spectral.hpp:28-29
* ``run_emrkc``                        — the emRKC branch of run_simulation
  (P/src/simulate.cpp:151-229)
* ``NumericalAbort``                   — P/include/mrkc/core.hpp:18-24

Everything computes on the GPU through the C ABI (include/emrkc.h); this
module only marshals host buffers. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import Partition, Problem, RhoResult, RunResult, StepReport, dptr

kDefaultDamping = 0.05


class NumericalAbort(RuntimeError):
    """Non-finite stage or norm guard (P/include/mrkc/core.hpp:18-24)."""

    def __init__(self, what: str, stage: int = -1, step_index: int = -1, inner: bool = False):
        super().__init__(what)
        self.stage = stage
        self.step_index = step_index
        self.inner = inner


class CudaError(RuntimeError):
    pass


def _lib():
    return capi.load()


def _check(rc: int, handle=None):
    if rc == capi.EMRKC_OK:
        return
    lib = _lib()
    msg = (lib.emrkc_last_error(handle) if handle else lib.emrkc_global_error()).decode()
    if rc == capi.EMRKC_EINVAL:
        raise ValueError(msg)
    if rc == capi.EMRKC_ENONFINITE:
        raise NumericalAbort(msg)
    if rc == capi.EMRKC_ESTATE:
        raise RuntimeError(msg)
    raise CudaError(msg)


# ---- integrator numerics (host) ---------------------------------------------

@dataclass
class StagePlan:
    s: int
    ell: float
    beta: float


def get_stages(dt: float, rho: float, epsilon: float = kDefaultDamping) -> StagePlan:
    s = C.c_int32()
    ell = C.c_double()
    beta = C.c_double()
    _check(_lib().emrkc_get_stages(dt, rho, epsilon, C.byref(s), C.byref(ell), C.byref(beta)))
    return StagePlan(s.value, ell.value, beta.value)


@dataclass
class RkcCoeffs:
    s: int
    epsilon: float
    omega0: float
    omega1: float
    b: np.ndarray
    mu: np.ndarray
    nu: np.ndarray
    kappa: np.ndarray
    c: np.ndarray


def rkc_coeffs(s: int, epsilon: float = kDefaultDamping) -> RkcCoeffs:
    n = max(int(s), 0) + 1
    arr = {k: np.zeros(n) for k in ("b", "mu", "nu", "kappa", "c")}
    w0 = C.c_double()
    w1 = C.c_double()
    _check(_lib().emrkc_rkc_coeffs(s, epsilon, C.byref(w0), C.byref(w1),
                                   *(dptr(arr[k]) for k in ("b", "mu", "nu", "kappa", "c"))))
    return RkcCoeffs(s, epsilon, w0.value, w1.value, **arr)


def plan_step(dt: float, rho_F: float, rho_S: float, epsilon: float = kDefaultDamping) -> StepReport:
    rep = StepReport()
    _check(_lib().emrkc_plan_step(dt, rho_F, rho_S, epsilon, C.byref(rep)))
    return rep


def resting_state(model: int = capi.EMRKC_MODEL_HH):
    V = C.c_double()
    z = np.zeros(3)
    _check(_lib().emrkc_resting_state(model, C.byref(V), dptr(z)))
    return V.value, z


# ---- problem + operator -----------------------------------------------------

def make_problem(dim: int, n, dx, sigma, chi=140.0, C_m=0.01, stim_amplitude=0.0,
                 stim_lo=(0.0, 0.0, 0.0), stim_hi=(0.0, 0.0, 0.0), stim_t0=0.0,
                 stim_t1=0.0, n_aux: int = 0) -> Problem:
    """Problem struct (grid by node counts; units mm, ms, mS/mm, uA/mm^3).
    n_aux > 0 selects EMRKC_MODEL_HH_AUX, the SYNTHETIC width stand-in (HH
    plus n_aux passive auxiliary variables; include/emrkc.h)."""
    p = Problem()
    p.dim = dim
    p.model = capi.EMRKC_MODEL_HH_AUX if n_aux else capi.EMRKC_MODEL_HH
    p.n_aux = n_aux
    n = list(n) + [1] * (3 - len(n))
    dx = list(dx) + [0.0] * (3 - len(dx))
    sigma = list(sigma) + [0.0] * (3 - len(sigma))
    for a in range(3):
        p.n[a] = int(n[a]) if a < dim else 1
        p.dx[a] = float(dx[a]) if a < dim else 0.0
        p.sigma[a] = float(sigma[a]) if a < dim else 0.0
        p.stim_lo[a] = float(stim_lo[a]) if a < len(stim_lo) else 0.0
        p.stim_hi[a] = float(stim_hi[a]) if a < len(stim_hi) else 0.0
    p.chi = chi
    p.C_m = C_m
    p.stim_chi_amplitude = stim_amplitude
    p.stim_t0 = stim_t0
    p.stim_t1 = stim_t1
    return p


@dataclass
class StateLayout:
    """P/include/mrkc/monodomain.hpp:51-60"""

    n_nodes: int
    n_gates: int = 3
    n_aux: int = 0

    def size(self) -> int:
        return self.n_nodes * (1 + self.n_gates + self.n_aux)

    def v_offset(self) -> int:
        return 0

    def gate_offset(self, g: int) -> int:
        return self.n_nodes * (1 + g)

    def aux_offset(self, a: int) -> int:
        return self.n_nodes * (1 + self.n_gates + a)


@dataclass
class RhoEstimate:
    """P/include/mrkc/spectral.hpp:10-16"""

    rho: float
    iterations: int
    converged: bool
    safety: float = 1.05
    v: np.ndarray | None = None


class MonodomainOperator:
    """Device-resident monodomain operator (one z-slab or the whole grid).

    Replaces ``mrkc::MonodomainOperator`` + the SplitRhs binding of
    run_simulation (P/src/simulate.cpp:153-157). The state lives in HBM;
    ``set_state``/``get_state`` move it in reference Vec layout.
    """

    def __init__(self, problem: Problem, device: int = 0, partition: Partition | None = None):
        self.problem = problem
        self.partition = partition
        h = C.c_void_p()
        _check(_lib().emrkc_create(C.byref(problem), device,
                                   C.byref(partition) if partition is not None else None,
                                   C.byref(h)))
        self._h = h
        self.len = int(_lib().emrkc_local_len(h))
        self.layout_ = StateLayout(self.len // problem.n_fields, 3, int(problem.n_aux))

    def close(self):
        if self._h:
            _lib().emrkc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def layout(self) -> StateLayout:
        return self.layout_

    def initial_state(self) -> np.ndarray:
        """Uniform resting state (P/src/monodomain.cpp:306-319) of this
        handle's slab (the whole grid without a partition)."""
        p = self.problem
        y = np.empty(p.state_len())
        _check(_lib().emrkc_initial_state(C.byref(p), dptr(y), y.size))
        if self.partition is None:
            return y
        nn, nf = p.n_nodes, p.n_fields
        plane = nn // int(p.n[p.dim - 1])
        a, b = int(self.partition.z_begin) * plane, int(self.partition.z_end) * plane
        return np.concatenate([y[k * nn + a:k * nn + b] for k in range(nf)])

    def set_state(self, y: np.ndarray):
        y = np.ascontiguousarray(y, dtype=np.float64)
        _check(_lib().emrkc_set_state(self._h, dptr(y), y.size), self._h)

    def get_state(self) -> np.ndarray:
        y = np.empty(self.len)
        _check(_lib().emrkc_get_state(self._h, dptr(y), y.size), self._h)
        return y

    def synchronize(self):
        _check(_lib().emrkc_synchronize(self._h), self._h)

    # SplitRhs callbacks evaluated on the device (host buffers in/out)
    def f_F(self, t: float, y: np.ndarray) -> np.ndarray:
        return self._rhs(capi.EMRKC_RHS_F, t, y)

    def f_S(self, t: float, y: np.ndarray) -> np.ndarray:
        return self._rhs(capi.EMRKC_RHS_S, t, y)

    def _rhs(self, which, t, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.empty_like(y)
        _check(_lib().emrkc_eval_rhs(self._h, which, t, dptr(y), dptr(out), y.size), self._h)
        return out

    def exp_part(self, y: np.ndarray):
        y = np.ascontiguousarray(y, dtype=np.float64)
        lam = np.empty_like(y)
        yinf = np.empty_like(y)
        _check(_lib().emrkc_exp_part(self._h, dptr(y), dptr(lam), dptr(yinf), y.size), self._h)
        return lam, yinf

    def estimate_spectral_radius(self, which: int, t: float = 0.0, v0: np.ndarray | None = None,
                                 rho0: float = 0.0, want_v: bool = False) -> RhoEstimate:
        """Power iteration on the current device state (P/src/spectral.cpp:26-71)."""
        res = RhoResult()
        v = np.empty(self.len) if want_v else None
        v0c = None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
        _check(_lib().emrkc_estimate_rho(self._h, which, t, dptr(v0c), rho0, C.byref(res), dptr(v)), self._h)
        return RhoEstimate(res.rho, res.iterations, bool(res.converged), res.safety, v)

    def step(self, t: float, dt: float, rho_F: float, rho_S: float,
             epsilon: float = kDefaultDamping,
             variant: int = capi.EMRKC_VARIANT_STANDARD) -> StepReport:
        """One emRKC step of the device-resident state (P/src/multirate.cpp:173-189)."""
        rep = StepReport()
        rc = _lib().emrkc_step(self._h, t, dt, epsilon, variant, rho_F, rho_S, C.byref(rep))
        if rc == capi.EMRKC_ENONFINITE:
            raise NumericalAbort(_lib().emrkc_last_error(self._h).decode(), rep.abort_stage,
                                 inner=bool(rep.abort_inner))
        _check(rc, self._h)
        return rep

    # ---- distributed slabs (paper_2401_01745_b200/dist.py) ----
    def ipc_export(self) -> bytes:
        n = int(_lib().emrkc_ipc_blob_size())
        buf = C.create_string_buffer(n)
        _check(_lib().emrkc_ipc_export(self._h, buf, n), self._h)
        return buf.raw

    def ipc_import(self, side: int, blob: bytes):
        _check(_lib().emrkc_ipc_import(self._h, side, blob, len(blob)), self._h)

    def set_slab_min_depth(self, planes: int):
        """Smallest slab depth of the partition: enables the K-plane d_1 halo
        of the temporally blocked inner stages (emrkc_set_slab_min_depth)."""
        _check(_lib().emrkc_set_slab_min_depth(self._h, int(planes)), self._h)

    def dist_run(self, step0, nsteps, dt, rho_F, rho_S, epsilon=kDefaultDamping) -> dict:
        res = RunResult()
        _check(_lib().emrkc_dist_run(self._h, step0, nsteps, dt, epsilon, capi.EMRKC_VARIANT_STANDARD,
                                     rho_F, rho_S, C.byref(res)), self._h)
        return res.as_dict()

    def dist_replay(self, step0, nsteps, dt, rho_F, rho_S, epsilon=kDefaultDamping) -> dict:
        res = RunResult()
        _check(_lib().emrkc_dist_replay(self._h, step0, nsteps, dt, epsilon,
                                        capi.EMRKC_VARIANT_STANDARD, rho_F, rho_S, C.byref(res)),
               self._h)
        return res.as_dict()

    def run_timed_dist(self, step0, nsteps, dt, rho_F, rho_S, epsilon=kDefaultDamping,
                       flush_bytes=256 << 20):
        rep = plan_step(dt, rho_F, rho_S, epsilon)
        launch_ms = np.zeros(nsteps * rep.s * rep.m)
        res = RunResult()
        _check(_lib().emrkc_run_timed(self._h, step0, nsteps, dt, epsilon, capi.EMRKC_VARIANT_STANDARD,
                                      rho_F, rho_S, flush_bytes, dptr(launch_ms), launch_ms.size,
                                      C.byref(res)), self._h)
        return launch_ms, res.as_dict()

    def run(self, step0: int, nsteps: int, dt: float, rho_F: float, rho_S: float,
            epsilon: float = kDefaultDamping,
            variant: int = capi.EMRKC_VARIANT_STANDARD) -> RunResult:
        """run_simulation's emRKC loop on the device (P/src/simulate.cpp:176-229);
        variant: EmrkcVariant (Method::emrkc / emrkc_progressive)."""
        res = RunResult()
        _check(_lib().emrkc_run(self._h, step0, nsteps, dt, epsilon, variant,
                                rho_F, rho_S, C.byref(res)), self._h)
        return res

    def rel_l2_error(self, ref: np.ndarray, block: int = 0) -> float:
        """rel_l2_error of SoA block ``block`` of the device state against a
        host field (P/src/monodomain.cpp:88-110), reduced on the device."""
        ref = np.ascontiguousarray(ref, dtype=np.float64)
        out = C.c_double(0.0)
        _check(_lib().emrkc_rel_l2_error(self._h, block, dptr(ref), 0, C.byref(out)), self._h)
        return out.value

    # ---- mRKC with the stiff-gate split (P/src/multirate.cpp:158-171) ----
    def set_stiff_gates(self, mask: int):
        """Gates (bit g) in the fast part f_F (P/src/simulate.cpp:132-150)."""
        _check(_lib().emrkc_set_stiff_gates(self._h, mask), self._h)

    def mrkc_step(self, t: float, dt: float, rho_F: float, rho_S: float,
                  epsilon: float = kDefaultDamping) -> StepReport:
        rep = StepReport()
        rc = _lib().emrkc_mrkc_step(self._h, t, dt, epsilon, rho_F, rho_S, C.byref(rep))
        if rc == capi.EMRKC_ENONFINITE:
            raise NumericalAbort(_lib().emrkc_last_error(self._h).decode(), rep.abort_stage,
                                 inner=bool(rep.abort_inner))
        _check(rc, self._h)
        return rep

    def mrkc_run(self, step0: int, nsteps: int, dt: float, rho_F: float, rho_S: float,
                 epsilon: float = kDefaultDamping) -> RunResult:
        res = RunResult()
        _check(_lib().emrkc_mrkc_run(self._h, step0, nsteps, dt, epsilon, rho_F, rho_S,
                                     C.byref(res)), self._h)
        return res

    # ---- IMEX-RL (P/src/baselines.cpp:132-190) ----
    def imex_step(self, t: float, dt: float, rel_tol: float = 1e-8, max_iters: int = 0,
                  jacobi: bool = True):
        """One IMEX-RL step; returns (report, CG iterations)."""
        rep = StepReport()
        it = C.c_int64(0)
        rc = _lib().emrkc_imex_step(self._h, t, dt, rel_tol, max_iters, int(jacobi),
                                    C.byref(rep), C.byref(it))
        if rc == capi.EMRKC_ENONFINITE:
            raise NumericalAbort(_lib().emrkc_last_error(self._h).decode(), -1)
        _check(rc, self._h)
        return rep, it.value

    def imex_run(self, step0: int, nsteps: int, dt: float, rel_tol: float = 1e-8,
                 max_iters: int = 0, jacobi: bool = True):
        """run_simulation's imex_rl loop; returns (RunResult, cg_iters_total)."""
        res = RunResult()
        it = C.c_int64(0)
        _check(_lib().emrkc_imex_run(self._h, step0, nsteps, dt, rel_tol, max_iters, int(jacobi),
                                     C.byref(res), C.byref(it)), self._h)
        return res, it.value

    def exex_step(self, t: float, dt: float) -> StepReport:
        """One EXEX-RL step of the device state (exex_rl_step,
        P/src/baselines.cpp:192-210); never raises NumericalAbort."""
        rep = StepReport()
        _check(_lib().emrkc_exex_step(self._h, t, dt, C.byref(rep)), self._h)
        return rep

    def exex_run(self, step0: int, nsteps: int, dt: float) -> RunResult:
        """run_simulation's exex_rl loop (P/src/simulate.cpp:164-165,176-229)."""
        res = RunResult()
        _check(_lib().emrkc_exex_run(self._h, step0, nsteps, dt, C.byref(res)), self._h)
        return res


@dataclass
class SplitRhs:
    """P/include/mrkc/multirate.hpp:25-35, bound to a device operator."""

    op: MonodomainOperator
    rho_F: float = 0.0
    rho_S: float = 0.0
    counters: dict = field(default_factory=lambda: {"n_fF": 0, "n_fS": 0, "n_exp_steps": 0})


def bind_split_rhs(op: MonodomainOperator) -> SplitRhs:
    return SplitRhs(op)


def estimate_spectral_radius(op: MonodomainOperator, which: int, y: np.ndarray, t: float = 0.0,
                             v0=None, rho0: float = 0.0) -> RhoEstimate:
    op.set_state(y)
    return op.estimate_spectral_radius(which, t, v0, rho0, want_v=True)


def emrkc_step(t: float, y: np.ndarray, dt: float, rhs: SplitRhs,
               epsilon: float = kDefaultDamping, report: StepReport | None = None,
               variant: int = capi.EMRKC_VARIANT_STANDARD) -> np.ndarray:
    """Drop-in of ``Vec emrkc_step(t, y, dt, rhs, eps, variant, report)``:
    host vector in, host vector out, one device step in between."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(y)
    rep = report if report is not None else StepReport()
    h = rhs.op.handle
    rc = _lib().emrkc_step_host(h, t, dptr(y), dptr(out), y.size, dt, epsilon,
                                variant, rhs.rho_F, rhs.rho_S, C.byref(rep))
    if rc == capi.EMRKC_ENONFINITE:
        raise NumericalAbort(_lib().emrkc_last_error(h).decode(), rep.abort_stage,
                             inner=bool(rep.abort_inner))
    _check(rc, h)
    rhs.counters["n_fF"] += rep.n_fF
    rhs.counters["n_fS"] += rep.n_fS
    rhs.counters["n_exp_steps"] += rep.n_exp
    return out


def identify_stiff_gates(V: np.ndarray, model: int = capi.EMRKC_MODEL_HH) -> list:
    """identify_stiff_gates (P/src/ionic.cpp:130-146): gates by their largest
    alpha + beta over the V samples, stiffest first."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    out = (C.c_int32 * 3)()
    _check(_lib().emrkc_identify_stiff_gates(model, dptr(V), V.size, out))
    return list(out)


def exex_rl_step(t: float, y: np.ndarray, dt: float, op: MonodomainOperator) -> np.ndarray:
    """Drop-in of ``Vec exex_rl_step(t, y, dt, prob, counters)``
    (P/src/baselines.cpp:192-210): host vector in, one device step, host out."""
    op.set_state(np.ascontiguousarray(y, dtype=np.float64))
    op.exex_step(t, dt)
    return op.get_state()


def run_emrkc(problem: Problem, y0: np.ndarray, dt: float, n_steps: int,
              epsilon: float = kDefaultDamping, device: int = 0, rho=None):
    """run_simulation's emRKC branch: estimate rho_F, rho_S once at t = 0
    (P/src/simulate.cpp:158-159), then step with t = step*dt. Returns
    (final_state, RunResult, (rho_F, rho_S))."""
    op = MonodomainOperator(problem, device)
    try:
        op.set_state(y0)
        if rho is None:
            rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F, 0.0).rho
            rS = op.estimate_spectral_radius(capi.EMRKC_RHS_S, 0.0).rho
        else:
            rF, rS = rho
        res = op.run(0, n_steps, dt, rF, rS, epsilon)
        return op.get_state(), res, (rF, rS)
    finally:
        op.close()
