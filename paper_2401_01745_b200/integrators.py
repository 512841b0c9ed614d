"""The reference's generic integrator layer on the device (include/emrkc.h,
``emrkc_generic.cu``): Python mirror of

* ``rkc_iteration(t, y, dt, f, s, epsilon)``        P/include/mrkc/cheb.hpp:60-63
* ``exponential_euler_step(y, eta, lambda, y_inf)``  P/include/mrkc/multirate.hpp:19
* ``averaged_force_emrkc`` / ``averaged_force_mrkc`` P/include/mrkc/multirate.hpp:57-67
* ``emrkc_step`` / ``mrkc_step`` over a generic SplitRhs   multirate.hpp:72-81
* ``estimate_spectral_radius(t, y, f, v0, rho0)``   P/include/mrkc/spectral.hpp:28-29

over arbitrary right-hand sides. The recurrences, exponential updates,
finite checks and power-iteration norms run in sm_100a kernels; a Python
callable ``f(t, y) -> out`` (numpy in, numpy out) is wrapped as a device
callback that reads its argument back from the device, calls ``f`` and
uploads the result (the reference's scalar known-answer tests run this way,
tests/test_gpu_integrators.py). ``bind(op)`` instead returns the SplitRhs of
a device MonodomainOperator, whose callbacks stay on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import capi
from .capi import Counters, RhoResult, SplitRhsC, StepReport, dptr
from .monodomain import CudaError, NumericalAbort, RhoEstimate, kDefaultDamping


def _lib():
    return capi.load()


class DeviceContext:
    """emrkc_vctx: a device + stream for the generic layer."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        rc = _lib().emrkc_vctx_create(device, C.byref(h))
        if rc:
            raise CudaError(f"emrkc_vctx_create failed ({rc}): no usable device")
        self.h = h
        self._bufs = []

    def close(self):
        if self.h:
            lib = _lib()
            for b in self._bufs:
                lib.emrkc_vctx_free(self.h, b)
            self._bufs = []
            lib.emrkc_vctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def err(self) -> str:
        return _lib().emrkc_vctx_last_error(self.h).decode()

    def check(self, rc: int, stage: int = -1, inner: bool = False):
        if rc == capi.EMRKC_OK:
            return
        msg = self.err()
        if rc == capi.EMRKC_EINVAL:
            raise ValueError(msg)
        if rc == capi.EMRKC_ENONFINITE:
            raise NumericalAbort(msg, stage, inner=inner)
        if rc == capi.EMRKC_ECALLBACK:
            if _CB_ERROR:
                ex = _CB_ERROR[0]
                _CB_ERROR.clear()
                raise RuntimeError(msg) from ex
            raise RuntimeError(msg)
        raise CudaError(msg)

    # device buffers ------------------------------------------------------
    def alloc(self, n: int) -> int:
        p = C.c_void_p()
        self.check(_lib().emrkc_vctx_alloc(self.h, n, C.byref(p)))
        self._bufs.append(p.value)
        return p.value

    def free(self, p: int):
        if p in self._bufs:
            self._bufs.remove(p)
            _lib().emrkc_vctx_free(self.h, p)

    def upload(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a, dtype=np.float64)
        p = self.alloc(a.size)
        self.check(_lib().emrkc_vctx_upload(self.h, p, dptr(a), a.size))
        return p

    def write(self, p: int, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        self.check(_lib().emrkc_vctx_upload(self.h, p, dptr(a), a.size))

    def download(self, p: int, n: int) -> np.ndarray:
        out = np.empty(n)
        self.check(_lib().emrkc_vctx_download(self.h, dptr(out), p, n))
        return out


_CTX: Optional[DeviceContext] = None


def context() -> DeviceContext:
    global _CTX
    if _CTX is None:
        _CTX = DeviceContext(0)
    return _CTX


# The first exception a Python callback raised inside the C library (it
# returns non-zero there, EMRKC_ECALLBACK); re-raised by DeviceContext.check.
_CB_ERROR: list = []


def _wrap_rhs(ctx: DeviceContext, f: Callable, counter: Optional[list] = None):
    """Python f(t, y) -> out as a device RhsFn (read back, call, upload)."""

    def cb(_c, t, y, out, n, _stream):
        try:
            yy = ctx.download(y, n)
            oo = np.ascontiguousarray(f(t, yy), dtype=np.float64)
            if oo.shape != (n,):
                raise ValueError(f"RhsFn returned shape {oo.shape}, expected ({n},)")
            ctx.write(out, oo)
            if counter is not None:
                counter[0] += 1
            return 0
        except Exception as ex:  # noqa: BLE001 - handed back to the caller
            _CB_ERROR.append(ex)
            return 1

    return capi.RHS_FN(cb)


def _wrap_exp(ctx: DeviceContext, e: Callable):
    """Python exp_part(y) -> (lambda, y_inf) as a device callback."""

    def cb(_c, y, lam, yinf, n, _stream):
        try:
            l, yi = e(ctx.download(y, n))
            ctx.write(lam, np.broadcast_to(np.asarray(l, dtype=np.float64), (n,)))
            ctx.write(yinf, np.broadcast_to(np.asarray(yi, dtype=np.float64), (n,)))
            return 0
        except Exception as ex:  # noqa: BLE001 - handed back to the caller
            _CB_ERROR.append(ex)
            return 1

    return capi.EXP_FN(cb)


@dataclass
class GenericSplitRhs:
    """SplitRhs (P/include/mrkc/multirate.hpp:25-35) over Python callables:
    f_F(t, y), f_S(t, y) -> out; exp_part(y) -> (lambda, y_inf) or None."""

    f_F: Callable
    f_S: Callable
    exp_part: Optional[Callable] = None
    rho_F: float = 0.0
    rho_S: float = 0.0
    counters: dict = field(default_factory=lambda: {"n_fF": 0, "n_fS": 0, "n_exp_steps": 0})


class _Bound:
    """A SplitRhsC plus the objects that keep its callbacks alive."""

    def __init__(self, ctx: DeviceContext, rhs):
        self.keep = []
        self.ctr = Counters()
        self.src = rhs
        self.c = SplitRhsC()
        if isinstance(rhs, SplitRhsC):
            self.c = rhs
        else:
            self.c.f_F = _wrap_rhs(ctx, rhs.f_F)
            self.c.f_S = _wrap_rhs(ctx, rhs.f_S)
            if rhs.exp_part is not None:
                self.c.exp_part = _wrap_exp(ctx, rhs.exp_part)
            self.keep += [self.c.f_F, self.c.f_S, self.c.exp_part]
            self.c.rho_F = rhs.rho_F
            self.c.rho_S = rhs.rho_S
        self.c.counters = C.pointer(self.ctr)

    def fold(self):
        if isinstance(self.src, GenericSplitRhs):
            for k in ("n_fF", "n_fS", "n_exp_steps"):
                self.src.counters[k] += getattr(self.ctr, k)


def bind(op) -> SplitRhsC:
    """SplitRhs of a device MonodomainOperator (emrkc_bind_split_rhs): f_F,
    f_S and exp_part stay on the device (the grid problem through the
    generic layer)."""
    out = SplitRhsC()
    rc = _lib().emrkc_bind_split_rhs(op.handle, C.byref(out))
    if rc:
        raise ValueError(_lib().emrkc_last_error(op.handle).decode())
    return out


# ---- the reference functions -------------------------------------------------

def rkc_iteration(t: float, y, dt: float, f: Callable, s: int,
                  epsilon: float = kDefaultDamping, ctx: DeviceContext | None = None):
    ctx = ctx or context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    dy = ctx.upload(y)
    dout = ctx.alloc(y.size)
    cb = _wrap_rhs(ctx, f)
    st = C.c_int32(0)
    try:
        rc = _lib().emrkc_rkc_iteration(ctx.h, t, dy, y.size, dt, cb, None, s, epsilon, dout,
                                        C.byref(st))
        ctx.check(rc, st.value)
        return ctx.download(dout, y.size)
    finally:
        ctx.free(dy)
        ctx.free(dout)


def stability_poly(s: int, epsilon: float, z: float, ctx: DeviceContext | None = None) -> float:
    """R_s(z) by the stage iteration on y' = z y, y = 1, dt = 1
    (P/src/cheb.cpp:114-118)."""
    return float(rkc_iteration(0.0, [1.0], 1.0, lambda t, u: z * u, s, epsilon, ctx)[0])


def exponential_euler_step(y, eta: float, lambda_diag, y_inf, ctx: DeviceContext | None = None):
    ctx = ctx or context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    bufs = [ctx.upload(a) for a in (y, lambda_diag, y_inf)]
    dout = ctx.alloc(y.size)
    try:
        ctx.check(_lib().emrkc_exponential_euler(ctx.h, bufs[0], eta, bufs[1], bufs[2], y.size,
                                                 dout))
        return ctx.download(dout, y.size)
    finally:
        for b in bufs + [dout]:
            ctx.free(b)


def _averaged(t, y, eta, rhs, m, variant, epsilon, ctx):
    ctx = ctx or context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = _Bound(ctx, rhs)
    dy = ctx.upload(y)
    dout = ctx.alloc(y.size)
    st = C.c_int32(0)
    try:
        if variant == "mrkc":
            rc = _lib().emrkc_averaged_force_mrkc(ctx.h, t, dy, y.size, eta, C.byref(b.c), m,
                                                  epsilon, dout, C.byref(st))
        else:
            rc = _lib().emrkc_averaged_force(ctx.h, t, dy, y.size, eta, C.byref(b.c), m, variant,
                                             epsilon, dout, C.byref(st))
        b.fold()
        ctx.check(rc, st.value, inner=True)
        return ctx.download(dout, y.size)
    finally:
        ctx.free(dy)
        ctx.free(dout)


def averaged_force_emrkc(t: float, y, eta: float, rhs, m: int,
                         variant: int = capi.EMRKC_VARIANT_STANDARD,
                         epsilon: float = kDefaultDamping, ctx: DeviceContext | None = None):
    return _averaged(t, y, eta, rhs, m, variant, epsilon, ctx)


def averaged_force_mrkc(t: float, y, eta: float, rhs, m: int,
                        epsilon: float = kDefaultDamping, ctx: DeviceContext | None = None):
    return _averaged(t, y, eta, rhs, m, "mrkc", epsilon, ctx)


def _step(t, y, dt, rhs, epsilon, variant, ctx):
    ctx = ctx or context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    b = _Bound(ctx, rhs)
    dy = ctx.upload(y)
    dout = ctx.alloc(y.size)
    rep = StepReport()
    try:
        if variant == "mrkc":
            rc = _lib().emrkc_mrkc_step_split(ctx.h, t, dy, y.size, dt, C.byref(b.c), epsilon,
                                              dout, C.byref(rep))
        else:
            rc = _lib().emrkc_step_split(ctx.h, t, dy, y.size, dt, C.byref(b.c), epsilon, variant,
                                         dout, C.byref(rep))
        b.fold()
        ctx.check(rc, rep.abort_stage, bool(rep.abort_inner))
        return ctx.download(dout, y.size), rep
    finally:
        ctx.free(dy)
        ctx.free(dout)


def emrkc_step(t: float, y, dt: float, rhs, epsilon: float = kDefaultDamping,
               variant: int = capi.EMRKC_VARIANT_STANDARD, ctx: DeviceContext | None = None):
    """emrkc_step over a generic SplitRhs (P/src/multirate.cpp:173-189):
    returns (y_next, MultirateStepReport)."""
    return _step(t, y, dt, rhs, epsilon, variant, ctx)


def mrkc_step(t: float, y, dt: float, rhs, epsilon: float = kDefaultDamping,
              ctx: DeviceContext | None = None):
    """mrkc_step (P/src/multirate.cpp:158-171)."""
    return _step(t, y, dt, rhs, epsilon, "mrkc", ctx)


def estimate_spectral_radius(t: float, y, f, v0=None, rho0: float = 0.0,
                             ctx: DeviceContext | None = None) -> RhoEstimate:
    """estimate_spectral_radius over a generic RhsFn (Python callable, or a
    device RHS_FN with its ctx as a (fn, ctx) pair)."""
    ctx = ctx or context()
    y = np.ascontiguousarray(y, dtype=np.float64)
    if isinstance(f, tuple):
        cb, fctx = f
    else:
        cb, fctx = _wrap_rhs(ctx, f), None
    dy = ctx.upload(y)
    dv0 = ctx.upload(v0) if v0 is not None else None
    dv = ctx.alloc(y.size)
    r = RhoResult()
    try:
        ctx.check(_lib().emrkc_estimate_spectral_radius(ctx.h, t, dy, y.size, cb, fctx, dv0, rho0,
                                                        C.byref(r), dv))
        return RhoEstimate(r.rho, r.iterations, bool(r.converged), r.safety,
                           ctx.download(dv, y.size))
    finally:
        for b in (dy, dv0, dv):
            if b is not None:
                ctx.free(b)
