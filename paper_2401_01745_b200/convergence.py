"""Convergence / efficiency harness on the device.

Mirrors the reference's experiment layer for the emRKC path
(P/src/experiments.cpp:114-189, P/src/config.cpp:204-217):

* ``reference_solution``: EXEX-RL at a small ``dt_ref`` on the device
  (``emrkc_exex_run``), cached on disk in the reference's ``MREF0001`` format
  (magic, u64 count, raw fp64 state; experiments.cpp:70-97) under a key
  hashed with FNV-1a (:39-52);
* ``run_convergence``: one run per dt (snapped so that t_end is an integer
  number of steps, config.cpp:214-217), the error of the final V block
  against the reference by the trapezoid-weighted ``rel_l2_error`` reduced on
  the device (``emrkc_rel_l2_error``), the observed order between rows;
* ``write_convergence_csv``: the reference's column layout (:307-322).

The reference keys its cache on a RunConfig; here the problem is given
directly (emrkc_problem + initial state), so the key serialises the problem
fields and a digest of the initial state instead.
"""
from __future__ import annotations

import hashlib
import math
import os
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import Problem
from .monodomain import MonodomainOperator, NumericalAbort

REF_MAGIC = b"MREF0001"
METHODS = ("emrkc", "emrkc-progressive", "exex-rl")  # method_name, config.cpp:9-19


def snap_dt(t_end: float, dt: float) -> float:
    """config.cpp:214-217."""
    n = max(1, int(round(t_end / dt)))
    return t_end / n


def step_count(t_end: float, dt: float) -> int:
    """config.cpp:204-212."""
    if not dt > 0.0:
        raise ValueError("dt must be > 0")
    if not t_end > 0.0:
        raise ValueError("t_end must be > 0")
    ratio = t_end / dt
    n = int(round(ratio))
    if n < 1 or abs(ratio - n) > 1e-9 * ratio:
        raise ValueError("t_end must be an integer multiple of dt")
    return n


def fnv1a(s: str) -> int:
    """experiments.cpp:45-52 (64-bit FNV-1a over the bytes of s)."""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def physical_key(p: Problem, y0: np.ndarray, t_end: float, dt_ref: float) -> str:
    dig = hashlib.blake2b(np.ascontiguousarray(y0, dtype=np.float64).tobytes(),
                          digest_size=16).hexdigest()
    f = lambda x: repr(float(x))  # noqa: E731  (round-trip, like %.17g)
    return (f"dim={p.dim};n={p.n[0]},{p.n[1]},{p.n[2]};dx={f(p.dx[0])},{f(p.dx[1])},{f(p.dx[2])};"
            f"sigma={f(p.sigma[0])},{f(p.sigma[1])},{f(p.sigma[2])};chi={f(p.chi)};Cm={f(p.C_m)};"
            f"model={p.model};stim={f(p.stim_chi_amplitude)};"
            f"box={f(p.stim_lo[0])},{f(p.stim_hi[0])},{f(p.stim_lo[1])},{f(p.stim_hi[1])},"
            f"{f(p.stim_lo[2])},{f(p.stim_hi[2])};window={f(p.stim_t0)},{f(p.stim_t1)};"
            f"y0={dig};t_end={f(t_end)};dt_ref={f(dt_ref)}")


def load_reference(path: str, expect: int):
    """experiments.cpp:72-86: None unless magic and size match."""
    try:
        with open(path, "rb") as fh:
            magic = fh.read(8)
            n = struct.unpack("<Q", fh.read(8))[0]
            if magic != REF_MAGIC or n != expect:
                return None
            data = np.frombuffer(fh.read(8 * n), dtype=np.float64)
            return data.copy() if data.size == n else None
    except (OSError, struct.error):
        return None


def store_reference(path: str, state: np.ndarray):
    """experiments.cpp:88-97."""
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    state = np.ascontiguousarray(state, dtype=np.float64)
    with open(path, "wb") as fh:
        fh.write(REF_MAGIC)
        fh.write(struct.pack("<Q", state.size))
        fh.write(state.tobytes())


def default_reference_dt(t_end: float, dt: float, dts) -> float:
    """experiments.cpp:114-123 (no explicit reference_dt)."""
    dt_min = min([dt, *dts])
    return snap_dt(t_end, min(1e-4, dt_min / 20.0))


def reference_solution(p: Problem, y0: np.ndarray, t_end: float, dt_ref: float,
                       cache_dir: str | None = None, device: int = 0):
    """EXEX-RL to t_end at dt_ref on the device, cached as MREF0001
    (experiments.cpp:125-149). Returns (state, cache_path)."""
    path = None
    if cache_dir is not None:
        path = os.path.join(cache_dir, f"ref_{fnv1a(physical_key(p, y0, t_end, dt_ref)):016x}.bin")
        got = load_reference(path, y0.size)
        if got is not None:
            return got, path
    op = MonodomainOperator(p, device)
    try:
        op.set_state(y0)
        res = op.exex_run(0, step_count(t_end, dt_ref), dt_ref)
        if res.aborted:
            raise NumericalAbort("reference run aborted", step_index=res.abort_step)
        state = op.get_state()
    finally:
        op.close()
    if path is not None:
        store_reference(path, state)
    return state, path


@dataclass
class ConvergenceRow:
    """experiments.hpp:24-32."""
    dt: float = 0.0
    err: float = 0.0
    order: float = 0.0
    s: int = 0
    m: int = 0
    counters: dict = field(default_factory=dict)
    stable: bool = True


@dataclass
class ConvergenceTable:
    method: str
    dt_ref: float
    rows: list


def _is_stable(res, v: np.ndarray) -> bool:
    """run_is_stable, experiments.cpp:107-112."""
    return not res.aborted and bool(np.all(np.isfinite(v))) and float(np.max(np.abs(v))) <= 1e3


def run_convergence(p: Problem, y0: np.ndarray, t_end: float, dts, method: str = "emrkc",
                    epsilon: float = 0.05, dt_ref: float | None = None,
                    cache_dir: str | None = None, device: int = 0) -> ConvergenceTable:
    """run_convergence (experiments.cpp:151-189) with every run on the device."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method}")
    dts = list(dts)
    dt_ref = snap_dt(t_end, dt_ref) if dt_ref is not None else \
        default_reference_dt(t_end, dts[0], dts)
    ref, _ = reference_solution(p, y0, t_end, dt_ref, cache_dir, device)
    nn = p.n_nodes
    rows = []
    op = MonodomainOperator(p, device)
    try:
        for d in dts:
            row = ConvergenceRow(dt=snap_dt(t_end, d))
            n = step_count(t_end, row.dt)
            op.set_state(y0)
            t0 = time.perf_counter()
            if method == "exex-rl":
                res = op.exex_run(0, n, row.dt)
            else:
                # rho_F, rho_S once at t = 0 (P/src/simulate.cpp:158-159)
                rF = op.estimate_spectral_radius(capi.EMRKC_RHS_F, 0.0).rho
                rS = op.estimate_spectral_radius(capi.EMRKC_RHS_S, 0.0).rho
                variant = (capi.EMRKC_VARIANT_PROGRESSIVE if method == "emrkc-progressive"
                           else capi.EMRKC_VARIANT_STANDARD)
                res = op.run(0, n, row.dt, rF, rS, epsilon, variant)
                row.s, row.m = res.s, res.m
            wall = time.perf_counter() - t0
            row.counters = {"n_fF": res.n_fF, "n_fS": res.n_fS, "n_exp": res.n_exp,
                            "n_linsolves": 0, "cg_iters": 0, "wall_s": wall}
            v = op.get_state()[:nn]
            row.stable = _is_stable(res, v)
            row.err = op.rel_l2_error(ref[:nn], 0) if row.stable else math.inf
            rows.append(row)
    finally:
        op.close()
    for i in range(1, len(rows)):
        a, b = rows[i - 1], rows[i]
        if a.stable and b.stable and a.err > 0 and b.err > 0:
            b.order = math.log(a.err / b.err) / math.log(a.dt / b.dt)
        else:
            b.order = math.nan
    if rows:
        rows[0].order = math.nan
    return ConvergenceTable(method, dt_ref, rows)


def _field(x) -> str:
    """csv::field (P/src/csv.cpp): shortest round-trip doubles, nan/inf, 1/0."""
    if isinstance(x, bool):
        return "1" if x else "0"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    x = float(x)
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    r = repr(x)
    return r[:-2] if r.endswith(".0") else r


def write_convergence_csv(path: str, t: ConvergenceTable):
    """write_convergence_csv, experiments.cpp:307-322 (per-part timers are not
    split on the device: t_fF/t_fS/t_exp are 0 and wall time is 'other')."""
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w", newline="") as fh:
        fh.write("method,dt,rel_l2_err,order,s,m,stable,n_fF,n_fS,n_exp,n_linsolves,cg_iters,"
                 "wall_s,t_fF_s,t_fS_s,t_exp_s,t_other_s\n")
        for r in t.rows:
            c = r.counters
            fh.write(",".join([t.method, _field(r.dt), _field(r.err), _field(r.order),
                               _field(r.s), _field(r.m), _field(bool(r.stable)),
                               _field(c.get("n_fF", 0)), _field(c.get("n_fS", 0)),
                               _field(c.get("n_exp", 0)), _field(0), _field(0),
                               _field(c.get("wall_s", 0.0)), _field(0.0), _field(0.0),
                               _field(0.0), _field(c.get("wall_s", 0.0))]) + "\n")
