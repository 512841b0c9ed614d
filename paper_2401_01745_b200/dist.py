"""One process per GPU: z-slab distributed emRKC runs.

No reference counterpart (the reference never partitions).
Each rank owns a contiguous z-slab (``emrkc_partition_slab``); V halo planes
travel by peer stores from the producing kernel into the neighbour's ghost
planes (CUDA IPC-mapped), with device-side arrival counters, so no host
synchronisation happens inside a run. The host side here only

* exchanges the IPC blobs (``exchange``: an all-gather of bytes),
* reduces per-rank run records into the reference's single record
  (``reduce``: an all-gather of small dicts), and
* replays from the run's checkpoint when some rank aborted, so that every
  slab ends on the state the reference would return (the first abort over
  all slabs wins; a norm-guard trip keeps that step's result).

``exchange`` / ``reduce`` are injected (torch.distributed in bench.py, gloo
in tests/test_dist_gloo.py), which keeps this logic testable on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import Partition, Problem, RunResult
from .monodomain import MonodomainOperator, _check, _lib

RECORD_KEYS = [k for k, _ in RunResult._fields_]


def partition(problem: Problem, world: int, rank: int) -> Partition:
    part = Partition()
    nz = int(problem.n[problem.dim - 1])
    _check(_lib().emrkc_partition_slab(nz, world, rank, C.byref(part)))
    return part


def min_slab_depth(problem: Problem, world: int) -> int:
    """Smallest slab (planes) of the world-rank partition."""
    return min(int(p.z_end - p.z_begin) for p in (partition(problem, world, r) for r in range(world)))


def slab_of(problem: Problem, part: Partition, y_global: np.ndarray) -> np.ndarray:
    """Local slab of a global reference-layout state."""
    nn = problem.n_nodes
    plane = nn // int(problem.n[problem.dim - 1])
    z0, z1 = int(part.z_begin), int(part.z_end)
    return np.concatenate([y_global[b * nn + z0 * plane: b * nn + z1 * plane]
                           for b in range(problem.n_fields)])


def first_event_key(rec: dict):
    """Program-order key of a rank's abort (None if it did not abort): step,
    then a non-finite stage before the norm guard of the same step."""
    if not rec["aborted"]:
        return None
    kind = 0 if rec["abort_kind"] == capi.EMRKC_ABORT_NONFINITE else 1
    # within a step: outer stage j, then its inner stages before its check
    inner_pos = rec["abort_stage"] if rec["abort_inner"] else 1 << 30
    return (rec["abort_step"], kind, rec.get("abort_outer_stage", 0), inner_pos)


def combine(records: list[dict]) -> dict:
    """Reference run record from per-rank records of the SAME run."""
    out = dict(records[0])
    keyed = [(first_event_key(r), i) for i, r in enumerate(records)]
    aborted = [(k, i) for k, i in keyed if k is not None]
    if aborted:
        _, i = min(aborted)
        for k in ("aborted", "abort_kind", "abort_step", "abort_stage", "abort_inner",
                  "abort_outer_stage", "steps_done", "n_fF", "n_fS", "n_exp", "s", "m", "eta"):
            out[k] = records[i][k]
    out["gate_min"] = min(r["gate_min"] for r in records)
    out["gate_max"] = max(r["gate_max"] for r in records)
    out["device_ms"] = max(r["device_ms"] for r in records)
    return out


def replay_steps(rec: dict, step0: int) -> int:
    """Steps to replay from the checkpoint after a global abort."""
    k = rec["abort_step"] - step0
    return k + 1 if rec["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD else k


@dataclass
class DistContext:
    rank: int
    world: int
    exchange: object  # callable(bytes) -> list[bytes] (all ranks, rank order)
    reduce: object    # callable(dict) -> list[dict]   (all ranks, rank order)
    # slab power iteration (slab_rho): halo(lo_plane, hi_plane) -> (ghost_lo,
    # ghost_hi) sends this slab's first plane down and last plane up and
    # returns the neighbours' (None at the global boundary); chain(fn, acc)
    # runs acc = fn(acc) on rank 0, 1, ... in turn and returns the last
    # rank's result on every rank
    halo: object = None
    chain: object = None


def slab_rho(sp, ctx: DistContext, which: int, t: float = 0.0, v0_slab=None,
             rho0: float = 0.0):
    """estimate_spectral_radius (P/src/spectral.cpp:26-71) over the z-slabs
    of ``ctx.world`` ranks, ``sp`` this rank's slab (emrkc_slab_power_*
    through ``DeviceSlabPower``, or a host stand-in in the CPU tests).

    Every norm is the reference's serial sum (P/src/spectral.cpp:10-14) over
    the global vector: SoA block by block, each rank continuing the running
    sum of the rank below (``ctx.chain``); V ghost planes of y (once) and of
    v (each iteration) come from the neighbours (``ctx.halo``). So q, z =
    y + q v, f(z) - f(y) and rho are bit-identical to the single-grid
    estimate for ANY partition, with the reference's iteration count."""
    import math

    from .monodomain import RhoEstimate

    sp.begin(which, v0_slab)

    def norm(field):
        acc = 0.0
        for b in range(sp.n_fields):
            acc = ctx.chain(lambda a, b=b: sp.sumsq(field, b, a), acc)
        return math.sqrt(acc)

    def ghosts(field):
        return ctx.halo(sp.plane(field, 0), sp.plane(field, 1))

    nv = norm(0)
    if nv == 0.0:
        sp.end()
        raise ValueError("estimate_spectral_radius: v0 must be nonzero")
    ny = norm(1)
    delta = max(ny, 1e-8) * 1e-8
    gy = ghosts(1)
    sp.fy(t, *gy)
    rho, rho_old, it, converged = rho0, 0.0, 0, True
    while it == 0 or abs(rho - rho_old) >= 1e-2 * rho:
        if it >= 50:
            converged = False
            break
        rho_old = rho
        q = delta / nv
        gv = ghosts(0)
        sp.step(t, q, gy[0], gy[1], gv[0], gv[1])
        nv = norm(0)
        if nv < 1e-300:  # locally null operator (P/src/spectral.cpp:61-66)
            return RhoEstimate(0.0, it + 1, True, 1.05, sp.end())
        rho = nv / delta
        it += 1
    return RhoEstimate(rho * 1.05, it, converged, 1.05, sp.end())


class DeviceSlabPower:
    """This rank's slab of the power iteration on the device
    (emrkc_slab_power_*); planes travel as torch CUDA tensors."""

    def __init__(self, op):
        import torch

        self.op = op
        self.lib = _lib()
        prob = op.problem
        self.n_fields = prob.n_fields
        self.plane_len = int(prob.n_nodes // int(prob.n[prob.dim - 1]))
        self.torch = torch

    def _ptr(self, x):
        return None if x is None else C.c_void_p(x.data_ptr())

    def begin(self, which, v0_slab=None):
        v0 = None if v0_slab is None else np.ascontiguousarray(v0_slab, dtype=np.float64)
        _check(self.lib.emrkc_slab_power_begin(self.op.handle, which,
                                               None if v0 is None else capi.dptr(v0)),
               self.op.handle)

    def plane(self, field, side):
        out = self.torch.empty(self.plane_len, dtype=self.torch.float64, device="cuda")
        _check(self.lib.emrkc_slab_power_plane(self.op.handle, field, side,
                                               C.c_void_p(out.data_ptr())), self.op.handle)
        return out

    def sumsq(self, field, block, acc):
        out = C.c_double()
        _check(self.lib.emrkc_slab_power_sumsq(self.op.handle, field, block, acc,
                                               C.byref(out)), self.op.handle)
        return out.value

    def fy(self, t, glo, ghi):
        _check(self.lib.emrkc_slab_power_fy(self.op.handle, t, self._ptr(glo), self._ptr(ghi)),
               self.op.handle)

    def step(self, t, q, gylo, gyhi, gvlo, gvhi):
        _check(self.lib.emrkc_slab_power_step(self.op.handle, t, q, self._ptr(gylo),
                                              self._ptr(gyhi), self._ptr(gvlo), self._ptr(gvhi)),
               self.op.handle)

    def end(self):
        v = np.empty(self.op.len)
        _check(self.lib.emrkc_slab_power_end(self.op.handle, capi.dptr(v)), self.op.handle)
        return v


class DistSlab:
    """This rank's slab of a distributed run."""

    def __init__(self, problem: Problem, ctx: DistContext, device: int = 0, op=None):
        self.problem = problem
        self.ctx = ctx
        self.part = partition(problem, ctx.world, ctx.rank)
        self.op = op if op is not None else MonodomainOperator(problem, device, self.part)

    @property
    def whole(self) -> bool:
        """One rank: the slab is the whole grid (a plain handle, no halos)."""
        return self.ctx.world == 1

    def step_run(self, step0, nsteps, dt, rho_F, rho_S, epsilon=0.05) -> dict:
        """This rank's part of one distributed emrkc_run (no record reduction)."""
        if self.whole:
            return self.op.run(step0, nsteps, dt, rho_F, rho_S, epsilon).as_dict()
        return self.op.dist_run(step0, nsteps, dt, rho_F, rho_S, epsilon)

    def link(self):
        """Exchange IPC blobs and import the lower / upper neighbours."""
        if self.whole:
            return
        blob = self.op.ipc_export()
        blobs = self.ctx.exchange(blob)
        if self.ctx.rank > 0:
            self.op.ipc_import(0, blobs[self.ctx.rank - 1])
        if self.ctx.rank + 1 < self.ctx.world:
            self.op.ipc_import(1, blobs[self.ctx.rank + 1])
        # every rank derives the same partition, hence the same smallest slab
        # depth: the wide d_1 halo is switched on (or off) consistently
        self.op.set_slab_min_depth(min_slab_depth(self.problem, self.ctx.world))

    def set_global_state(self, y_global: np.ndarray):
        self.op.set_state(slab_of(self.problem, self.part, y_global))

    def run(self, step0: int, nsteps: int, dt: float, rho_F: float, rho_S: float,
            epsilon: float = 0.05) -> dict:
        """Distributed emrkc_run: the reference's run record, every slab left
        on the reference's final state."""
        rec = self.step_run(step0, nsteps, dt, rho_F, rho_S, epsilon)
        recs = self.ctx.reduce(rec)
        glob = combine(recs)
        if glob["aborted"] and not self.whole:
            k = replay_steps(glob, step0)
            rrec = self.op.dist_replay(step0, k, dt, rho_F, rho_S, epsilon)
            rrecs = self.ctx.reduce(rrec)
            glob["gate_min"] = min(r["gate_min"] for r in rrecs)
            glob["gate_max"] = max(r["gate_max"] for r in rrecs)
        return glob


# ---- bench.py's multi-GPU arm ------------------------------------------------

def torch_context():
    import pickle

    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()

    def exchange(b: bytes):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    def reduce(d: dict):
        out = [None] * world
        dist.all_gather_object(out, pickle.loads(pickle.dumps(d)))
        return out

    return DistContext(rank, world, exchange, reduce, *torch_p2p(rank, world))


def torch_p2p(rank: int, world: int):
    """(halo, chain) over torch.distributed point-to-point (NCCL: device
    planes; gloo: host tensors)."""
    import torch
    import torch.distributed as dist

    def halo(lo, hi):
        # gloo moves host tensors: device planes go through host copies
        dev = lo.device
        host = dist.get_backend() != "nccl" and dev.type == "cuda"
        if host:
            lo, hi = lo.cpu(), hi.cpu()
        ops, glo, ghi = [], None, None
        if rank > 0:
            glo = torch.empty_like(lo)
            ops += [dist.P2POp(dist.isend, lo, rank - 1), dist.P2POp(dist.irecv, glo, rank - 1)]
        if rank + 1 < world:
            ghi = torch.empty_like(hi)
            ops += [dist.P2POp(dist.isend, hi, rank + 1), dist.P2POp(dist.irecv, ghi, rank + 1)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if host:
            glo = None if glo is None else glo.to(dev)
            ghi = None if ghi is None else ghi.to(dev)
        return glo, ghi

    def chain(fn, acc):
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        buf = torch.tensor([acc], dtype=torch.float64, device=dev)
        if rank > 0:
            dist.recv(buf, rank - 1)
        buf.fill_(fn(float(buf[0])))
        if rank + 1 < world:
            dist.send(buf, rank + 1)
        dist.broadcast(buf, world - 1)
        return float(buf[0])

    return halo, chain


def slab_initial_state(w, part: Partition) -> np.ndarray:
    """This rank's slab of ``w.initial_state()`` (identical values) without
    materialising the other blocks of the global state."""
    from .monodomain import resting_state

    p = w.problem
    nn = w.n_nodes
    plane = nn // int(p.n[p.dim - 1])
    a, b = int(part.z_begin) * plane, int(part.z_end) * plane
    from .workloads import aux_rest

    V, z = resting_state()
    rng = np.random.default_rng(w.seed)
    nf = p.n_fields
    blocks = [np.full(b - a, V)] + [np.full(b - a, z[g]) for g in range(3)] + \
        [np.full(b - a, aux_rest(q, V)) for q in range(nf - 4)]
    if w.noise == "v_normal_0.1":
        blocks[0] += rng.normal(0.0, 0.1, nn)[a:b]
    elif w.noise == "mult_uniform_0.01":
        f = rng.uniform(0.99, 1.01, nf * nn)
        for k in range(nf):
            blocks[k] *= f[k * nn + a:k * nn + b]
    return np.concatenate(blocks)


def rho_slabs(ctx, w, slab):
    """rho_F, rho_S once at t = 0 (P/src/simulate.cpp:158-159) by the
    distributed power iteration over the ranks' slabs (``slab_rho``): no
    rank holds the whole grid, and the result is bit-identical to the
    single-grid estimate."""
    sp = DeviceSlabPower(slab.op)
    rF = slab_rho(sp, ctx, capi.EMRKC_RHS_F, 0.0).rho
    rS = (w.rho_S_forced if w.rho_S_forced is not None
          else slab_rho(sp, ctx, capi.EMRKC_RHS_S, 0.0).rho)
    return rF, rS


def _timed(ctx, w, local, warmup, steps, ClockSampler=None, rho=None):
    """Device time of ``steps`` distributed steps of ``w`` (L2 flushed before
    every step), max over ranks; returns (ms, record, clocks, slab, rho).
    ``rho``: given (rho_F, rho_S) instead of the distributed estimate."""
    import torch
    import torch.distributed as dist

    slab = DistSlab(w.problem, ctx, local)
    slab.link()
    y0 = slab_initial_state(w, slab.part)
    slab.op.set_state(y0)
    rF, rS = rho if rho is not None else rho_slabs(ctx, w, slab)
    slab.run(0, warmup, w.dt, rF, rS, w.eps)
    slab.op.set_state(y0)
    dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local) if ClockSampler else None
    if clk:
        clk.__enter__()
    try:
        launch_ms, rec = slab.op.run_timed_dist(0, steps, w.dt, rF, rS, w.eps)
    finally:
        if clk:
            clk.__exit__(None, None, None)
    torch.cuda.synchronize()
    dist.barrier()
    # a slab that hit NumericalAbort / the norm guard skips the later steps'
    # work: time every rank over the steps before the earliest abort only
    kr = torch.tensor([int(rec["abort_step"]) if rec["aborted"] else steps],
                      dtype=torch.int64, device="cuda")
    dist.all_reduce(kr, op=dist.ReduceOp.MIN)
    k = max(1, int(kr[0]))
    per = launch_ms.size // max(1, steps)
    tot = torch.tensor([float(launch_ms[:k * per].sum())], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    rec = dict(rec, timed_steps=k)
    return float(tot[0]), rec, (clk.summary() if clk else None), slab, (rF, rS), y0


def _e2e(ctx, slab, w, y0, rho, k):
    """Per-step host API at N GPUs: every rank copies its slab in from pinned
    host memory (emrkc_set_state), takes one distributed step
    (emrkc_dist_run) and copies its slab back (emrkc_get_state); wall time,
    max over ranks."""
    import time

    import torch
    import torch.distributed as dist

    hin = torch.from_numpy(y0.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    lib = _lib()

    def one(step):
        _check(lib.emrkc_set_state(slab.op._h, C.cast(hin.data_ptr(), capi.DP), hin.numel()),
               slab.op._h)
        slab.step_run(step, 1, w.dt, rho[0], rho[1], w.eps)
        _check(lib.emrkc_get_state(slab.op._h, C.cast(hout.data_ptr(), capi.DP), hout.numel()),
               slab.op._h)

    one(0)
    dist.barrier()
    t0 = time.perf_counter()
    for s in range(k):
        one(s)
    wall = time.perf_counter() - t0
    t = torch.tensor([wall], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall = float(t[0])
    return {"value": w.n_nodes * k / wall, "unit": "node-steps/s",
            "h2d_bytes_per_step": 8 * hin.numel() * ctx.world,
            "d2h_bytes_per_step": 8 * hout.numel() * ctx.world, "steps": k,
            "ms_per_step": wall * 1e3 / k,
            "api": "per rank: emrkc_set_state + emrkc_dist_run (1 step) + emrkc_get_state"}


def bench_main(args, w, metric, config_of, hbm_peak, ClockSampler):
    """bench.py --gpus N under torchrun. Main line: STRONG scaling of ``w``
    (the N = 1 headline, config 4's grid) split into N z-slabs, so the
    driver's per-N ratio v(N) / (N v(1)) is north_star's parallel
    efficiency E(N); value = global nodes x K / max over ranks of the device
    time. rho comes from the distributed power iteration over the slabs.
    ``also``: WEAK scaling of BASELINE configs[1] (128^3 repeated N times
    along z, one copy per GPU)."""
    import json
    import os

    import torch
    import torch.distributed as dist

    from . import workloads

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    ctx = torch_context()
    ms, rec, clocks, slab, rho, y0 = _timed(ctx, w, local, args.warmup, args.steps, ClockSampler)
    value = w.n_nodes * rec["timed_steps"] / (ms * 1e-3)
    try:
        e2e = _e2e(ctx, slab, w, y0, rho, min(args.steps, 10))
    except Exception as ex:  # reported, not fatal: the device line stands
        e2e = {"error": f"{type(ex).__name__}: {ex}"}
    slab.op.close()
    del slab
    peak, kind = hbm_peak()
    also = []
    if not args.no_extra:
        try:
            wk = workloads.z_scaled(workloads.get("hh3d_128x128x128"), ctx.world)
            kk = max(5, min(args.steps, 50))
            msk, reck, _, slabk, _, _ = _timed(ctx, wk, local, args.warmup, kk)
            slabk.op.close()
            del slabk
            kk = reck["timed_steps"]
            vk = wk.n_nodes * kk / (msk * 1e-3)
            also.append({"workload": wk.name, "scaling": "weak", "n_gpus": ctx.world,
                         "value": vk, "unit": "node-steps/s", "steps": kk,
                         "ms_per_step": msk / kk, "s": reck["s"], "m": reck["m"],
                         "step_frac_per_gpu": 64 * vk / ctx.world / 1e9 / peak})
        except Exception as ex:
            also.append({"workload": "hh3d_128x128x128 (weak)",
                         "error": f"{type(ex).__name__}: {ex}"})
        # strong scaling of config 4's grid at the TTP state width (19
        # fields, the SYNTHETIC width stand-in; rho of the HH state of the
        # same grid, the plan is the same): per-N values next to the N = 1
        # line's also entry give E(N) at 304 B/node
        if w.name == "hh3d_512x512x256":
            try:
                w19 = workloads.get("hh3d_512x512x256_w19")
                k19 = max(5, min(args.steps, 40))
                ms19, rec19, _, slab19, _, _ = _timed(ctx, w19, local, args.warmup, k19,
                                                      rho=rho)
                slab19.op.close()
                del slab19
                k19 = rec19["timed_steps"]
                v19 = w19.n_nodes * k19 / (ms19 * 1e-3)
                also.append({"workload": w19.name, "scaling": "strong", "n_gpus": ctx.world,
                             "value": v19, "unit": "node-steps/s", "steps": k19,
                             "ms_per_step": ms19 / k19, "s": rec19["s"], "m": rec19["m"],
                             "state_fields": 19,
                             "step_frac_per_gpu": 304 * v19 / ctx.world / 1e9 / peak,
                             "note": w19.note})
            except Exception as ex:
                also.append({"workload": "hh3d_512x512x256_w19 (strong)",
                             "error": f"{type(ex).__name__}: {ex}"})
    if ctx.rank == 0:
        gbs = 64 * value / 1e9 / ctx.world
        cfg = config_of(w, ctx.world)
        cfg["nodes_per_gpu"] = w.n_nodes // ctx.world
        line = {
            "metric": metric, "value": value, "unit": "node-steps/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / rec["timed_steps"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded HH resting state + N(0, 0.1 mV) V noise)",
            "config": cfg,
            "plan": {"s": rec["s"], "m": rec["m"], "rho_F": rho[0], "rho_S": rho[1],
                     "rho": "distributed power iteration over the slabs (norms chained "
                            "across ranks in the reference's serial order)",
                     "timed_steps": rec["timed_steps"],
                     "timed_note": "one run of the steps from the seeded state; if a slab hits "
                                   "NumericalAbort/the guard, every rank is timed up to the "
                                   "earliest abort step"},
            "gpu_launches": int(rec["timed_steps"] * rec["s"] * rec["m"]),
            "clocks": clocks,
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "traffic": None, "per": "GPU (step-level)",
                         "kernel": "whole step (all launches)",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({kind})"},
            "also": also,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
