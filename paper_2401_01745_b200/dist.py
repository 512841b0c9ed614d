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
    return np.concatenate([y_global[b * nn + z0 * plane: b * nn + z1 * plane] for b in range(4)])


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

    return DistContext(rank, world, exchange, reduce)


def slab_initial_state(w, part: Partition) -> np.ndarray:
    """This rank's slab of ``w.initial_state()`` (identical values) without
    materialising the other blocks of the global state."""
    from .monodomain import resting_state

    p = w.problem
    nn = w.n_nodes
    plane = nn // int(p.n[p.dim - 1])
    a, b = int(part.z_begin) * plane, int(part.z_end) * plane
    V, z = resting_state()
    rng = np.random.default_rng(w.seed)
    blocks = [np.full(b - a, V)] + [np.full(b - a, z[g]) for g in range(3)]
    if w.noise == "v_normal_0.1":
        blocks[0] += rng.normal(0.0, 0.1, nn)[a:b]
    elif w.noise == "mult_uniform_0.01":
        f = rng.uniform(0.99, 1.01, 4 * nn)
        for k in range(4):
            blocks[k] *= f[k * nn + a:k * nn + b]
    return np.concatenate(blocks)


def _rho_rank0(ctx, w, local):
    """rho_F, rho_S once at t = 0 on the whole grid (P/src/simulate.cpp:158-159),
    estimated on rank 0 and broadcast."""
    import torch
    import torch.distributed as dist

    rho = torch.zeros(2, dtype=torch.float64, device="cuda")
    if ctx.rank == 0:
        full = MonodomainOperator(w.problem, local)
        full.set_state(w.initial_state())
        rho[0] = full.estimate_spectral_radius(capi.EMRKC_RHS_F).rho
        rho[1] = (w.rho_S_forced if w.rho_S_forced is not None
                  else full.estimate_spectral_radius(capi.EMRKC_RHS_S).rho)
        full.close()
    dist.broadcast(rho, 0)
    return float(rho[0]), float(rho[1])


def _timed(ctx, w, local, warmup, steps, ClockSampler=None):
    """Device time of ``steps`` distributed steps of ``w`` (L2 flushed before
    every step), max over ranks; returns (ms, record, clocks, slab, rho)."""
    import torch
    import torch.distributed as dist

    rF, rS = _rho_rank0(ctx, w, local)
    slab = DistSlab(w.problem, ctx, local)
    slab.link()
    y0 = slab_initial_state(w, slab.part)
    slab.op.set_state(y0)
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
    """bench.py --gpus N under torchrun. Main line: weak scaling -- ``w``
    repeated N times along z, one copy per GPU (``workloads.z_scaled``), so
    per-GPU work equals the N = 1 line; value = global nodes x K / max over
    ranks of the device time. ``also``: strong scaling of the config-4 grid
    (BASELINE's partitioned config, north_star's efficiency target) over the
    same N GPUs."""
    import json
    import os

    import torch
    import torch.distributed as dist

    from . import workloads

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    ctx = torch_context()
    ww = workloads.z_scaled(w, ctx.world)
    ms, rec, clocks, slab, rho, y0 = _timed(ctx, ww, local, args.warmup, args.steps, ClockSampler)
    value = ww.n_nodes * rec["timed_steps"] / (ms * 1e-3)
    try:
        e2e = _e2e(ctx, slab, ww, y0, rho, 20)
    except Exception as ex:  # reported, not fatal: the device line stands
        e2e = {"error": f"{type(ex).__name__}: {ex}"}
    slab.op.close()
    del slab
    peak, kind = hbm_peak()
    also = []
    if not args.no_extra:
        try:
            w4 = workloads.get("hh3d_512x512x256")
            k4 = max(5, min(args.steps, 50))
            ms4, rec4, _, slab4, _, _ = _timed(ctx, w4, local, args.warmup, k4)
            slab4.op.close()
            del slab4
            k4 = rec4["timed_steps"]
            v4 = w4.n_nodes * k4 / (ms4 * 1e-3)
            also.append({"workload": w4.name, "scaling": "strong", "n_gpus": ctx.world,
                         "value": v4, "unit": "node-steps/s", "steps": k4,
                         "ms_per_step": ms4 / k4, "s": rec4["s"], "m": rec4["m"],
                         "step_frac_per_gpu": 64 * v4 / ctx.world / 1e9 / peak})
        except Exception as ex:
            also.append({"workload": "hh3d_512x512x256", "error": f"{type(ex).__name__}: {ex}"})
    if ctx.rank == 0:
        gbs = 64 * value / 1e9 / ctx.world
        cfg = config_of(ww, ctx.world)
        cfg["weak_scaling_of"] = w.name
        cfg["nodes_per_gpu"] = w.n_nodes
        line = {
            "metric": metric, "value": value, "unit": "node-steps/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / rec["timed_steps"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded HH resting state + N(0, 0.1 mV) V noise)",
            "config": cfg,
            "plan": {"s": rec["s"], "m": rec["m"], "rho_F": rho[0], "rho_S": rho[1],
                     "timed_steps": rec["timed_steps"],
                     "timed_note": "one run of the steps from the seeded state; if a slab hits "
                                   "NumericalAbort/the guard, every rank is timed up to the "
                                   "earliest abort step"},
            "gpu_launches": int(args.steps * rec["s"] * rec["m"]),
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
