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

    def link(self):
        """Exchange IPC blobs and import the lower / upper neighbours."""
        blob = self.op.ipc_export()
        blobs = self.ctx.exchange(blob)
        if self.ctx.rank > 0:
            self.op.ipc_import(0, blobs[self.ctx.rank - 1])
        if self.ctx.rank + 1 < self.ctx.world:
            self.op.ipc_import(1, blobs[self.ctx.rank + 1])

    def set_global_state(self, y_global: np.ndarray):
        self.op.set_state(slab_of(self.problem, self.part, y_global))

    def run(self, step0: int, nsteps: int, dt: float, rho_F: float, rho_S: float,
            epsilon: float = 0.05) -> dict:
        """Distributed emrkc_run: the reference's run record, every slab left
        on the reference's final state."""
        rec = self.op.dist_run(step0, nsteps, dt, rho_F, rho_S, epsilon)
        recs = self.ctx.reduce(rec)
        glob = combine(recs)
        if glob["aborted"]:
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


def bench_main(args, w, metric, config_of, hbm_peak, ClockSampler):
    """bench.py --gpus N under torchrun: strong scaling of one workload over
    N z-slabs; value = global nodes x K / max over ranks of the device time."""
    import json
    import os

    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    ctx = torch_context()
    p = w.problem
    y0 = w.initial_state()
    # rho once at t = 0 on the whole grid (P/src/simulate.cpp:158-159), rank 0
    rho = torch.zeros(2, dtype=torch.float64, device="cuda")
    if ctx.rank == 0:
        full = MonodomainOperator(p, local)
        full.set_state(y0)
        rho[0] = full.estimate_spectral_radius(capi.EMRKC_RHS_F).rho
        rho[1] = (w.rho_S_forced if w.rho_S_forced is not None
                  else full.estimate_spectral_radius(capi.EMRKC_RHS_S).rho)
        full.close()
    dist.broadcast(rho, 0)
    rF, rS = float(rho[0]), float(rho[1])
    slab = DistSlab(p, ctx, local)
    slab.link()
    slab.set_global_state(y0)
    slab.run(0, args.warmup, w.dt, rF, rS, w.eps)
    slab.set_global_state(y0)
    dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    with clk:
        launch_ms, rec = slab.op.run_timed_dist(0, args.steps, w.dt, rF, rS, w.eps)
    torch.cuda.synchronize()
    dist.barrier()
    tot = torch.tensor([float(launch_ms.sum())], dtype=torch.float64, device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    value = w.n_nodes * args.steps / (float(tot[0]) * 1e-3)
    peak, kind = hbm_peak()
    if ctx.rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "node-steps/s", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(tot[0]) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded HH resting state + N(0, 0.1 mV) V noise)",
            "config": config_of(w, ctx.world),
            "gpu_launches": int(args.steps * rec["s"] * rec["m"] * ctx.world),
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "achieved": 64 * w.n_nodes * args.steps /
                         (float(tot[0]) * 1e-3) / 1e9 / ctx.world, "peak": peak,
                         "unit": "GB/s", "frac": 64 * w.n_nodes * args.steps /
                         (float(tot[0]) * 1e-3) / 1e9 / ctx.world / peak,
                         "traffic": None, "per": "GPU (step-level)",
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({kind})"},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0
