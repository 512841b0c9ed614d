"""Host-side logic of the multi-GPU path on CPU: two gloo ranks route the
IPC blobs to the right neighbours, combine per-rank run records into the
reference's single record (first abort in program order wins, gate range
over all slabs) and agree on the replay. The device calls are replaced by a
recording stand-in (no GPU here)."""
import os
import pickle
import socket

import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2401_01745_b200 import capi, dist
from paper_2401_01745_b200.workloads import hh3d_128


def rec(**kw):
    r = {k: 0 for k in dist.RECORD_KEYS}
    r.update(n_steps=10, steps_done=10, abort_step=-1, gate_min=0.1, gate_max=0.6, s=1, m=1,
             eta=0.05, n_fF=10, n_fS=10, n_exp=10)
    r.update(kw)
    return r


class FakeOp:
    def __init__(self, rank, abort=None):
        self.rank = rank
        self.abort = abort
        self.imported = {}
        self.calls = []

    def ipc_export(self):
        return f"blob-of-{self.rank}".encode()

    def ipc_import(self, side, blob):
        self.imported[side] = blob

    def set_slab_min_depth(self, planes):
        self.min_depth = planes

    def dist_run(self, step0, nsteps, *a):
        self.calls.append(("run", step0, nsteps))
        if self.abort is None:
            return rec(gate_min=0.1 + self.rank * 0.01, gate_max=0.6 - self.rank * 0.01)
        step, kind = self.abort
        return rec(aborted=1, abort_kind=kind, abort_step=step, steps_done=step if kind == 1 else step + 1,
                   abort_stage=1, abort_inner=1, n_fF=step + 1, gate_min=-3.0, gate_max=9.0)

    def dist_replay(self, step0, nsteps, *a):
        self.calls.append(("replay", step0, nsteps))
        return rec(steps_done=nsteps, gate_min=0.2 + self.rank * 0.01, gate_max=0.5)


def _worker(rank, world, port, scenario, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(b):
        out = [None] * world
        tdist.all_gather_object(out, b)
        return out

    def reduce(d):
        out = [None] * world
        tdist.all_gather_object(out, pickle.loads(pickle.dumps(d)))
        return out

    ctx = dist.DistContext(rank, world, exchange, reduce)
    abort = scenario.get(rank)
    op = FakeOp(rank, abort)
    slab = dist.DistSlab(hh3d_128().problem, ctx, op=op)
    slab.link()
    # the smallest slab of the partition, the same on every rank
    assert op.min_depth == min(dist.partition(slab.problem, world, r).z_end -
                               dist.partition(slab.problem, world, r).z_begin for r in range(world))
    glob = slab.run(0, 10, 0.05, 15.0, 0.7)
    q.put((rank, {k: v for k, v in glob.items()}, op.imported, op.calls,
           (slab.part.z_begin, slab.part.z_end)))
    tdist.destroy_process_group()


def run_world(scenario, world=2):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, glob, imported, calls, part = q.get(timeout=120)
        out[r] = (glob, imported, calls, part)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_blob_routing_and_clean_run():
    out = run_world({})
    g0, imp0, calls0, part0 = out[0]
    g1, imp1, calls1, part1 = out[1]
    assert part0 == (0, 64) and part1 == (64, 128)
    assert imp0 == {1: b"blob-of-1"} and imp1 == {0: b"blob-of-0"}
    assert calls0 == [("run", 0, 10)] and calls1 == [("run", 0, 10)]
    assert g0 == g1 and not g0["aborted"]
    assert g0["gate_min"] == 0.1 and g0["gate_max"] == 0.6


def test_first_abort_wins_and_everyone_replays():
    # rank 1 trips the norm guard at step 6, rank 0 goes non-finite at step 6:
    # the non-finite stage comes first in program order (the guard follows a
    # completed step), so the state is the input of step 6 -> replay 6 steps.
    out = run_world({0: (6, capi.EMRKC_ABORT_NONFINITE), 1: (6, capi.EMRKC_ABORT_NORM_GUARD)})
    for r in (0, 1):
        g, _, calls, _ = out[r]
        assert g["aborted"] and g["abort_step"] == 6
        assert g["abort_kind"] == capi.EMRKC_ABORT_NONFINITE
        assert calls == [("run", 0, 10), ("replay", 0, 6)]
        assert g["gate_min"] == 0.2 and g["gate_max"] == 0.5  # from the replay


def test_guard_replays_the_tripping_step():
    out = run_world({1: (3, capi.EMRKC_ABORT_NORM_GUARD)})
    for r in (0, 1):
        g, _, calls, _ = out[r]
        assert g["abort_kind"] == capi.EMRKC_ABORT_NORM_GUARD and g["abort_step"] == 3
        assert calls[-1] == ("replay", 0, 4)


def test_combine_is_order_independent():
    a = rec(aborted=1, abort_kind=1, abort_step=4, abort_inner=0, abort_stage=2)
    b = rec(aborted=1, abort_kind=1, abort_step=4, abort_inner=1, abort_stage=1)
    c = rec()
    assert dist.combine([a, b, c])["abort_inner"] == 1
    assert dist.combine([c, b, a]) == dist.combine([a, b, c]) | {}


# ---- distributed power iteration (dist.slab_rho) ------------------------------

class HostSlabPower:
    """CPU stand-in for DeviceSlabPower: a z-slab of a 4-block state
    (nz planes of P nodes per block); f = z-Laplacian on the V block (mirror
    at the global ends, ghosts at slab faces) plus a pointwise nonlinearity,
    gate rows pointwise. Norms continue the running sum in serial order."""

    P, NZ = 6, 24
    n_fields = 4

    def __init__(self, y_global, v_global, z0, z1):
        import numpy as np
        import torch

        self.np, self.torch = np, torch
        self.z0, self.z1 = z0, z1
        nn = self.P * self.NZ
        sl = lambda g: np.concatenate([g[b * nn + z0 * self.P: b * nn + z1 * self.P] for b in range(4)])
        self.y = sl(y_global)
        self.v0 = sl(v_global)
        self.nl = (z1 - z0) * self.P

    def f(self, x, glo, ghi):
        np = self.np
        nl, P = self.nl, self.P
        V = x[:nl].reshape(-1, P)
        lo = glo.numpy().reshape(1, P) if glo is not None else V[1:2]
        hi = ghi.numpy().reshape(1, P) if ghi is not None else V[-2:-1]
        ext = np.concatenate([lo, V, hi])
        out = np.empty_like(x)
        out[:nl] = (2.5 * ((ext[:-2] - 2.0 * V) + ext[2:]) - 0.01 * V * V * V).ravel()
        for b in range(1, 4):
            out[b * nl:(b + 1) * nl] = -(0.5 + 0.1 * b) * x[b * nl:(b + 1) * nl] * x[:nl]
        return out

    def begin(self, which, v0_slab=None):
        self.v = self.v0.copy() if v0_slab is None else v0_slab.copy()

    def plane(self, field, side):
        x = self.v if field == 0 else self.y
        V = x[:self.nl]
        return self.torch.from_numpy((V[:self.P] if side == 0 else V[-self.P:]).copy())

    def sumsq(self, field, block, acc):
        np = self.np
        x = (self.v if field == 0 else self.y)[block * self.nl:(block + 1) * self.nl]
        return float(np.add.accumulate(np.concatenate([[acc], x * x]))[-1])  # serial order

    def fy(self, t, glo, ghi):
        self.fyv = self.f(self.y, glo, ghi)

    def step(self, t, q, gylo, gyhi, gvlo, gvhi):
        zl = None if gylo is None else gylo + q * gvlo
        zh = None if gyhi is None else gyhi + q * gvhi
        self.v = self.f(self.y + q * self.v, zl, zh) - self.fyv

    def end(self):
        return self.v


def _rho_worker(rank, world, port, q):
    import numpy as np

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    halo, chain = dist.torch_p2p(rank, world)
    ctx = dist.DistContext(rank, world, None, None, halo, chain)
    P, NZ = HostSlabPower.P, HostSlabPower.NZ
    rng = np.random.default_rng(3)
    y = np.concatenate([-65.0 + rng.normal(0, 2.0, NZ * P)] + [rng.uniform(0, 1, NZ * P)] * 3)
    v = rng.uniform(-1, 1, 4 * NZ * P)
    z0, z1 = NZ * rank // world, NZ * (rank + 1) // world
    est = dist.slab_rho(HostSlabPower(y, v, z0, z1), ctx, 0)
    q.put((rank, est.rho, est.iterations, est.converged))
    tdist.destroy_process_group()


def rho_world(world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rho_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, rho, it, conv = q.get(timeout=120)
        res[r] = (rho, it, conv)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_slab_rho_bitwise_independent_of_partition():
    """The norms chained across ranks in serial order: rho and the iteration
    count are bit-identical for 1, 2 and 3 slabs, on every rank."""
    one = rho_world(1)[0]
    assert one[1] > 1 and one[2]
    for world in (2, 3):
        res = rho_world(world)
        assert all(res[r] == one for r in range(world)), (world, res, one)
