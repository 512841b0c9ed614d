"""The distributed (one process per GPU) protocol, exercised on one GPU:
adjacent slab handles are linked directly (no IPC) and every launch is
serialised, so each device-side arrival wait is already satisfied when its
kernel starts (never a kernel waiting on a concurrent one). Checks the
peer-store halos, arrival counters, prime level, checkpoint and replay."""
import ctypes as C

import numpy as np
import pytest

from paper_2401_01745_b200 import capi, dist, workloads
from paper_2401_01745_b200.capi import RunResult
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem

pytestmark = pytest.mark.gpu


def setup_slabs(p, y0, nslab):
    lib = capi.load()
    ops = []
    for r in range(nslab):
        part = dist.partition(p, nslab, r)
        op = MonodomainOperator(p, 0, part)
        op.set_state(dist.slab_of(p, part, y0))
        ops.append((op, part))
    for (lo, _), (hi, _) in zip(ops, ops[1:]):
        assert lib.emrkc_dist_link_local(lo.handle, hi.handle) == 0, lib.emrkc_global_error()
    return ops


def lockstep(ops, replay, step0, n, dt, rF, rS):
    lib = capi.load()
    arr = (C.c_void_p * len(ops))(*[o.handle.value for o, _ in ops])
    res = RunResult()
    rc = lib.emrkc_dist_lockstep_run(arr, len(ops), replay, step0, n, dt, 0.05, 0, rF, rS,
                                     C.byref(res))
    assert rc == 0, lib.emrkc_global_error()
    return res


def gather(p, ops):
    nn = p.n_nodes
    plane = nn // int(p.n[p.dim - 1])
    y = np.empty(4 * nn)
    for op, part in ops:
        loc = op.get_state()
        nl = plane * (part.z_end - part.z_begin)
        for b in range(4):
            s0 = b * nn + part.z_begin * plane
            y[s0:s0 + nl] = loc[b * nl:(b + 1) * nl]
    return y


# *_tb: rho_F forced so that 2 <= K = m - 1 <= 4 inner stages run temporally
# blocked (k_vin_tb) on every slab, with the K-plane d_1 halo between slabs
TB_CASES = {"3d_tb_m3": (3, 1), "3d_tb_m5": (5, 1), "3d_tb_s2m4": (4, 2)}


# *@pair: the pair-per-thread node kernel forced on these small grids
# (EMRKC_PAIR=2; it is the default on large 3-D grids): ghost planes, halo
# puts and arrival counts of k_node_pair on slabs
@pytest.mark.parametrize("nslab", [2, 3, 4])
@pytest.mark.parametrize("case", ["3d_m2", "2d_m1", "3d_m1", *TB_CASES, "3d_m2@pair",
                                  "3d_m1@pair", "3d_tb_m3@pair", "3d_tb_s2m4@pair"])
def test_dist_protocol_bitwise(case, nslab, monkeypatch):
    monkeypatch.setenv("EMRKC_PAIR", "2" if case.endswith("@pair") else "0")
    case = case.split("@")[0]
    if case in TB_CASES:
        monkeypatch.setenv("EMRKC_TB", "1")  # the default
    if case == "3d_m2":
        w = workloads.parity_3d()
        p, y0, dt, rF, rS, n = w.problem, w.initial_state(), w.dt, 400.0, 50.0, 6
    elif case == "3d_tb_m3":
        w = workloads.hh3d_sweep(25)
        p, y0, dt, rF, rS, n = w.problem, w.initial_state(), w.dt, 250.0, 0.7, 10
    elif case == "3d_tb_m5":
        w = workloads.parity_3d()
        p, y0, dt, rF, rS, n = w.problem, w.initial_state(), w.dt, 700.0, 0.7, 6
    elif case == "3d_tb_s2m4":
        w = workloads.parity_3d()
        p, y0, dt, rF, rS, n = w.problem, w.initial_state(), w.dt, 1500.0, 50.0, 6
    elif case == "2d_m1":
        p = make_problem(2, [96, 64], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                         [-0.125, -0.125], [3.875, 3.875], 0.0, 1.0)
        w = None
        y0 = MonodomainOperator(p).initial_state()
        y0[: p.n_nodes] += np.random.default_rng(0).normal(0, 0.1, p.n_nodes)
        dt, rF, rS, n = 0.05, 10.0, 0.7, 20
    else:
        w = workloads.hh3d_sweep(25)
        p, y0, dt, rF, rS, n = w.problem, w.initial_state(), w.dt, 6.0, 0.7, 10
    whole = MonodomainOperator(p)
    whole.set_state(y0)
    rw = whole.run(0, n, dt, rF, rS)
    yw = whole.get_state()
    ops = setup_slabs(p, y0, nslab)
    res = lockstep(ops, 0, 0, n, dt, rF, rS)
    assert np.array_equal(gather(p, ops), yw)
    assert (res.s, res.m, res.n_fF, res.aborted) == (rw.s, rw.m, rw.n_fF, 0)
    if case in TB_CASES:
        assert (res.m, res.s) == TB_CASES[case]
    # a second run continues the counters / level bookkeeping consistently
    res2 = lockstep(ops, 0, n, 3, dt, rF, rS)
    whole.run(n, 3, dt, rF, rS)
    assert np.array_equal(gather(p, ops), whole.get_state())
    assert res2.aborted == 0


def test_dist_abort_then_replay():
    """Rank 1 hits a non-finite gate: ranks do not fold abort words in a
    distributed run, so the host combines the records and every slab replays
    the steps before the first abort from the run's checkpoint."""
    p = make_problem(2, [64, 60], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0,
                     [-0.125, -0.125], [3.875, 3.875], 0.0, 1.0)
    whole = MonodomainOperator(p)
    y0 = whole.initial_state()
    y0[: p.n_nodes] += np.random.default_rng(1).normal(0, 0.1, p.n_nodes)
    y0[p.n_nodes + 64 * 45 + 3] = 5.0  # an out-of-range gate: blows up later
    whole.set_state(y0)
    rw = whole.run(0, 30, 0.05, 10.0, 0.7)
    ops = setup_slabs(p, y0, 2)
    # (never drive linked slabs one at a time from one thread: a slab's
    # boundary blocks would wait for a neighbour that is not running)
    res = lockstep(ops, 0, 0, 30, 0.05, 10.0, 0.7)  # min over slabs, no folding
    glob = res.as_dict()
    assert glob["aborted"] == rw.aborted
    if glob["aborted"]:
        assert glob["abort_step"] == rw.abort_step and glob["abort_kind"] == rw.abort_kind
        k = dist.replay_steps(glob, 0)
        lockstep(ops, 1, 0, k, 0.05, 10.0, 0.7)
    assert np.array_equal(gather(p, ops), whole.get_state(), equal_nan=True)
