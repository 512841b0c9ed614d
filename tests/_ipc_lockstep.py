"""Two ranks on ONE GPU drive the real cross-process path (CUDA IPC export /
import, peer stores into the neighbour's ghost arena, system-scope arrival
counters) in lockstep: a level hook syncs each rank's stream and meets the
other rank at a gloo barrier after every stencil level, so no kernel ever
spins on a concurrently running one (ranks sharing a GPU must not).
Launched by tests/test_gpu_ipc.py under torch.distributed.run; rank 0
writes the gathered state and records to argv[1]."""
import os
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_01745_b200 import capi, dist as pdist, workloads  # noqa: E402
from paper_2401_01745_b200.monodomain import _lib  # noqa: E402

HOOK = capi.LEVEL_HOOK


def main(out):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = pdist.DistContext(rank, world,
                            lambda b: _gather(b, world), lambda d: _gather(d, world),
                            *pdist.torch_p2p(rank, world))
    results = {}
    # key@tb: rho_F forced up to m = 5 with s = 1, so the inner stages 2..5
    # run temporally blocked with the wide (K = 4 plane) d_1 halo
    cases = [("p3d_48_s2m2", 12), ("hh2d_256x256", 10), ("hh3d_sweep_25", 15),
             ("p3d_48_s2m2@tb", 6)]
    for key, n in cases:
        name = key.split("@")[0]
        w = workloads.get(name)
        rF = 16.0 if w.problem.dim == 3 else 9.1
        rS = w.rho_S_forced if w.rho_S_forced is not None else 0.7114
        if key.endswith("@tb"):
            rF, rS = 700.0, 0.7114
        # handles read EMRKC_TB when created (on by default)
        os.environ["EMRKC_TB"] = "1" if key.endswith("@tb") else "0"
        slab = pdist.DistSlab(w.problem, ctx, 0)
        slab.link()
        barrier = HOOK(lambda _c: dist.barrier())
        lib = _lib()
        assert lib.emrkc_set_level_hook(slab.op._h, barrier, None) == 0
        slab.set_global_state(w.initial_state())
        # rho by the distributed power iteration over the slabs (norms
        # chained across ranks): bit-identical to the whole-grid estimate
        sp = pdist.DeviceSlabPower(slab.op)
        dF = pdist.slab_rho(sp, ctx, capi.EMRKC_RHS_F, 0.0)
        dS = pdist.slab_rho(sp, ctx, capi.EMRKC_RHS_S, 0.0)
        rec = slab.run(0, n, w.dt, rF, rS, w.eps)
        y = slab.op.get_state()
        ys = _gather(y, world)
        assert lib.emrkc_set_level_hook(slab.op._h, HOOK(), None) == 0
        slab.op.close()
        if rank == 0:
            nn = w.n_nodes
            parts = [pdist.partition(w.problem, world, r) for r in range(world)]
            plane = nn // int(w.problem.n[w.problem.dim - 1])
            full = np.empty(4 * nn)
            for r, part in enumerate(parts):
                a, b = int(part.z_begin) * plane, int(part.z_end) * plane
                m = b - a
                for k in range(4):
                    full[k * nn + a:k * nn + b] = ys[r][k * m:(k + 1) * m]
            results[key + "/y"] = full
            results[key + "/rec"] = np.array([rec["s"], rec["m"], rec["aborted"], rec["n_fF"]])
            results[key + "/rho"] = np.array([rF, rS])
            results[key + "/n"] = np.array([n])
            results[key + "/drho"] = np.array([dF.rho, dF.iterations, dS.rho, dS.iterations])
    if rank == 0:
        np.savez(out, **results)
    dist.barrier()
    dist.destroy_process_group()


def _gather(obj, world):
    lst = [None] * world
    dist.all_gather_object(lst, obj)
    return lst


if __name__ == "__main__":
    main(sys.argv[1])
