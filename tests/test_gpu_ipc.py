"""The cross-process z-slab path on one GPU: two and three torch.distributed ranks
(gloo) export / import CUDA IPC ghost arenas and run emrkc_dist_run in
lockstep (tests/_ipc_lockstep.py); the gathered state must be bitwise the
whole-grid run's (the stencil has no order-dependent reductions)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2401_01745_b200 import workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", params=[2, 3])
def ranks(request, tmp_path_factory):
    out = tmp_path_factory.mktemp("ipc") / f"ipc{request.param}.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={request.param}", "--master-addr", "127.0.0.1",
           "--master-port", str(29617 + request.param), os.path.join(HERE, "_ipc_lockstep.py"),
           str(out)]
    subprocess.run(cmd, check=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("name", ["p3d_48_s2m2", "hh2d_256x256", "hh3d_sweep_25",
                                  "p3d_48_s2m2@tb"])
def test_ipc_slabs_bitwise(ranks, name):
    two_ranks = ranks
    w = workloads.get(name.split("@")[0])
    rF, rS = two_ranks[name + "/rho"]
    n = int(two_ranks[name + "/n"][0])
    op = MonodomainOperator(w.problem)
    op.set_state(w.initial_state())
    res = op.run(0, n, w.dt, float(rF), float(rS), w.eps)
    y = op.get_state()
    op.close()
    s, m, aborted, nff = two_ranks[name + "/rec"]
    assert (res.s, res.m, res.aborted, res.n_fF) == (s, m, aborted, nff)
    if name.endswith("@tb"):
        assert (s, m) == (1, 5)  # K = 4 blocked stages: the widest halo
    got = two_ranks[name + "/y"]
    assert np.array_equal(got, y), np.abs(got - y).max()


@pytest.mark.parametrize("name", ["p3d_48_s2m2", "hh2d_256x256", "hh3d_sweep_25"])
def test_distributed_rho_bitwise(ranks, name):
    """rho_F / rho_S by the distributed power iteration over 2 / 3 ranks'
    slabs (dist.slab_rho, emrkc_slab_power_*) equal the whole-grid estimate
    bit for bit, with the same iteration counts."""
    from paper_2401_01745_b200 import capi

    w = workloads.get(name)
    op = MonodomainOperator(w.problem)
    op.set_state(w.initial_state())
    eF = op.estimate_spectral_radius(capi.EMRKC_RHS_F)
    eS = op.estimate_spectral_radius(capi.EMRKC_RHS_S)
    op.close()
    rF, iF, rS, iS = ranks[name + "/drho"]
    assert (rF, int(iF)) == (eF.rho, eF.iterations)
    assert (rS, int(iS)) == (eS.rho, eS.iterations)

