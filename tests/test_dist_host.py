"""Host logic of bench.py's N > 1 arm (no GPU): weak-scaling workloads and
per-rank initial slabs."""
import numpy as np
import pytest

from paper_2401_01745_b200 import dist, workloads


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_z_scaled_slabs_hold_one_copy(world):
    base = workloads.get("hh3d_sweep_25")
    w = workloads.z_scaled(base, world)
    p = w.problem
    assert [int(p.n[a]) for a in range(3)] == [25, 25, 25 * world]
    assert w.n_nodes == world * base.n_nodes
    for r in range(world):
        part = dist.partition(p, world, r)
        assert int(part.z_end) - int(part.z_begin) == 25
    # same physics apart from the z extent
    for a in range(3):
        assert p.dx[a] == base.problem.dx[a] and p.sigma[a] == base.problem.sigma[a]
        assert p.stim_lo[a] == base.problem.stim_lo[a] and p.stim_hi[a] == base.problem.stim_hi[a]


@pytest.mark.parametrize("name,world", [("hh3d_sweep_25", 3), ("hh3d_sweep_25", 4),
                                        ("hh3d_256x256x128", 2)])
def test_slab_initial_state_matches_global(name, world):
    w = workloads.get(name)
    if w.n_nodes > 2_000_000:
        w = workloads.get("hh3d_sweep_50")
        w.noise = "mult_uniform_0.01"  # the other noise kind on a small grid
    y = w.initial_state()
    for r in range(world):
        part = dist.partition(w.problem, world, r)
        np.testing.assert_array_equal(dist.slab_initial_state(w, part),
                                      dist.slab_of(w.problem, part, y))


@pytest.mark.parametrize("nz,world,expect", [(200, 8, 25), (48, 5, 9), (25, 4, 6), (128, 1, 128)])
def test_min_slab_depth(nz, world, expect):
    """Every rank derives the same smallest slab depth (the switch of the
    K-plane d_1 halo must agree across ranks)."""
    w = workloads.get("hh3d_sweep_25")
    p = workloads.z_scaled(w, 1).problem
    p.n[2] = nz
    depths = [int(dist.partition(p, world, r).z_end - dist.partition(p, world, r).z_begin)
              for r in range(world)]
    assert sum(depths) == nz
    assert dist.min_slab_depth(p, world) == min(depths) == expect
