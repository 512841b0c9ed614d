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


def test_z_slab_sample_is_the_central_planes(oracle):
    """bench.py's bounded CPU sample (workloads.z_slab_sample): the planes
    [z0, z0 + depth) of the workload's seeded initial state, the same
    spacing and conductivities, the stimulus box in the same global
    coordinates (the same nodes are stimulated), and the initial state from
    the reference's own resting state is the product's bit for bit."""
    w = workloads.get("hh3d_sweep_50")
    z0, d = 3, 9  # the 8^3 corner stimulus covers sample planes 0..4
    ws, ys = workloads.z_slab_sample(w, z0, d)
    p, q = w.problem, ws.problem
    assert [int(q.n[a]) for a in range(3)] == [50, 50, d]
    y = w.initial_state()
    nn, plane = p.n_nodes, 50 * 50
    for b in range(4):
        np.testing.assert_array_equal(ys[b * q.n_nodes:(b + 1) * q.n_nodes],
                                      y[b * nn + z0 * plane: b * nn + (z0 + d) * plane])
    for a in range(3):
        assert q.dx[a] == p.dx[a] and q.sigma[a] == p.sigma[a]
    # stimulated nodes: global z in the box <=> sample z + z0 in the box
    hits = 0
    for z in range(d):
        for node in (0, 7, 55):
            i_s = node + plane * z
            i_g = node + plane * (z + z0)
            st = oracle.stimulus_rate(q, 0.5, i_s) > 0
            assert st == (oracle.stimulus_rate(p, 0.5, i_g) > 0)
            hits += st
    assert hits == 3 * 5  # nodes 0, 7, 55 (x, y <= 7) on planes z + z0 = 3..7
    from oracle.oracle import Oracle

    np.testing.assert_array_equal(w.initial_state(resting=Oracle().resting_state), y)
