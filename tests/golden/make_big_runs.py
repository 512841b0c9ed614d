"""Generate tests/golden/big_<workload>.npz from the REFERENCE ITSELF
(oracle/_ref, the unmodified reference sources) for the BASELINE grids too
large to store whole: config 3's grid (256x256x128, 400 steps = T) and
config 4's grid (512x512x256, run to T or to the reference's own abort),
both with HH standing in for the absent CRN / TTP models (SURVEY §8(c)
option 1), plus re-runs of smaller grids.

The run is run_simulation's emRKC loop (P/src/simulate.cpp:176-229) from the
workload's seeded initial state (paper_2401_01745_b200.workloads, numpy
PCG64: identical bytes on every machine; the resting state comes from the
reference's own resting_state, so this script never maps the product
library). Stored per run:

* the run record (s, m, eta, counters, gate range, abort step / kind /
  stage), rho_F / rho_S with their iteration counts;
* per block (V, m, h, n): the L2 norm, the sum, per-plane (slowest axis)
  sums and sums of squares, and 65,536 seeded sample nodes;
* with ``--sens SEED ...``: the reference's divergence from ITSELF when its
  initial state is perturbed by 1e-15 relative (trapezoid rel_l2_error per
  block, P/src/monodomain.cpp:92-110), one entry per seed.

    python tests/golden/make_big_runs.py hh3d_512x512x256 [--steps N] [--sens 5 6 7]

Run here, where /root/reference exists (the .npz files travel to the GPU
box; the reference does not).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402
from paper_2401_01745_b200 import workloads  # noqa: E402

NSAMP = 65536


def block_stats(y, nn, n_planes):
    out = {}
    for b in range(len(y) // nn):
        blk = y[b * nn:(b + 1) * nn]
        pl = blk.reshape(n_planes, -1)
        out[f"norm2_{b}"] = np.float64(np.linalg.norm(blk))
        out[f"sum_{b}"] = np.float64(blk.sum())
        out[f"plane_sum_{b}"] = pl.sum(axis=1)
        out[f"plane_sq_{b}"] = np.einsum("ij,ij->i", pl, pl)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--steps", type=int, default=0, help="0: the workload's T")
    ap.add_argument("--sens", type=int, nargs="*", default=[])
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ref = Reference()
    w = workloads.get(a.workload)
    p = w.problem
    n = a.steps or w.n_steps
    y0 = w.initial_state(resting=ref.resting_state)
    t0 = time.time()
    rF, _ = ref.estimate_rho(p, 0, 0.0, y0)
    rS, _ = ref.estimate_rho(p, 1, 0.0, y0)
    print(f"{w.name}: rho_F {rF.rho!r} ({rF.iterations} it), rho_S {rS.rho!r} "
          f"({rS.iterations} it), {time.time() - t0:.0f} s", flush=True)
    y, res, wall = ref.run(p, y0, 0, n, w.dt, w.eps, rF.rho, rS.rho)
    rec = {k: (float(v) if isinstance(v, float) else int(v))
           for k, v in res.as_dict().items() if k != "device_ms"}
    print(w.name, rec, f"{wall:.0f} s", flush=True)
    nn = p.n_nodes
    n_planes = int(p.n[p.dim - 1])
    idx = np.sort(np.random.default_rng(1234).choice(nn, min(NSAMP, nn), replace=False))
    sens = []
    for seed in a.sens:
        y1 = y0 * (1.0 + 1e-15 * np.random.default_rng(seed).uniform(-1.0, 1.0, y0.size))
        yp, resp, _ = ref.run(p, y1, 0, n, w.dt, w.eps, rF.rho, rS.rho)
        sv = [float(ref_rel_l2(ref, p, yp[b * nn:(b + 1) * nn], y[b * nn:(b + 1) * nn]))
              for b in range(p.n_fields)]
        same = bool(resp.abort_step == res.abort_step and resp.aborted == res.aborted)
        sens.append({"seed": seed, "rel_l2": sv, "same_abort": same})
        print(w.name, "sensitivity seed", seed, sv, "same abort", same, flush=True)
        del yp, y1
    meta = {"workload": w.name, "steps": n, "dt": w.dt, "eps": w.eps,
            "rho_F": rF.rho, "rho_F_iterations": rF.iterations,
            "rho_S": rS.rho, "rho_S_iterations": rS.iterations,
            "record": rec, "ref_wall_s": wall, "sensitivity": sens,
            "generator": "tests/golden/make_big_runs.py (oracle/_ref = reference sources)"}
    st = block_stats(y, nn, n_planes)
    out = a.out or os.path.join(HERE, f"big_{w.name}.npz")
    np.savez_compressed(out, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
                        sample_index=idx.astype(np.int64),
                        sample=np.stack([y[b * nn:(b + 1) * nn][idx] for b in range(p.n_fields)]),
                        **st)
    print("wrote", out, flush=True)


def ref_rel_l2(ref, p, a, b):
    """The reference's own trapezoid rel_l2_error (oracle/_ref)."""
    return ref.rel_l2(p, a, b)


if __name__ == "__main__":
    main()
