"""Quick timing probe (not the bench): device ms/step of emrkc_run per workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_01745_b200 import workloads  # noqa: E402
from paper_2401_01745_b200.monodomain import MonodomainOperator  # noqa: E402

names = sys.argv[1:] or ["hh3d_128x128x128", "hh3d_512x512x256"]
for fast in (("1",) if os.environ.get("EMRKC_PROBE_FAST_ONLY") else ("1", "0")):
    os.environ["EMRKC_FAST"] = fast
    for name in names:
        w = workloads.get(name)
        t0 = time.time()
        y0 = w.initial_state()
        op = MonodomainOperator(w.problem)
        op.set_state(y0)
        t1 = time.time()
        rF = op.estimate_spectral_radius(0).rho
        rS = op.estimate_spectral_radius(1).rho
        t2 = time.time()
        op.run(0, 3, w.dt, rF, rS)
        n = 20
        res = op.run(3, n, w.dt, rF, rS)
        ms = res.device_ms / n
        nsps = w.n_nodes / (ms * 1e-3)
        gbs = 64 * w.n_nodes / (ms * 1e-3) / 1e9
        print(f"fast={fast} {name}: s={res.s} m={res.m} rho_F={rF:.4f} rho_S={rS:.4f} "
              f"{ms:.4f} ms/step {nsps:.3e} node-steps/s alg {gbs:.0f} GB/s "
              f"(setup {t1-t0:.1f}s rho {t2-t1:.1f}s)", flush=True)
        op.close()
