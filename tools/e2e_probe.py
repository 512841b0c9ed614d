"""e2e per-call step time (emrkc_step_host, pinned buffers) on one workload."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_01745_b200 import capi, workloads  # noqa: E402
from paper_2401_01745_b200.monodomain import MonodomainOperator  # noqa: E402

w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "hh3d_128x128x128")
lib = capi.load()
op = MonodomainOperator(w.problem)
y0 = w.initial_state()
op.set_state(y0)
rF = op.estimate_spectral_radius(0).rho
rS = op.estimate_spectral_radius(1).rho
hin = torch.from_numpy(y0.copy()).pin_memory()
hout = torch.empty_like(hin).pin_memory()
rep = capi.StepReport()
P = lambda x: C.cast(x.data_ptr(), capi.DP)  # noqa: E731
for _ in range(3):
    lib.emrkc_step_host(op.handle, 0.0, P(hin), P(hout), hin.numel(), w.dt, w.eps, 0, rF, rS, C.byref(rep))
k = 30
t0 = time.perf_counter()
for r in range(k):
    lib.emrkc_step_host(op.handle, r * w.dt, P(hin), P(hout), hin.numel(), w.dt, w.eps, 0, rF, rS,
                        C.byref(rep))
    hin, hout = hout, hin
dt = (time.perf_counter() - t0) / k
print(f"{w.name} chunks={os.environ.get('EMRKC_HOST_CHUNKS', '16')}: {dt * 1e3:.3f} ms/step "
      f"{w.n_nodes / dt:.3e} node-steps/s")
