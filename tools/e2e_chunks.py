import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import bench
from paper_2401_01745_b200 import workloads
from paper_2401_01745_b200.monodomain import MonodomainOperator
w = workloads.get("hh3d_128x128x128")
op = MonodomainOperator(w.problem)
y0 = w.initial_state()
op.set_state(y0)
rF = op.estimate_spectral_radius(0).rho
rS = op.estimate_spectral_radius(1).rho
r = bench.measure_e2e(op, w, y0, rF, rS, 20)
print(os.environ.get("EMRKC_HOST_CHUNKS"), round(r["ms_per_step"], 3), "%.3e" % r["value"])
