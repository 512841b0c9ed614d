import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from oracle.oracle import Oracle
from paper_2401_01745_b200 import convergence as cv
from paper_2401_01745_b200.monodomain import make_problem
o = Oracle()
p = make_problem(2, [64, 48], [0.25, 0.25], [0.1, 0.1], 140.0, 0.01, 70.0, [-0.125, -0.125], [3.875, 3.875], 0.0, 1.0)
y0 = o.initial_state(p); y0[:p.n_nodes] += np.random.default_rng(1).normal(0.0, 0.1, p.n_nodes)
for t_end, dts, dref in [(2.0, [0.1, 0.05, 0.025, 0.0125], 0.0005), (1.0, [0.02, 0.01, 0.005], 0.0001), (0.5, [0.05, 0.025, 0.0125], 0.0001)]:
    tab = cv.run_convergence(p, y0, t_end, dts, "emrkc", dt_ref=dref)
    print(t_end, [(r.dt, r.err, r.order, r.s, r.m) for r in tab.rows])
