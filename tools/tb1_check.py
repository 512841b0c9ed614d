"""EMRKC_TB=2 (m = 2 through k_vin_tb<1>) against the default inner-stage kernel: bitwise."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem
orc = Oracle()
def run(p, y0, n, rF, rS, tb):
    os.environ["EMRKC_TB"] = str(tb)
    op = MonodomainOperator(p); op.set_state(y0)
    res = op.run(0, n, 0.05, rF, rS).as_dict(); res.pop("device_ms")
    y = op.get_state(); op.close(); return y, res
ok = True
for shape, rF, rS in [((72, 18, 21), 100.0, 0.7), ((130, 34, 9), 100.0, 0.7), ((40, 36, 50), 100.0, 50.0), ((256, 128, 64), 100.0, 0.7)]:
    p = make_problem(3, list(shape), [0.1]*3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, [-0.05]*3, [0.75]*3, 0.0, 1.0)
    y0 = orc.initial_state(p); y0[:p.n_nodes] += np.random.default_rng(1).normal(0, 0.1, p.n_nodes)
    ya, ra = run(p, y0, 6, rF, rS, 2); yb, rb = run(p, y0, 6, rF, rS, 1)
    same = np.array_equal(ya, yb) and ra == rb; ok &= same
    print(shape, "s", ra["s"], "m", ra["m"], "bitwise", same, flush=True)
print("ALL OK" if ok else "MISMATCH")
