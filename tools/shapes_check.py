import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from oracle.oracle import Oracle
from paper_2401_01745_b200 import capi
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem
orc = Oracle()
def run(p, y0, n, rF, rS, pair):
    os.environ["EMRKC_PAIR"] = str(pair)
    op = MonodomainOperator(p); op.set_state(y0)
    res = op.run(0, n, 0.05, rF, rS).as_dict(); res.pop("device_ms")
    nk = capi.load().emrkc_node_kernel(op.handle)
    y = op.get_state(); op.close(); return y, res, nk
ok = True
for shape, rF in [((1024, 512, 2), 16.0), ((66, 1000, 3), 100.0), ((2, 4000, 40), 16.0), ((512, 2, 300), 100.0),
                  ((130, 6, 40), 100.0), ((64, 4, 600), 500.0), ((192, 190, 17), 16.0)]:
    h = 0.1
    p = make_problem(3, list(shape), [h]*3, [0.2, 0.1, 0.05], 140.0, 0.01, 70.0, [-0.05]*3, [0.75]*3, 0.0, 1.0)
    y0 = orc.initial_state(p); rng = np.random.default_rng(1)
    y0[:p.n_nodes] += rng.normal(0, 0.1, p.n_nodes)
    ya, ra, ka = run(p, y0, 5, rF, 0.7, 1)
    yb, rb, kb = run(p, y0, 5, rF, 0.7, 0)
    same = np.array_equal(ya, yb) and ra == rb
    ok &= same
    print(shape, "m", ra["m"], "node_kernel", ka, kb, "bitwise", same, flush=True)
print("ALL OK" if ok else "MISMATCH")
