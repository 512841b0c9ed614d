"""One small run per staged-kernel family; compares EMRKC_PIPE=$1 with the
march kernels (EMRKC_PIPE=0) bit for bit (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

case = sys.argv[1]
pipe = sys.argv[2] if len(sys.argv) > 2 else "3"
from paper_2401_01745_b200 import workloads  # noqa: E402
from paper_2401_01745_b200.monodomain import MonodomainOperator, make_problem  # noqa: E402

if case == "3d":
    p = make_problem(3, (64, 32, 16), (0.1, 0.1, 0.1), (0.1, 0.1, 0.1))
    rF, rS, dt = None, None, 0.05
elif case == "3d_m2":
    p = make_problem(3, (64, 32, 16), (0.1, 0.1, 0.1), (0.1, 0.1, 0.1))
    rF, rS, dt = None, None, 0.5
elif case == "2d":
    p = make_problem(2, (256, 40), (0.1, 0.1), (0.1, 0.1))
    rF, rS, dt = None, None, 0.05
else:
    raise SystemExit(case)
nn = p.n_nodes
rng = np.random.default_rng(1)
outs = []
for pp in ("0", pipe):
    os.environ["EMRKC_PIPE"] = pp
    op = MonodomainOperator(p)
    y = op.initial_state()
    y[:nn] += rng.normal(0, 5.0, nn) if not outs else 0
    if not outs:
        y0 = y.copy()
    op.set_state(y0)
    if rF is None:
        rF = op.estimate_spectral_radius(0).rho
        rS = op.estimate_spectral_radius(1).rho
    res = op.run(0, 3, dt, rF, rS)
    outs.append(op.get_state())
    print(f"pipe={pp} s={res.s} m={res.m} aborted={res.aborted}", flush=True)
    op.close()
d = np.abs(outs[0] - outs[1])
print(case, "max |diff| per block", [float(d[b * nn:(b + 1) * nn].max()) for b in range(4)])
if d.max() > 0:
    i = int(np.argmax(d[:nn]))
    print("worst V node", i, outs[0][i], outs[1][i])
