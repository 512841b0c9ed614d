"""Step-by-step GPU vs oracle comparison of a golden case (debug aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2401_01745_b200.capi import Problem  # noqa: E402
from paper_2401_01745_b200.monodomain import MonodomainOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "g1d_201_dt0.1"
H = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
meta = json.load(open(os.path.join(H, "golden.json")))[name]
d = np.load(os.path.join(H, name + ".npz"))
p = Problem.from_dict(meta["problem"])
orc = Oracle()
for fast in ("0", "1"):
    os.environ["EMRKC_FAST"] = fast
    op = MonodomainOperator(p)
    y = d["y0"].copy()
    op.set_state(y)
    nn = p.n_nodes
    for k in range(meta["n_steps"]):
        res = op.run(k, 1, meta["dt"], meta["rho_F"], meta["rho_S"])
        yg = op.get_state()
        y, ro, _ = orc.run(p, y, k, 1, meta["dt"], 0.05, meta["rho_F"], meta["rho_S"])
        errs = [orc.rel_l2(p, yg[b * nn:(b + 1) * nn], y[b * nn:(b + 1) * nn]) for b in range(4)]
        if res.aborted or max(errs) > 1e-12 or k % 20 == 0:
            print(f"fast={fast} step {k} s={res.s} m={res.m} aborted={res.aborted} kind={res.abort_kind} "
                  f"stage={res.abort_stage} errs={['%.2e' % e for e in errs]} "
                  f"Vmax={np.nanmax(np.abs(yg[:nn])):.3f} Vmax_ref={np.abs(y[:nn]).max():.3f}")
        if res.aborted or max(errs) > 1e-6:
            i = np.nanargmax(np.abs(yg[:nn] - y[:nn]))
            print("  worst node", i, yg[i], y[i], "gates", yg[nn + i::nn][:3], y[nn + i::nn][:3])
            break
    op.close()
