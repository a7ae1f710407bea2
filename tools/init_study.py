"""Initialisation study (Table 1) on the B200 path.

For the BASELINE configurations 0-2 and the three hidden-layer schemes of the paper -- suggested
eqn:init (l = sqrt(n)/8, b = -w.xi), manual (l = 1, reading R8) and He (l = sqrt(2/n_N), b = 0,
P:549) -- solve with the CUDA path and report the interface RMSE sqrt(mean (u_Gamma - u_exact)^2)
(the quantity of Table 1) and the relative L2 error on the 101^2 grid.  The paper's numbers are
for its own (2^8+1)^2 lattice workload and are printed as context only.
usage: python tools/init_study.py [out.json]   (GPU box)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402

SCHEMES = {0: "suggested (eqn:init, l = sqrt(n)/8)", 1: "manual (l = 1)", 2: "He (l = sqrt(2/n_N), b = 0)"}
PAPER = {"He": [8.4230e-03, 1.7173e-04, 1.1454e-05], "Manual": [4.9389e-10, 4.0850e-09, 6.5790e-08],
         "Suggested": [2.8926e-10, 7.5946e-10, 2.9894e-09], "N": ["2x2", "4x4", "8x8"],
         "source": "PAPER.md Table 1 (tab:initial, P:554-566): n = 2^16 total neurons, (2^8+1)^2 lattice"}


def interface_rmse(prob, res):
    ctx = res["ctx"]
    xy = ctx.interface_points()
    if xy.shape[0] == 0:
        return 0.0
    ue = WL.exact(prob.problem, xy)
    return float(np.sqrt(np.mean((res["uG"].numpy() - ue) ** 2)))


def main(out=None):
    xy = WL.eval_grid()
    rows = []
    for k in (0, 1, 2):
        for sch in (0, 1, 2):
            c = WL.config(k, init_scheme=sch)
            prob = E.Problem.from_config(c)
            res = E.solve(prob, xy, return_all=True)
            ue = WL.exact(c["problem"], xy)
            u = res["u"].numpy()
            row = {"config": k, "P": c["P"], "M": c["M"], "scheme": SCHEMES[sch], "init_scheme": sch,
                   "interface_rmse": interface_rmse(prob, res),
                   "rel_l2_grid": float(np.linalg.norm(u - ue) / np.linalg.norm(ue))}
            rows.append(row)
            print(json.dumps(row), flush=True)
    d = {"rows": rows, "paper_table1_context": PAPER}
    if out:
        json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
