"""The paper's CG interface solver vs the direct envelope Cholesky:
iterations to the paper's relative residual 1e-9, device time, and the error vs the
exact solution, for configs 0-2 (and 3 with --big).  usage: python tools/cg_study.py [out.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402


def main(out=None, ks=(0, 1, 2)):
    rows = []
    xy = WL.eval_grid()
    for k in ks:
        c = WL.config(k)
        ctx = E.Context(E.Problem.from_config(c))
        buf = ctx.alloc()
        xy_t = torch.as_tensor(xy.reshape(-1), device="cuda")
        u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
        ctx.run(buf, xy_t, u)  # Cholesky solution (and all buffers)
        torch.cuda.synchronize()
        ue = WL.exact(c["problem"], xy)
        err_chol = float(np.linalg.norm(u.cpu().numpy() - ue) / np.linalg.norm(ue))
        uG_chol = buf["uG"].clone()
        ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, rr = ctx.interface_cg(buf["Mband"], buf["g"], buf["uG"], buf["work"], tol=1e-9)
        t_cg = time.perf_counter() - t0
        ctx.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"])
        ctx.evaluate(buf["W"], buf["b"], buf["coef"], xy_t, u)
        torch.cuda.synchronize()
        G = ctx.sizes["G"]
        row = {"config": k, "G": G, "cg_iterations": it, "cg_relres": rr, "cg_seconds": t_cg,
               "rel_l2_vs_exact_cg": float(np.linalg.norm(u.cpu().numpy() - ue) / np.linalg.norm(ue)),
               "rel_l2_vs_exact_cholesky": err_chol,
               "uG_cg_vs_cholesky": float((buf["uG"][:G] - uG_chol[:G]).norm() / uG_chol[:G].norm())}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ctx, buf
    if out:
        json.dump({"rows": rows, "tolerance": "relative residual 1e-9 (PAPER.md P:439)"}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
