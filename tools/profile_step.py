"""One (or a few) hot-path steps of config k on cuda:0 -- a short command for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
c = WL.config(a.config)
ctx = E.Context(E.Problem.from_config(c))
buf = ctx.alloc()
xy = torch.as_tensor(WL.eval_grid().reshape(-1), device="cuda")
u = torch.zeros(xy.numel() // 2, dtype=torch.float64, device="cuda")
for _ in range(a.steps):
    ctx.run(buf, xy, u)
torch.cuda.synchronize()
print("ok", ctx.timing()["launches"])
