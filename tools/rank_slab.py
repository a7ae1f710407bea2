"""Local phases of ONE rank's slab on one GPU: the per-rank work of a world-size-W run of config
k (subdomains [0, N/W)), timed per phase with CUDA events -- used to tune the QR stream grouping
for the multi-GPU slabs without a multi-GPU box.  usage: python tools/rank_slab.py K W [groups...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402


def run(k, world, groups):
    if groups:
        os.environ["ELMDDM_QR_GROUPS"] = str(groups)
    c = WL.config(k)
    N = c["P"] ** 2
    s0, s1 = E.partition(N, world, 0)
    ctx = E.Context(E.Problem.from_config(c), s0, s1)
    buf = ctx.alloc()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for rep in range(3):
        ev[0].record()
        ctx.init_hidden(buf["W"], buf["b"])
        ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
        ev[1].record()
        ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
        ev[2].record()
        ctx.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"])
        ev[3].record()
        ctx.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"])
        ev[4].record()
        torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    print(f"cfg{k} world {world} slab [{s0},{s1}) groups {groups or 'default'}: assemble {t[0]:.2f} "
          f"local_factor {t[1]:.2f} schur {t[2]:.2f} back {t[3]:.2f} total {sum(t):.2f} ms", flush=True)


if __name__ == "__main__":
    k, world = int(sys.argv[1]), int(sys.argv[2])
    for g in (sys.argv[3:] or [0]):
        run(k, world, int(g))
