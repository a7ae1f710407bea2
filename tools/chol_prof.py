"""Timeline of the persistent interface Cholesky (profiling build with -DELM_CHOL_PROF).
usage: python tools/chol_prof.py [config]   (on a GPU box)"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.path.join(ROOT, "paper_2406_15959_b200", "libelmddm_prof.so")
os.environ["ELMDDM_LIB"] = lib  # before the package import: _lib reads it at import time
from paper_2406_15959_b200 import build as B  # noqa: E402

B.build(force=True, extra=["-DELM_CHOL_PROF"], lib=lib)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = WL.config(k)
ctx = E.Context(E.Problem.from_config(c))
buf = ctx.alloc()
ctx.run(buf)
torch.cuda.synchronize()
ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
torch.cuda.synchronize()
L = E._lib.load()
_, _, tasks = ctx.chol_plan()
n = len(tasks)
arr = np.zeros(n * 6, dtype=np.uint64)
L.elmddm_debug_chol_prof.argtypes = [C.c_void_p, C.c_int]
L.elmddm_debug_chol_prof(arr.ctypes.data_as(C.c_void_p), n)
a = arr.reshape(n, 6).astype(np.float64)
t0 = a[:, 0].min()
st, en, fw, dw, ep, cta = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2] / 1e3, a[:, 3] / 1e3, (a[:, 4] - t0) / 1e3, a[:, 5]
I, J = tasks[:, 0], tasks[:, 1]
span = en.max()
ncta = int(cta.max()) + 1
print(f"cfg{k}: {n} tasks on {ncta} CTAs, span {span:.0f} us")
busy = (en - st).sum()
print(f"task time {busy / ncta:.0f} us/CTA ({100 * busy / ncta / span:.0f}% of span); flag waits {fw.sum() / ncta:.0f} us/CTA, "
      f"data waits {dw.sum() / ncta:.0f} us/CTA, epilogues {(en - ep).sum() / ncta:.0f} us/CTA")
# gaps between consecutive tasks of a CTA
gaps = 0.0
for b in range(ncta):
    idx = np.where(cta == b)[0]
    s_, e_ = st[idx], en[idx]
    o = np.argsort(s_)
    gaps += (s_[o][1:] - e_[o][:-1]).sum() + s_[o][0]
print(f"idle between tasks {gaps / ncta:.0f} us/CTA")
diag = {int(j): i for i, (ii, j) in enumerate(zip(I, J)) if ii == j}
nb = int(J.max()) + 1
dend = np.array([en[diag[j]] for j in range(nb)])
srt = np.sort(dend)
print("diag ends sorted at 0,10%,..,100%:", [round(float(srt[int(f * (nb - 1))]), 0) for f in np.linspace(0, 1, 11)])
print("last 64 columns: diag end (us):", [round(float(x)) for x in dend[-64:]])
steps = np.diff(dend[-64:])
print(f"last-64 frontier step: median {np.median(steps):.1f} us, mean {steps.mean():.1f} us")
ntask_col = np.bincount(J, minlength=nb)
print("tasks per column (last 64):", ntask_col[-64:].tolist())
# critical chain of a column: tile (j, j-1) when it exists
for j in [nb // 4, nb // 2, 3 * nb // 4, nb - 30, nb - 2]:
    sub = {(int(x), int(y)): i for i, (x, y) in enumerate(zip(I, J)) if y in (j - 1, j) and x <= j}
    t1 = sub.get((j, j - 1))
    if t1 is None:
        continue
    d0, d1 = diag[j - 1], diag[j]
    print(f"col {j}: diag{j-1} end {en[d0]:.1f}; tile({j},{j-1}) start {st[t1]:.1f} epi {ep[t1]:.1f} end {en[t1]:.1f} "
          f"(flagwait {fw[t1]:.1f}); diag{j} start {st[d1]:.1f} epi {ep[d1]:.1f} end {en[d1]:.1f} (flagwait {fw[d1]:.1f} datawait {dw[d1]:.1f})")

# diagonal-task stages: [epi start, flags seen, loads landed, trsm done, C stored, potrf done, stores done, fence done]
nb = int(J.max()) + 1
dp = np.zeros(min(nb, 4096) * 8, dtype=np.uint64)
L.elmddm_debug_chol_dprof.argtypes = [C.c_void_p, C.c_int]
L.elmddm_debug_chol_dprof(dp.ctypes.data_as(C.c_void_p), min(nb, 4096))
dp = dp.reshape(-1, 8).astype(np.float64) / 1e3
names = ["flags", "loads", "trsm", "update", "potrf", "stores", "fence"]
sel = dp[1:, :]
sel = sel[(sel[:, 1] > 0)]
d = np.diff(sel, axis=1)
print("diag-task stage medians (us):", {n: round(float(np.median(d[:, i])), 1) for i, n in enumerate(names)})
print("diag-task stage means   (us):", {n: round(float(np.mean(d[:, i])), 1) for i, n in enumerate(names)})

# ---- the top dissection node: when do its tiles' pre-aggregation tasks (kind 1) and the rest run?
kind = tasks[:, 2].astype(int)
nupd_t = tasks[:, 3]
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"chol_prof_cfg{k}.npz"), tasks=tasks, st=st, en=en, fw=fw, dw=dw,
                    ep=ep, cta=cta)
top0 = nb - 64
for kd in (0, 1, 2):
    m = (J >= top0) & (kind == kd)
    if m.sum():
        nk = None
        print(f"top-64 columns, kind {kd}: {m.sum()} tasks, {nupd_t[m].sum()} updates, start {np.percentile(st[m], [0, 50, 100]).round(0).tolist()} "
              f"end {np.percentile(en[m], [0, 50, 100]).round(0).tolist()} us, CTA time {(en[m] - st[m]).sum() / 1e3:.0f} ms "
              f"(flag waits {fw[m].sum() / 1e3:.0f} ms)")
# CTA activity in the last 30% of the span: what were the CTAs doing?
t_tail = 0.7 * span
m = en > t_tail
busy_tail = (np.minimum(en[m], span) - np.maximum(st[m], t_tail)).sum()
print(f"last 30% of the span: CTA-time {busy_tail / 1e3:.0f} ms of {ncta * 0.3 * span / 1e3:.0f} ms available; "
      f"tasks overlapping it by kind: {np.bincount(kind[m], minlength=3).tolist()}, by column >= top0: {(J[m] >= top0).sum()}")
