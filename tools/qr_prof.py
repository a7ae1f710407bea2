"""Per-CTA timeline of the batched QR phase (profiling build with -DELM_QR_PROF): which SMs hold
panel (k_panel_t) and trailing-update (k_wy_tma) CTAs over time, and what the trailing-update
CTAs cost alone on an SM, beside another trailing-update CTA, or beside a panel CTA.
usage: python tools/qr_prof.py [config]   (on a GPU box)"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.path.join(ROOT, "paper_2406_15959_b200", "libelmddm_qrprof.so")
os.environ["ELMDDM_LIB"] = lib  # before the package import: _lib reads it at import time
from paper_2406_15959_b200 import build as B  # noqa: E402

B.build(force=True, extra=["-DELM_QR_PROF"], lib=lib)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = WL.config(k)
ctx = E.Context(E.Problem.from_config(c))
buf = ctx.alloc()
ctx.run(buf)
torch.cuda.synchronize()
L = E._lib.load()
L.elmddm_debug_qr_prof.argtypes = [C.c_void_p, C.c_int]
ctx.init_hidden(buf["W"], buf["b"])
ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
torch.cuda.synchronize()
L.elmddm_debug_qr_prof_reset()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
ev1.record()
torch.cuda.synchronize()
n = L.elmddm_debug_qr_prof(None, 0)
arr = np.zeros((n, 4), dtype=np.uint64)
L.elmddm_debug_qr_prof(arr.ctypes.data_as(C.c_void_p), n)
t0 = arr[:, 0].min()
st = (arr[:, 0] - t0).astype(np.float64) / 1e3
en = (arr[:, 1] - t0).astype(np.float64) / 1e3
sm = (arr[:, 2] & 0xFFFF).astype(int)
kind = ((arr[:, 2] >> 16) & 0xF).astype(int)
j0 = (arr[:, 3] >> 20).astype(int)
span = en.max()
nsm = sm.max() + 1
print(f"cfg{k}: local_factor {ev0.elapsed_time(ev1):.2f} ms (events); {n} CTAs on {nsm} SMs, span {span / 1e3:.2f} ms")
for kd, name in ((0, "panel"), (1, "trailing")):
    m = kind == kd
    d = en[m] - st[m]
    print(f"  {name}: {m.sum()} CTAs, CTA time {d.sum() / 1e3:.1f} SM-ms (/{nsm} = {d.sum() / 1e3 / nsm:.1f} ms), "
          f"per CTA median {np.median(d):.1f} us")
# per-SM occupancy over time on a 2 us grid
dt = 2.0
nt = int(span / dt) + 1
occ_p = np.zeros((nsm, nt), dtype=np.int16)
occ_w = np.zeros((nsm, nt), dtype=np.int16)
for i in range(n):
    a, b = int(st[i] / dt), int(en[i] / dt)
    (occ_p if kind[i] == 0 else occ_w)[sm[i], a:b + 1] += 1
states = {}
for pp in range(3):
    for ww in range(4):
        f = ((occ_p == pp) & (occ_w == ww)).mean()
        if f > 0.001:
            states[f"p{pp}w{ww}"] = round(float(f), 4)
print("  SM-time fraction by (panel CTAs, trailing CTAs) resident:", states)
# trailing-update CTA duration by company: mean occupancy of the other slot over the CTA's life
wm = np.where(kind == 1)[0]
comp_p = np.array([occ_p[sm[i], int(st[i] / dt):int(en[i] / dt) + 1].mean() for i in wm[::7]])
comp_w = np.array([occ_w[sm[i], int(st[i] / dt):int(en[i] / dt) + 1].mean() - 1 for i in wm[::7]])
dur = en[wm[::7]] - st[wm[::7]]
rows = arr[wm[::7], 3] >> 20
for lab, msk in (("beside a panel", comp_p > 0.5), ("beside a trailing CTA", (comp_p < 0.1) & (comp_w > 0.8)),
                 ("alone", (comp_p < 0.1) & (comp_w < 0.2))):
    if msk.sum():
        # normalise by rows (the CTA's work is proportional to ld - j0)
        ld = ctx.sizes["ld"]
        print(f"  trailing CTA {lab}: {msk.sum()} samples, us per 1000 rows median "
              f"{np.median(dur[msk] / (ld - rows[msk]) * 1000):.1f}")
# timeline: per 5% of the span, mean panel / trailing CTAs resident per SM
tl = []
for f in range(20):
    a, b = int(f * nt / 20), int((f + 1) * nt / 20)
    tl.append((round(float(occ_p[:, a:b].mean()), 2), round(float(occ_w[:, a:b].mean()), 2)))
print("  per 5% of span, (panel, trailing) CTAs per SM:", tl)
# panel chain per group: time from a panel's first CTA start to its last CTA end, by step
for jj in sorted(set(j0[kind == 0]))[:3] + sorted(set(j0[kind == 0]))[-2:]:
    m = (kind == 0) & (j0 == jj)
    print(f"  panel j0={jj}: {m.sum()} CTAs, first start {st[m].min():.0f} us, last end {en[m].max():.0f} us")
np.save(os.path.join(ROOT, "gpurun_out", f"qr_prof_cfg{k}.npy"), arr)
