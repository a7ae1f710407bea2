"""Timeline of the interface triangular solves (profiling build with -DELM_CHOL_PROF).
usage: python tools/trsv_prof.py [config]   (on a GPU box; ELMDDM_TRSV_CHUNK as in the product)"""
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

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = WL.config(k)
ctx = E.Context(E.Problem.from_config(c))
buf = ctx.alloc()
ctx.run(buf)
torch.cuda.synchronize()
ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
torch.cuda.synchronize()
L = E._lib.load()
L.elmddm_debug_trsv_tasks.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L.elmddm_debug_trsv_prof.argtypes = [C.c_void_p, C.c_int, C.c_int]
for d in (0, 1):
    n = L.elmddm_debug_trsv_tasks(ctx.h, d, None)
    tk = np.zeros((n, 4), dtype=np.int32)
    L.elmddm_debug_trsv_tasks(ctx.h, d, tk.ctypes.data_as(C.c_void_p))
    arr = np.zeros(n * 4, dtype=np.uint64)
    L.elmddm_debug_trsv_prof(arr.ctypes.data_as(C.c_void_p), d, n)
    a = arr.reshape(n, 4).astype(np.float64)
    t0 = a[:, 0].min()
    st, en, fw, cta = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2] / 1e3, a[:, 3]
    ntile = tk[:, 2] - tk[:, 1]
    ncta = int(cta.max()) + 1
    span = en.max()
    busy = (en - st).sum()
    print(f"dir {d}: {n} tasks ({(tk[:, 3] >= 0).sum()} partial), {ntile.sum()} tiles on {ncta} CTAs, span {span:.0f} us")
    print(f"  task time {busy / ncta:.0f} us/CTA ({100 * busy / ncta / span:.0f}% of span), flag waits {fw.sum() / ncta:.0f} us/CTA")
    per = (en - st - fw) / np.maximum(ntile + 1, 1)
    print(f"  non-wait time per tile: median {np.median(per):.2f} us, mean {per.mean():.2f} us")
    o = np.argsort(st)
    for f in (0.25, 0.5, 0.75, 0.9, 0.95, 0.99, 1.0):
        idx = o[min(n - 1, int(f * (n - 1)))]
        print(f"  task #{idx} ({100 * f:.0f}% by start): start {st[idx]:.0f} end {en[idx]:.0f} tiles {ntile[idx]} wait {fw[idx]:.0f}")
    last = np.argsort(en)[-12:]
    print("  last-ending tasks (row, tiles, start, end, wait):",
          [(int(tk[i, 0]), int(ntile[i]), round(st[i]), round(en[i]), round(fw[i])) for i in last])
    # how many tasks were running over time
    ts = np.linspace(0, span, 21)
    print("  running tasks at 0..100% of span:", [int(((st <= t) & (en > t)).sum()) for t in ts])
