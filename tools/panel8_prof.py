"""Phase breakdown of the 8-CTA cluster panel kernel (profiling build with -DELM_PANEL_PROF).
usage: python tools/panel8_prof.py [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.path.join(ROOT, "paper_2406_15959_b200", "libelmddm_pprof.so")
os.environ["ELMDDM_LIB"] = lib
os.environ["ELMDDM_PANEL8"] = "1"
from paper_2406_15959_b200 import build as B  # noqa: E402

B.build(force=True, extra=["-DELM_PANEL_PROF"], lib=lib)
import torch  # noqa: E402

import paper_2406_15959_b200 as E  # noqa: E402
import workloads as WL  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = E.Context(E.Problem.from_config(WL.config(k)))
buf = ctx.alloc()
ctx.init_hidden(buf["W"], buf["b"])
ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
torch.cuda.synchronize()
