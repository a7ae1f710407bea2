"""Full oracle solve of a BASELINE config, cached for the GPU parity tests at configs 3-4.

Calls only oracle/ (the plain-C fp64 CPU oracle) and workloads.py (the seeded input recipe):
no value here comes from the CUDA path.  Writes
  tests/golden/oracle_cfg<k>.npz   uG (strip order, reading R14), u on the 101^2 grid (R15),
                                   resid r_s (R17), the per-phase times and the thread count
  profiles/r02_oracle_cfg<k>.json  the oracle's time-to-solution per phase on this host
usage: python tools/oracle_cache.py K [--threads T] [--no-write]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import workloads as WL  # noqa: E402


def ocfg(c):
    return O.cfg(c["P"], c["M"], c["p"], c["q"], c["problem"], c.get("init_scheme", 0), c.get("init_c", 0.125),
                 c.get("r_over_diam", 0.5), c["seed"], c.get("tikhonov", 0.0), c.get("layout", 0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("k", type=int)
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--no-write", action="store_true")
    ap.add_argument("--tag", default="r02")
    a = ap.parse_args()
    c = WL.config(a.k)
    oc = ocfg(c)
    xy = WL.eval_grid()
    t0 = time.time()
    W, b, _, _ = O.init_hidden(oc)
    t_init = time.time() - t0
    t0 = time.time()
    r = O.solve(oc, W, b, xy, nthreads=a.threads)
    wall = time.time() - t0
    ue = WL.exact(c["problem"], xy)
    err = float(np.linalg.norm(r["u"] - ue) / np.linalg.norm(ue))
    times = dict(r["times"], init_hidden=t_init)
    rec = {"config": a.k, "workload": c["name"], "threads": a.threads, "host": platform.node(),
           "cpu": platform.processor() or platform.machine(), "wall_s": wall + t_init, "times_s": times,
           "G": int(len(r["uG"])), "N": int(len(r["resid"])), "rel_l2_vs_exact": err,
           "interface": "banded Cholesky in strip order (oracle.c orc_band_cholesky)" if len(r["uG"]) > 20000
           else "dense Cholesky (oracle.c orc_cholesky)"}
    print(json.dumps(rec))
    if not a.no_write:
        np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"oracle_cfg{a.k}.npz"), uG=r["uG"], u=r["u"],
                            resid=r["resid"], threads=a.threads, wall_s=wall + t_init,
                            times=np.array([times[k] for k in ("local", "iface_assemble", "iface_solve", "back",
                                                               "eval")]))
        json.dump(rec, open(os.path.join(ROOT, "profiles", f"{a.tag}_oracle_cfg{a.k}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
