"""Thin Python layer over the C ABI: one context per rank/device, torch tensors as device memory,
torch.distributed (NCCL) for the two exchange steps of Algorithm 1.

    rank r:  init_hidden -> assemble -> local_factor -> schur_accumulate        (own subdomains)
             gather(Pbuf, Sbuf slabs) to rank 0                                  (NCCL, NVLink)
    rank 0:  interface_solve  (eqn:schur)
             broadcast(status, u_Gamma)                                          (NCCL)
    rank r:  back_solve -> evaluate                                              (own subdomains)

The wrappers below do argument marshalling only; every arithmetic step runs in libelmddm.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):  # raw device pointer (a library-owned buffer, e.g. elmddm_dist_pool)
        return C.c_void_p(t)
    if not t.is_cuda:
        raise _lib.ElmddmError("elmddm arrays must be CUDA tensors")
    if t.dtype != torch.float64:
        raise _lib.ElmddmError("elmddm arrays must be float64")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def partition(N: int, world: int, rank: int):
    """Contiguous row-major slab of subdomains for `rank`: ceil(N/world) each.
    Every rank must own at least one subdomain: with slabs of ceil(N/world) that needs
    (world - 1) * ceil(N/world) < N (e.g. world <= N for the BASELINE configs' power-of-two
    counts); otherwise every rank raises the same error before any collective."""
    per = -(-N // world) if world >= 1 else 0
    if world < 1 or (world - 1) * per >= N:
        raise _lib.ElmddmError(f"{world} ranks for {N} subdomains in slabs of {per}: some rank would own no "
                               f"subdomain (need (world - 1) * ceil(N / world) < N, so world <= N at least)")
    s0 = min(N, rank * per)
    s1 = min(N, s0 + per)
    return s0, s1


@dataclass
class Problem:
    P: int
    M: int
    p: int
    q: int
    problem: int = 0
    seed: int = 0
    init_scheme: int = 0
    init_c: float = 0.125
    r_over_diam: float = 0.5
    interface_mode: int = 0             # factorisation order: 0 auto | 1, 2 strip (envelope) | 3 nested dissection
    interface_solver: str = "cholesky"  # "cholesky" (direct, reading R12) | "cg" (the paper's)
    cg_tol: float = 1e-9                # relative residual of the CG solver
    tikhonov: float = 0.0               # lambda of the damped local LS (reading R29; 0 = off; < 0 the
                                        # rule lambda_s = eps max(m, M) ||K^s||_F, reading R33)
    layout: int = 0                     # 0 face points (R1) | 1 the paper's lattice with cross points (R32)
    grf: object = None                  # problem 6: eqn:grf draws [n][4] (a, w_x, w_y, b)

    @classmethod
    def from_config(cls, c: dict) -> "Problem":
        keys = cls.__dataclass_fields__.keys()
        return cls(**{k: v for k, v in c.items() if k in keys})


class Context:
    """One elmddm context (one device, one subdomain range)."""

    def __init__(self, prob: Problem, s_begin: int = 0, s_end: int | None = None, device: int | None = None):
        L = _lib.load()
        self.L = L
        self.prob = prob
        N = prob.P * prob.P
        if s_end is None:
            s_end = N
        self.device = torch.cuda.current_device() if device is None else device
        if prob.interface_solver not in ("cholesky", "cg"):
            raise _lib.ElmddmError(f"unknown interface_solver {prob.interface_solver!r}")
        cfg = _lib.Config(prob.P, prob.M, prob.p, prob.q, prob.problem, prob.init_scheme, prob.init_c,
                          prob.r_over_diam, prob.seed, s_begin, s_end, prob.interface_mode, prob.layout,
                          prob.tikhonov)
        h = C.c_void_p()
        rc = L.elmddm_create(C.byref(cfg), self.device, C.byref(h))
        if rc != 0:
            raise _lib.ElmddmError(f"elmddm_create failed: {_lib.STATUS.get(rc, rc)} (config {prob}, "
                                   f"range [{s_begin},{s_end}))")
        self.h = h
        sz = _lib.Sizes()
        self._check(L.elmddm_sizes(h, C.byref(sz)), "elmddm_sizes")
        self.sizes = sz.as_dict()
        self.s_begin, self.s_end = s_begin, s_end
        if prob.problem == 6:
            if prob.grf is None:
                raise _lib.ElmddmError("problem 6 (variable coefficient) needs Problem.grf")
            self.set_coefficient(prob.grf)

    def set_coefficient(self, params):
        """Coefficient field of problem 6 (eqn:varpoisson): params [n][4] = (a_i, w_ix, w_iy, b_i)."""
        import numpy as np

        p = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 4)
        self._check(self.L.elmddm_set_coefficient(self.h, p.ctypes.data_as(C.c_void_p), int(p.shape[0])),
                    "elmddm_set_coefficient")

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.L.elmddm_destroy(h)
            self.h = None

    def _check(self, rc, what):
        if rc == _lib.WRANK:  # a warning: the call completed
            import warnings

            msg = self.L.elmddm_last_error(self.h)
            warnings.warn(f"{what}: {msg.decode() if msg else ''}", _lib.RankWarning, stacklevel=3)
        elif rc != 0:
            msg = self.L.elmddm_last_error(self.h)
            raise _lib.ElmddmError(f"{what}: {_lib.STATUS.get(rc, rc)}: {msg.decode() if msg else ''}")

    # ---- buffers ---------------------------------------------------------------------------
    def _slot_elems(self, key: str) -> int:
        """Doubles per subdomain slot of the global Schur buffers (include/elmddm.h sizes)."""
        N = self.prob.P * self.prob.P
        return self.sizes["pbuf_elems" if key == "Pbuf" else "sbuf_elems"] // N

    def _padded_slots(self, world: int | None = None) -> int:
        import torch.distributed as dist

        if world is None:
            world = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
        N = self.prob.P * self.prob.P
        return -(-N // world) * world

    def _gather_slots(self, t, key: str, world: int, rank: int, to_all: bool, group=None):
        """Exchange step of Algorithm 1: every subdomain slot of the global buffer has
        exactly ONE writer (its owner), so the exchange is a gather of the slabs -- no arithmetic,
        bit-identical for any rank count.  to_all: every rank receives every slab (all_gather,
        the multi-rank factorisation); else only rank 0 (gather, the rank-0 interface solve)."""
        import torch.distributed as dist

        N = self.prob.P * self.prob.P
        per = -(-N // world)
        slot = self._slot_elems(key)
        need = per * world * slot
        full = t if t.numel() >= need else torch.cat([t[: N * slot], t.new_zeros(need - N * slot)])
        chunks = list(full[:need].view(world, per * slot).unbind(0))
        nccl = dist.get_backend(group) == "nccl"
        mine = chunks[rank] if nccl else chunks[rank].clone()
        if to_all and nccl:  # in place: the input is this rank's slab of the output
            dist.all_gather_into_tensor(full[:need], mine, group=group)
        elif to_all:
            dist.all_gather(chunks, mine, group=group)
        else:
            dist.gather(mine, gather_list=chunks if rank == 0 else None, dst=0, group=group)
        if full is not t:
            t[: N * slot].copy_(full[: N * slot])

    def alloc(self) -> dict:
        z, M = self.sizes, self.prob.M
        dev = torch.device("cuda", self.device)
        f = dict(dtype=torch.float64, device=dev)
        S, q = z["S"], self.prob.q
        return {
            "W": torch.empty(S * M * 2, **f), "b": torch.empty(S * M, **f), "xi": torch.empty(S * M * 2, **f),
            "Kaug": torch.empty(z["kaug_elems"], **f), "At": torch.empty(z["at_elems"], **f),
            "tau": torch.empty(z["tau_elems"], **f), "work": torch.empty(max(z["work_elems"], 2), **f),
            # padded to whole slabs of ceil(N / world) slots so the multi-rank gather is one
            # equal-count collective (the padding slots stay zero and are never read)
            "Pbuf": torch.zeros(self._slot_elems("Pbuf") * self._padded_slots(), **f),
            "Sbuf": torch.zeros(self._slot_elems("Sbuf") * self._padded_slots(), **f),
            "Mband": torch.empty(max(z["band_elems"], 2), **f), "g": torch.empty(z["G_pad"], **f),
            "uG": torch.zeros(z["G_pad"], **f), "coef": torch.empty(S * M, **f), "resid": torch.empty(S, **f),
        }

    # ---- the C ABI, one wrapper per entry point ----------------------------------------------
    def init_hidden(self, W, b, xi=None, stream=None):
        self._check(self.L.elmddm_init_hidden(self.h, _ptr(W), _ptr(b), _ptr(xi), _stream(stream)), "init_hidden")

    def assemble(self, W, b, Kaug, At, stream=None):
        self._check(self.L.elmddm_assemble(self.h, _ptr(W), _ptr(b), _ptr(Kaug), _ptr(At), _stream(stream)),
                    "assemble")

    def local_factor(self, Kaug, tau, work, stream=None):
        self._check(self.L.elmddm_local_factor(self.h, _ptr(Kaug), _ptr(tau), _ptr(work), _stream(stream)),
                    "local_factor")

    def schur_accumulate(self, Kaug, At, Pbuf, Sbuf, work, stream=None):
        self._check(self.L.elmddm_schur_accumulate(self.h, _ptr(Kaug), _ptr(At), _ptr(Pbuf), _ptr(Sbuf), _ptr(work),
                                                   _stream(stream)), "schur_accumulate")

    def interface_assemble(self, Pbuf, Sbuf, Mband, g, work, stream=None):
        self._check(self.L.elmddm_interface_assemble(self.h, _ptr(Pbuf), _ptr(Sbuf), _ptr(Mband), _ptr(g), _ptr(work),
                                                     _stream(stream)), "interface_assemble")

    def interface_factor_solve(self, Mband, g, uG, work, stream=None):
        self._check(self.L.elmddm_interface_factor_solve(self.h, _ptr(Mband), _ptr(g), _ptr(uG), _ptr(work),
                                                         _stream(stream)), "interface_factor_solve")

    def interface_cg(self, Mband, g, uG, work, tol=1e-9, maxit=100000, stream=None):
        """The paper's CG interface solver; returns (iterations, relative residual)."""
        it = C.c_int32()
        rr = C.c_double()
        self._check(self.L.elmddm_interface_cg(self.h, _ptr(Mband), _ptr(g), _ptr(uG), _ptr(work), float(tol), int(maxit),
                                               C.byref(it), C.byref(rr), _stream(stream)), "interface_cg")
        return int(it.value), float(rr.value)

    def interface_solve(self, Pbuf, Sbuf, Mband, g, uG, work, stream=None):
        self._check(self.L.elmddm_interface_solve(self.h, _ptr(Pbuf), _ptr(Sbuf), _ptr(Mband), _ptr(g), _ptr(uG),
                                                  _ptr(work), _stream(stream)), "interface_solve")

    def back_solve(self, Kaug, uG, coef, resid, work, stream=None):
        self._check(self.L.elmddm_back_solve(self.h, _ptr(Kaug), _ptr(uG), _ptr(coef), _ptr(resid), _ptr(work),
                                             _stream(stream)), "back_solve")

    def evaluate(self, W, b, coef, xy, u, stream=None):
        n = xy.numel() // 2
        self._check(self.L.elmddm_evaluate(self.h, _ptr(W), _ptr(b), _ptr(coef), _ptr(xy), n, _ptr(u),
                                           _stream(stream)), "evaluate")

    def sync(self, stream=None):
        self._check(self.L.elmddm_sync(self.h, _stream(stream)), "sync")

    def interface_points(self):
        import numpy as np

        xy = np.zeros((self.sizes["G"], 2))
        self._check(self.L.elmddm_interface_points(self.h, xy.ctypes.data_as(C.c_void_p)), "interface_points")
        return xy

    def set_timing(self, enable: bool):
        self._check(self.L.elmddm_set_timing(self.h, 1 if enable else 0), "set_timing")
        self._timing = bool(enable)

    def timing(self, reset: bool = True) -> dict:
        t = _lib.Timing()
        self._check(self.L.elmddm_timing(self.h, C.byref(t), 1 if reset else 0), "timing")
        return {"launches": int(t.launches),
                "count": {k: int(t.count[i]) for i, k in enumerate(_lib.KCLASSES)},
                "ms": {k: float(t.ms[i]) for i, k in enumerate(_lib.KCLASSES)}}

    def debug_dist_emulate(self, nrep, Mband, g, uG, work, stream=None) -> int:
        """One-GPU emulation of the multi-rank factorisation (elmddm_debug_dist_emulate); returns
        the number of doubles in which the replicas' factors differ (0 expected)."""
        nd = C.c_int64()
        self._check(self.L.elmddm_debug_dist_emulate(self.h, nrep, _ptr(Mband), _ptr(g), _ptr(uG), _ptr(work),
                                                       C.byref(nd), _stream(stream)), "elmddm_debug_dist_emulate")
        return nd.value

    def chol_plan(self):
        """(newidx[G], tile_map[chol_blocks, chol_blocks], tasks[chol_tasks, 4]) of the interface
        factorisation (host arrays): the factorisation-order index of every interface unknown,
        the tile id of every tile (I, J) of L (-1 outside its structure) and the task list
        (I, J, kind, updates; kind 1 = pre-aggregation of a split task, 2 = its rest)."""
        import numpy as np

        z = self.sizes
        nb = z["chol_blocks"]
        newidx = np.zeros(max(z["G"], 1), dtype=np.int32)
        tmap = np.zeros(nb * nb, dtype=np.int32)
        tasks = np.zeros((z["chol_tasks"], 4), dtype=np.int32)
        self._check(self.L.elmddm_chol_plan(self.h, newidx.ctypes.data_as(C.c_void_p), tmap.ctypes.data_as(C.c_void_p),
                                            tasks.ctypes.data_as(C.c_void_p)), "chol_plan")
        return newidx[: z["G"]], tmap.reshape(nb, nb), tasks

    def band_index(self, i, j):
        return int(self.L.elmddm_band_index(self.h, i, j))

    # ---- Algorithm 1 -------------------------------------------------------------------------
    # ---- multi-rank interface factorisation (include/elmddm.h elmddm_dist_*) ----
    def _dist_export(self):
        h = (C.c_uint8 * 64)()
        rc = self.L.elmddm_dist_export(self.h, C.cast(h, C.c_void_p))
        return bytes(h) if rc == 0 else None

    def _dist_import(self, rank, world, handles):
        blob = b"".join(handles)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self._dist_imported = self.L.elmddm_dist_import(self.h, rank, world, C.cast(buf, C.c_void_p)) == 0
        return self._dist_imported

    def _dist_handshake(self, phase):
        ok = C.c_int32(0)
        return self.L.elmddm_dist_handshake(self.h, phase, C.byref(ok)) == 0 and ok.value == 1

    def _dist_disable(self):
        self.L.elmddm_dist_import(self.h, 0, 1, None)

    def _dist_pool(self):
        p = C.c_void_p()
        self._check(self.L.elmddm_dist_pool(self.h, C.byref(p)), "elmddm_dist_pool")
        return int(p.value)

    def dist_setup(self, group=None) -> bool:
        """Collectively switch this context to the multi-rank interface factorisation: every
        rank exports its replica region, the CUDA IPC handles are all-gathered, every rank opens
        the others'.  All ranks agree on the outcome; on any failure (or unless
        ELMDDM_DIST_IFACE=1: opt-in, it has not yet run on several GPUs; or the CG solver) every
        rank keeps the rank-0 path.  Returns whether it is active."""
        import os

        import torch.distributed as dist

        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        # opt-in until the peer-memory path has run on several GPUs (this environment offers one)
        want = os.environ.get("ELMDDM_DIST_IFACE", "0") == "1" and self.prob.interface_solver == "cholesky"
        want = want and self.prob.layout == 0
        want = want and self.sizes["G"] > 0

        def agree(flag: bool) -> bool:
            t = torch.tensor([1 if flag else 0], dtype=torch.int32,
                             device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            return bool(t.item())

        self._dist_imported = False
        if not agree(want):
            return False
        h = self._dist_export()
        hs = [None] * world
        dist.all_gather_object(hs, h, group=group)
        if not agree(all(x is not None for x in hs)):
            return False
        ok = self._dist_import(rank, world, hs)
        if ok:  # peer stores and atomics really work before the factorisation relies on them
            ok = self._dist_handshake(0)
            dist.barrier(group=group)
            ok = self._dist_handshake(1) and ok
        else:
            dist.barrier(group=group)
        if not agree(ok):
            if ok or self._dist_imported:
                self._dist_disable()
            return False
        self._dist_pool_ptr = self._dist_pool()
        return True

    def _fence(self, device, group=None):
        import torch.distributed as dist

        dist.all_reduce(torch.zeros(1, dtype=torch.int32, device=device), group=group)

    def enqueue(self, buf: dict, xy=None, u=None, stream=None):
        """One rank's whole hot path (H1-H9 of Algorithm 1) enqueued on `stream` with no
        host synchronisation -- so it can be captured once in a CUDA graph (capture_graph) and
        replayed.  Single rank, direct interface solve only: the CG solver checks convergence on
        the host and the multi-rank path exchanges through NCCL between phases.  Device-side
        errors surface at the next sync()."""
        if self.prob.interface_solver != "cholesky":
            raise _lib.ElmddmError("enqueue / capture_graph: only the direct interface solver runs without host syncs")
        N = self.prob.P * self.prob.P
        if (self.s_begin, self.s_end) != (0, N):
            raise _lib.ElmddmError(f"enqueue / capture_graph: one rank owning every subdomain (this context owns "
                                   f"[{self.s_begin}, {self.s_end}) of {N}); the multi-rank path is run()")
        self.init_hidden(buf["W"], buf["b"], None, stream)
        self.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"], stream)
        self.local_factor(buf["Kaug"], buf["tau"], buf["work"], stream)
        self.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"], stream)
        if self.sizes["G"] > 0:
            self.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"], stream)
            self.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"], stream)
        self.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"], stream)
        if xy is not None:
            self.evaluate(buf["W"], buf["b"], buf["coef"], xy, u, stream)

    def capture_graph(self, buf: dict, xy=None, u=None):
        """Capture enqueue() once into a torch.cuda.CUDAGraph; graph.replay() then re-runs the whole
        solve on the same buffers with one launch from the host (follow it with sync() to read
        the device status).  One eager pass first creates the library's internal streams and its
        per-context launch state, so nothing is allocated while capturing."""
        if getattr(self, "_timing", False):
            raise _lib.ElmddmError("capture_graph: per-kernel timing (set_timing) records host-read events; turn it off")
        self.enqueue(buf, xy, u)  # (raises for the CG solver before any capture starts)
        self.sync()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=buf["W"].device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            self.enqueue(buf, xy, u, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        return g

    def run(self, buf: dict, xy=None, u=None, group=None, stream=None, timer=None):
        """One pass of the hot path on this rank (Algorithm 1).  With a process group of
        size > 1 the Schur contributions of every slab are gathered to rank 0 (one NCCL gather, no
        arithmetic: every slot has one writer), rank 0 solves the interface system and u_Gamma is
        broadcast back -- or, opt-in (ELMDDM_DIST_IFACE=1, see dist_setup), every rank receives
        every slab and all ranks factor the interface system together.  Errors: every rank
        synchronises at the end and raises its own device status (non-finite QR, ...); a failed
        rank-0 interface solve is broadcast as a status word, so every rank raises instead of
        waiting in a collective."""
        import torch.distributed as dist

        world = dist.get_world_size(group) if (group is not None or (dist.is_available() and dist.is_initialized())) else 1
        rank = dist.get_rank(group) if world > 1 else 0
        if world > 1 and getattr(self, "_dist", None) is None:
            self._dist = self.dist_setup(group)
        dmode = world > 1 and bool(getattr(self, "_dist", False))
        mark = timer.mark if timer is not None else (lambda name: None)
        self.init_hidden(buf["W"], buf["b"], None, stream)
        mark("init_hidden")
        self.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"], stream)
        mark("assemble")
        self.local_factor(buf["Kaug"], buf["tau"], buf["work"], stream)
        mark("local_factor")
        self.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"], stream)
        mark("schur_accumulate")
        if world > 1:
            self._gather_slots(buf["Pbuf"], "Pbuf", world, rank, dmode, group)
            self._gather_slots(buf["Sbuf"], "Sbuf", world, rank, dmode, group)
            mark("reduce")
        err = None
        failed = None
        if self.sizes["G"] > 0 and dmode:
            pool = self._dist_pool_ptr
            self.interface_assemble(buf["Pbuf"], buf["Sbuf"], pool, buf["g"], buf["work"], stream)
            # device-side fence: no rank's factorisation kernel may push a finished tile into a
            # peer's replica before that peer has assembled M into it (an all-reduce completes on
            # every rank only after every rank reached it on its stream)
            self._fence(buf["g"].device, group)
            mark("interface_assemble")
            self.interface_factor_solve(pool, buf["g"], buf["uG"], buf["work"], stream)
            mark("interface_factor_solve")
        elif self.sizes["G"] > 0:
            if rank == 0:
                try:
                    self.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"], stream)
                    mark("interface_assemble")
                    if self.prob.interface_solver == "cg":
                        self.cg_info = self.interface_cg(buf["Mband"], buf["g"], buf["uG"], buf["work"],
                                                         self.prob.cg_tol, stream=stream)
                    else:
                        self.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"], stream)
                    if world > 1:  # the outcome must be known before it is broadcast
                        self.sync(stream)
                    mark("interface_factor_solve")
                except _lib.ElmddmError as ex:
                    err = ex
            if world > 1:
                failed = torch.tensor([0 if err is None else 1], dtype=torch.int32, device=buf["g"].device
                                      if dist.get_backend(group) == "nccl" else "cpu")
                dist.broadcast(failed, src=0, group=group)
                dist.broadcast(buf["uG"], src=0, group=group)
                mark("broadcast")
        self.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"], stream)
        mark("back_solve")
        if xy is not None:
            if world > 1:
                u.zero_()
            self.evaluate(buf["W"], buf["b"], buf["coef"], xy, u, stream)
            if world > 1:
                dist.reduce(u, dst=0, group=group)
            mark("evaluate")
        if err is not None:
            raise err
        self.sync(stream)  # this rank's device status: non-finite QR, pivots, rank warnings
        if failed is not None and int(failed.item()) != 0:
            raise _lib.ElmddmError("the rank-0 interface solve failed (see rank 0's error)")
        return buf


def solve(prob: Problem, xy_host=None, device: int | None = None, group=None, return_all: bool = False):
    """Public one-call API: solve the configured DDM-ELM problem and return host results.

    xy_host: optional (n, 2) host array/tensor of evaluation points.  Returns a dict with
    u (on rank 0), uG, coef, resid (own subdomains) as host tensors."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    N = prob.P * prob.P
    s0, s1 = partition(N, world, rank)
    ctx = Context(prob, s0, s1, device)
    buf = ctx.alloc()
    dev = buf["W"].device
    xy = u = None
    if xy_host is not None:
        xy_t = torch.as_tensor(xy_host, dtype=torch.float64).reshape(-1)
        xy = xy_t.to(dev, non_blocking=True)
        u = torch.zeros(xy.numel() // 2, dtype=torch.float64, device=dev)
    ctx.run(buf, xy, u, group)
    out = {"uG": buf["uG"][: ctx.sizes["G"]].cpu(), "coef": buf["coef"].view(-1, prob.M).cpu(),
           "resid": buf["resid"].cpu(), "range": (s0, s1)}
    if u is not None:
        out["u"] = u.cpu()
    if return_all:
        out["ctx"], out["buf"] = ctx, buf
    return out


def plan_query(P: int, q: int, ordering: int = 1, workers: int = 0, arrays: bool = True) -> dict:
    """Host-only interface-factorisation plan (elmddm_plan_query; no GPU needed): stats and,
    with arrays=True, the renumbering, tile map and task list."""
    import numpy as np

    L = _lib.load()
    st = np.zeros(6, dtype=np.int64)
    vp = C.c_void_p
    rc = L.elmddm_plan_query(P, q, ordering, workers, st.ctypes.data_as(vp), None, None, None)
    if rc != 0:
        raise _lib.ElmddmError(f"elmddm_plan_query failed: {_lib.STATUS.get(rc, rc)}")
    out = {"n": int(st[0]), "nblk": int(st[1]), "ntiles": int(st[2]), "nupd": int(st[3]), "ntasks": int(st[4]),
           "sim_ms": st[5] * 1e-6}
    if arrays:
        G = 2 * P * (P - 1) * q
        nb = out["nblk"]
        newidx = np.zeros(G, dtype=np.int32)
        tmap = np.zeros(nb * nb, dtype=np.int32)
        tasks = np.zeros((out["ntasks"], 4), dtype=np.int32)
        rc = L.elmddm_plan_query(P, q, ordering, workers, st.ctypes.data_as(vp), newidx.ctypes.data_as(vp),
                                 tmap.ctypes.data_as(vp), tasks.ctypes.data_as(vp))
        if rc != 0:
            raise _lib.ElmddmError(f"elmddm_plan_query failed: {_lib.STATUS.get(rc, rc)}")
        out.update(newidx=newidx, tile_map=tmap.reshape(nb, nb), tasks=tasks)
    return out


def dmma_peak_tflops(device: int = 0, ms: float = 200.0) -> float:
    """Measured sustained FP64 tensor (DMMA) throughput of `device` (diagnostic)."""
    L = _lib.load()
    out = C.c_double()
    rc = L.elmddm_dmma_probe(device, ms, C.byref(out))
    if rc != 0:
        raise _lib.ElmddmError(f"elmddm_dmma_probe: {_lib.STATUS.get(rc, rc)}")
    return float(out.value)
