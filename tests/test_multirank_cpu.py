"""World-size-2/3 `gloo` tests (CPU) of the multi-rank plumbing of Context.run:
partition, zero-filled globally indexed Schur buffers summed by reduce(SUM) = exact union,
rank-0 interface solve, broadcast of u_Gamma, reduce of the slab-wise evaluation -- and the
multi-rank interface factorisation mode (dist_setup's collective agreement on the CUDA IPC
exchange; all-reduce of the buffers; every rank factors and solves; no broadcast), including the
collective fallback when one rank cannot export its region.

The CUDA kernels are replaced by a fake context whose calls write slab-tagged values, so the
test checks exactly the host-side collective sequence the GPU path uses."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_SUB = 9          # 3 x 3 subdomains
SLOT = 5           # doubles per Pbuf / Sbuf slot
G = 4
NPTS = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_ctx(rank, world, mode="off"):
    from paper_2406_15959_b200 import solver as S

    s0, s1 = S.partition(N_SUB, world, rank)

    class Fake(S.Context):
        def __init__(self):  # no CUDA context
            self.prob = S.Problem(P=3, M=8, p=3, q=2)   # N_SUB = 9 subdomains
            self.sizes = {"G": G, "pbuf_elems": N_SUB * SLOT, "sbuf_elems": N_SUB * SLOT}
            self.s_begin, self.s_end = s0, s1
            self.calls = []

        def __del__(self):
            pass

        # CUDA IPC hooks of dist_setup (the collective logic around them is the real one)
        def _dist_export(self):
            self.calls.append("dist_export")
            return None if (mode == "fail1" and rank == 1) else bytes([rank]) * 64

        def _dist_import(self, r, w, handles):
            self.calls.append("dist_import")
            assert r == rank and w == world and [h[0] for h in handles] == list(range(world))
            self._dist_imported = True
            return True

        def _dist_handshake(self, phase):
            self.calls.append(f"dist_handshake{phase}")
            return not (mode == "hs_fail2" and rank == 2 and phase == 1)

        def _dist_disable(self):
            self.calls.append("dist_disable")

        def _dist_pool(self):
            return 0

        def init_hidden(self, W, b, xi=None, stream=None):
            self.calls.append("init_hidden")

        def assemble(self, *a, **k):
            self.calls.append("assemble")

        def local_factor(self, *a, **k):
            self.calls.append("local_factor")

        def schur_accumulate(self, Kaug, At, Pbuf, Sbuf, work, stream=None):
            self.calls.append("schur_accumulate")
            for s in range(s0, s1):  # only own (global) slots are written
                Pbuf[s * SLOT:(s + 1) * SLOT] = float(s + 1)
                Sbuf[s * SLOT:(s + 1) * SLOT] = 0.5 * (s + 1)

        def interface_assemble(self, Pbuf, Sbuf, Mband, g, work, stream=None):
            self.calls.append("interface_assemble")
            g[:] = Pbuf.sum() + Sbuf.sum()

        def interface_factor_solve(self, Mband, g, uG, work, stream=None):
            self.calls.append("interface_factor_solve")
            if mode == "pivot_fail":
                raise S._lib.ElmddmError("interface_factor_solve: ELMDDM_ENUMERIC: non-positive pivot")
            uG[:] = g

        def sync(self, stream=None):
            self.calls.append("sync")

        def _fence(self, device, group=None):
            self.calls.append("fence")
            super()._fence(device, group)

        def back_solve(self, Kaug, uG, coef, resid, work, stream=None):
            self.calls.append("back_solve")
            coef[:] = uG[0]

        def evaluate(self, W, b, coef, xy, u, stream=None):
            self.calls.append("evaluate")
            for t in range(NPTS):  # point t "owned" by subdomain t % N_SUB
                if s0 <= t % N_SUB < s1:
                    u[t] = coef[0] + t

    return Fake()


def S_err():
    from paper_2406_15959_b200 import _lib

    return _lib.ElmddmError


def _worker(rank, world, port, q, mode="off"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ["ELMDDM_DIST_IFACE"] = "1" if mode in ("on", "fail1", "hs_fail2") else "0"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode == "too_many":
            from paper_2406_15959_b200 import solver as S

            try:
                S.partition(2, world, rank)
            except S._lib.ElmddmError as ex:
                q.put((rank, "raised", str(ex), None, None, None))
            return
        ctx = _fake_ctx(rank, world, mode)
        f64 = dict(dtype=torch.float64)
        buf = {"W": torch.zeros(1, **f64), "b": torch.zeros(1, **f64), "Kaug": torch.zeros(1, **f64),
               "At": torch.zeros(1, **f64), "tau": torch.zeros(1, **f64), "work": torch.zeros(1, **f64),
               "Pbuf": torch.full((N_SUB * SLOT,), -7.0, **f64), "Sbuf": torch.full((N_SUB * SLOT,), -7.0, **f64),
               "Mband": torch.zeros(1, **f64), "g": torch.zeros(G, **f64), "uG": torch.zeros(G, **f64),
               "coef": torch.zeros(3, **f64), "resid": torch.zeros(1, **f64)}
        xy = torch.zeros(2 * NPTS, **f64)
        u = torch.full((NPTS,), -1.0, **f64)
        try:
            ctx.run(buf, xy, u)
        except S_err() as ex:
            q.put((rank, ctx.calls, "raised", str(ex), None, None))
            return
        q.put((rank, ctx.calls, buf["Pbuf"].tolist(), buf["uG"].tolist(), buf["coef"].tolist(), u.tolist()))
    finally:
        dist.destroy_process_group()


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_dist_interface_mode_gloo(world):
    """Multi-rank factorisation mode: every rank sees the full union of the Schur buffers
    (all-reduce), assembles and factors, and ends with the same u_Gamma without a broadcast."""
    res = _run(world, "on")
    expect_P = [float(s + 1) for s in range(N_SUB) for _ in range(SLOT)]
    g_expect = sum(expect_P) + 0.5 * sum(expect_P)
    for r in range(world):
        calls, P, uG, coef, u = res[r]
        assert calls[:4] == ["dist_export", "dist_import", "dist_handshake0", "dist_handshake1"]
        assert "interface_assemble" in calls and "interface_factor_solve" in calls
        # the cross-rank fence sits between the assembly into the replica and the factorisation
        ia, fe, fs = calls.index("interface_assemble"), calls.index("fence"), calls.index("interface_factor_solve")
        assert ia < fe < fs
        assert calls[-1] == "sync"
        assert P == expect_P and uG == [g_expect] * G and coef == [g_expect] * 3
    assert res[0][4] == [g_expect + t for t in range(NPTS)]


@pytest.mark.parametrize("mode", ["fail1", "hs_fail2"])
def test_dist_interface_collective_fallback_gloo(mode):
    """One rank cannot export its region (no rank imports), or one rank's IPC handshake fails
    (every rank disables the imported peers): all keep the rank-0 path."""
    res = _run(3, mode)
    expect_P = [float(s + 1) for s in range(N_SUB) for _ in range(SLOT)]
    g_expect = sum(expect_P) + 0.5 * sum(expect_P)
    for r in range(3):
        calls, P, uG, coef, u = res[r]
        assert ("dist_import" in calls) == (mode == "hs_fail2")
        assert ("dist_disable" in calls) == (mode == "hs_fail2")
        assert ("interface_factor_solve" in calls) == (r == 0)
        assert uG == [g_expect] * G


@pytest.mark.parametrize("world", [2, 3])
def test_collective_sequence_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect_P = [float(s + 1) for s in range(N_SUB) for _ in range(SLOT)]
    calls0, P0, uG0, coef0, u0 = res[0]
    assert P0 == expect_P                                   # exact union on rank 0
    g_expect = sum(expect_P) + 0.5 * sum(expect_P)
    assert uG0 == [g_expect] * G
    assert "interface_factor_solve" in calls0
    for r in range(1, world):
        calls, P, uG, coef, u = res[r]
        assert "interface_assemble" not in calls and "interface_factor_solve" not in calls
        assert uG == uG0                                    # broadcast
        assert coef == [g_expect] * 3
    assert u0 == [g_expect + t for t in range(NPTS)]        # slab-wise evaluation summed


def test_default_is_the_rank0_path_gloo():
    """ELMDDM_DIST_IFACE unset: the multi-rank factorisation is opt-in (it has not yet run on
    several GPUs); the rank-0 path runs and no IPC region is exported."""
    res = _run(2, "default")
    for r in range(2):
        calls = res[r][0]
        assert "dist_export" not in calls
        assert ("interface_factor_solve" in calls) == (r == 0)
        assert calls[-1] == "sync"          # every rank reports its own device status


def test_rank0_interface_failure_raises_on_every_rank_gloo():
    """A non-positive pivot on rank 0 is broadcast as a status word: every rank raises, none
    waits forever in the broadcast of u_Gamma."""
    res = _run(3, "pivot_fail")
    for r in range(3):
        calls, tag, msg = res[r][0], res[r][1], res[r][2]
        assert tag == "raised"
        assert ("non-positive pivot" in msg) if r == 0 else ("rank-0 interface solve failed" in msg)


def test_more_ranks_than_subdomains_raise_everywhere_gloo():
    res = _run(3, "too_many")
    assert all(res[r][0] == "raised" and "world <= N" in res[r][1] for r in range(3))
