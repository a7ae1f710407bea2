"""The CUDA IPC exchange of the multi-rank interface factorisation for real (GPU): two processes
on cuda:0 (gloo for the host collectives) export their replica regions, open each other's with
cudaIpcOpenMemHandle, and pass the handshake (system-scope peer stores and atomics).  No
factorisation kernel runs across the processes (kernels that wait on each other must not share
a GPU between processes); the factorisation protocol itself is tested by the one-kernel
emulation in test_gpu_parity.py."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ELMDDM_DIST_IFACE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_15959_b200 as E
        import workloads as WL

        ctx = E.Context(E.Problem.from_config(WL.config(1)))
        ok = ctx.dist_setup()
        pool = ctx._dist_pool_ptr if ok else 0
        ctx._dist_disable()
        q.put((rank, ok, pool != 0))
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, repr(ex), False))
    finally:
        dist.destroy_process_group()


def test_ipc_export_import_handshake_two_processes():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
    assert res[0] == (True, True) and res[1] == (True, True), res
