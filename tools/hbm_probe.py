"""Write-only and copy HBM bandwidth on this GPU (torch kernels; CUDA events, best of 10):
the ceiling for the write-bound assembly kernel (k_assemble writes, reads almost nothing)."""
import json

import torch

n = 2 * 1024**3  # doubles: 16 GiB
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n // 2, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


t_fill = best(lambda: x.fill_(1.0))
t_zero = best(lambda: x.zero_())
t_copy = best(lambda: x[: n // 2].copy_(y))
print(json.dumps({"write_fill_GBps": n * 8 / t_fill / 1e6, "write_zero_GBps": n * 8 / t_zero / 1e6,
                  "copy_rw_GBps": 2 * (n // 2) * 8 / t_copy / 1e6, "bytes": n * 8}))
