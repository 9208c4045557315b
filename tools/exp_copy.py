"""Host<->device copy costs for a 10K x 128 f32 query batch (dev tool)."""
import time
import numpy as np
import torch

q = np.random.default_rng(0).standard_normal((10_000, 128)).astype(np.float32)
pin = torch.empty(q.shape, dtype=torch.float32).pin_memory()
dev = torch.empty(q.shape, dtype=torch.float32, device="cuda")


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    return np.median(ts) * 1e3


print("np.copyto -> pinned      %.3f ms" % t(lambda: np.copyto(pin.numpy(), q)))
print("pinned H2D               %.3f ms" % t(lambda: dev.copy_(pin, non_blocking=True)))
qt = torch.from_numpy(q)
print("pageable H2D (torch)     %.3f ms" % t(lambda: dev.copy_(qt)))
print("pageable H2D nonblocking %.3f ms" % t(lambda: dev.copy_(qt, non_blocking=True)))
print("copyto + pinned H2D      %.3f ms" % t(lambda: (np.copyto(pin.numpy(), q), dev.copy_(pin, non_blocking=True))))
import os
print("cpus", os.cpu_count(), open("/proc/cpuinfo").read().count("processor"))
