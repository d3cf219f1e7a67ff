"""Host<->device transfer options for one 7.4 MB fp64 vector (config-1 psi size)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 921600
a = np.random.rand(n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
pool = ThreadPoolExecutor(8)


def timeit(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:40s} {dt*1e3:7.3f} ms  {n*8/dt/1e9:6.1f} GB/s", flush=True)


timeit("numpy copy (memcpy)", lambda: np.copy(a))
timeit("copy into pinned", lambda: pin.numpy().__setitem__(slice(None), a))
def par():
    pn = pin.numpy()
    list(pool.map(lambda lo: pn.__setitem__(slice(lo, lo + 65536), a[lo:lo + 65536]), range(0, n, 65536)))
timeit("threaded copy into pinned (8)", par)
timeit("H2D from pinned", lambda: dev.copy_(pin, non_blocking=True))
timeit("H2D from pageable (torch)", lambda: dev.copy_(torch.from_numpy(a), non_blocking=False))
timeit("D2H into pinned", lambda: pin.copy_(dev, non_blocking=True))
timeit("D2H pageable (.cpu())", lambda: dev.cpu())
out = torch.empty(n, dtype=torch.float64)
timeit("D2H into preallocated pageable", lambda: out.copy_(dev))
import os
print("cpus", os.cpu_count())
