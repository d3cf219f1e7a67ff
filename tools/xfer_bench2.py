"""Host<->device transfer strategies for one config-1 vector (7.4 MB fp64)
from / into NumPy arrays (the reference-facing API's I/O)."""
import ctypes
import os
import time

import numpy as np
import torch

n = 921600
a = np.random.rand(n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
CH = 4
pins = [torch.empty(n // CH + 1, dtype=torch.float64, pin_memory=True) for _ in range(2)]
s_copy = torch.cuda.Stream()
cudart = torch.cuda.cudart()


def timeit(name, fn, reps=30):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:52s} {dt*1e3:7.3f} ms  {n*8/dt/1e9:6.1f} GB/s", flush=True)


def h2d_pageable():
    dev.copy_(torch.from_numpy(a))


def h2d_register():
    ptr = a.ctypes.data
    cudart.cudaHostRegister(ptr, a.nbytes, 0)
    dev.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cudart.cudaHostUnregister(ptr)


def h2d_chunked():
    at = torch.from_numpy(a)
    step = (n + CH - 1) // CH
    evs = [None, None]
    for i in range(CH):
        lo, hi = i * step, min(n, (i + 1) * step)
        b = i & 1
        if evs[b] is not None:
            evs[b].synchronize()
        pins[b][:hi - lo].copy_(at[lo:hi])
        dev[lo:hi].copy_(pins[b][:hi - lo], non_blocking=True)
        evs[b] = torch.cuda.Event()
        evs[b].record()


def d2h_fresh():
    out = np.empty(n)
    torch.from_numpy(out).copy_(dev)
    return out


def d2h_chunked():
    out = np.empty(n)
    ot = torch.from_numpy(out)
    step = (n + CH - 1) // CH
    evs = []
    for i in range(CH):
        lo, hi = i * step, min(n, (i + 1) * step)
        pins[i & 1]  # noqa
    # issue chunk 0, then overlap copy-out of chunk i with D2H of chunk i+1
    def issue(i):
        lo, hi = i * step, min(n, (i + 1) * step)
        pins[i & 1][:hi - lo].copy_(dev[lo:hi], non_blocking=True)
        e = torch.cuda.Event()
        e.record()
        return e
    e = issue(0)
    for i in range(CH):
        lo, hi = i * step, min(n, (i + 1) * step)
        e.synchronize()
        if i + 1 < CH:
            # the other buffer was consumed in the previous iteration
            e_next = issue(i + 1)
        ot[lo:hi].copy_(pins[i & 1][:hi - lo])
        if i + 1 < CH:
            e = e_next
    return out


def d2h_register():
    out = np.empty(n)
    ptr = out.ctypes.data
    cudart.cudaHostRegister(ptr, out.nbytes, 0)
    torch.from_numpy(out).copy_(dev, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cudart.cudaHostUnregister(ptr)
    return out


print("threads", torch.get_num_threads(), "cpus", os.cpu_count())
timeit("H2D pageable (current)", h2d_pageable)
timeit("H2D cudaHostRegister in place", h2d_register)
timeit(f"H2D {CH} chunks via 2 pinned buffers", h2d_chunked)
timeit("D2H fresh pageable (current)", d2h_fresh)
timeit("D2H fresh via cudaHostRegister", d2h_register)
timeit(f"D2H fresh {CH} chunks via 2 pinned buffers", d2h_chunked)
for CH in (2, 8):
    pins = [torch.empty(n // CH + 1, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    timeit(f"H2D {CH} chunks via 2 pinned buffers", h2d_chunked)
    timeit(f"D2H fresh {CH} chunks via 2 pinned buffers", d2h_chunked)
x = d2h_chunked(); assert np.array_equal(x, dev.cpu().numpy())
h2d_chunked(); torch.cuda.synchronize(); assert np.array_equal(dev.cpu().numpy(), a)
print("ok")
