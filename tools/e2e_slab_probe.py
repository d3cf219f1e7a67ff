"""Pieces of the slab-pipelined host D @ x (c1): host->pinned copy rate by size,
H2D / D2H DMA rates, and whether the two directions overlap."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

n = 921600
a = np.random.default_rng(0).standard_normal(n)
at = torch.from_numpy(a)
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
pin2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
dev2 = torch.empty(n, dtype=torch.float64, device="cuda")
print("threads", torch.get_num_threads(), "cpus", os.cpu_count())


def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for frac in (1, 2, 4, 8):
    m = n // frac
    print(f"host->pinned copy of {m * 8 / 1e6:.2f} MB: torch {t(lambda: pin[:m].copy_(at[:m])):.3f} ms   "
          f"numpy {t(lambda: np.copyto(pin.numpy()[:m], a[:m])):.3f} ms")
print(f"H2D pinned 7.4 MB: {t(lambda: dev.copy_(pin, non_blocking=True)):.3f} ms")
print(f"D2H pinned 7.4 MB: {t(lambda: pin2.copy_(dev2, non_blocking=True)):.3f} ms")
s2 = torch.cuda.Stream()


def both():
    dev.copy_(pin, non_blocking=True)
    with torch.cuda.stream(s2):
        pin2.copy_(dev2, non_blocking=True)


print(f"H2D + D2H on two streams: {t(both):.3f} ms")
print(f"pinned alloc+free 7.4 MB: {t(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True)):.3f} ms")

# the real path, step by step
from paper_2412_13733_b200 import disc as D, _lib  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402
import ctypes
cfg = CONFIGS["c1"]
inp = config_inputs(cfg)
d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
Dm = d.assemble_D(inp["psi"])
x = inp["x"]
print(f"Dm @ x: {t(lambda: Dm @ x):.3f} ms")
w = Dm._w
dx, dy = d._dev("in_x", n), d._dev("out_y", n)
out = torch.empty(n, dtype=torch.float64, pin_memory=True)
up = torch.cuda.Stream()
cur = torch.cuda.current_stream()
st = [torch.empty(n // 2, dtype=torch.float64, pin_memory=True) for _ in range(2)]
xt = torch.from_numpy(x)


def slabs(copy=True, sync=True):
    for k in range(2):
        if copy:
            st[k].copy_(xt[k * (n // 2):(k + 1) * (n // 2)])
        _lib.call("hpgApplyCachedHostSlab", d.plan.handle, D._vp(w), D._vp(st[k]), D._vp(dx), D._vp(dy), D._vp(out),
                  32 * k, 32 * (k + 1), ctypes.c_void_p(up.cuda_stream), D._stream())
    if sync:
        cur.synchronize()


print(f"2 slabs native (copy + sync each call): {t(slabs):.3f} ms")
print(f"2 slabs native, no host copy: {t(lambda: slabs(False)):.3f} ms")
print(f"2 slabs native, no per-call sync: {t(lambda: slabs(True, False)):.3f} ms")


def whole():
    dx.copy_(st_full, non_blocking=True)
    d.apply_cached_t(dx, out=dy, wcache=w)
    out.copy_(dy, non_blocking=True)
    cur.synchronize()


st_full = torch.empty(n, dtype=torch.float64, pin_memory=True)
print(f"whole vector pinned H2D + apply + D2H + sync: {t(whole):.3f} ms")


def slab1():
    _lib.call("hpgApplyCachedHostSlab", d.plan.handle, D._vp(w), D._vp(st_full), D._vp(dx), D._vp(dy), D._vp(out),
              0, 64, ctypes.c_void_p(up.cuda_stream), D._stream())
    cur.synchronize()


print(f"1 slab native (whole vector through the slab entry): {t(slab1):.3f} ms")
s3 = torch.cuda.Stream()
with torch.cuda.stream(s3):
    cur = torch.cuda.current_stream()
    print(f"2 slabs native on a side compute stream: {t(slabs):.3f} ms")
    print(f"1 slab native on a side compute stream: {t(slab1):.3f} ms")
cur = torch.cuda.current_stream()
# raw torch version of the 2-slab pipeline, no kernel
h = n // 2


def raw2():
    for k in range(2):
        with torch.cuda.stream(up):
            dx[k * h:(k + 1) * h].copy_(st[k], non_blocking=True)
            ev = torch.cuda.Event(); ev.record(up)
        cur.wait_event(ev)
        out[k * h:(k + 1) * h].copy_(dy[k * h:(k + 1) * h], non_blocking=True)
    cur.synchronize()


print(f"raw torch 2-slab H2D/D2H pipeline, no kernel: {t(raw2):.3f} ms")
