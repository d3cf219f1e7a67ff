"""Cached-apply time vs number of cells (p=16, Q=24): separates fixed per-launch
cost from per-element throughput."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import make_inputs, phi_sin  # noqa: E402

p, Q = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 24
for nc in (16, 32, 48, 64, 96, 128):
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, nc, p), 1.0, phi_sin, rule="gauss", nq=Q)
    psi, u, x, _ = make_inputs("obstacle", nc, nc, p)
    t = {k: torch.from_numpy(v).cuda() for k, v in (("psi", psi), ("u", u), ("x", x))}
    d.exp_moments_t(t["psi"], wcache=True)
    y = torch.empty_like(t["x"])
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        d.apply_cached_t(t["x"], out=y)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                d.apply_cached_t(t["x"], out=y)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 250 * 1e3
    print(f"cells={nc*nc:6d} us/apply={us:8.2f} us/1k-cells={us/(nc*nc)*1000:6.3f}")
