"""Warm timings (CUDA graphs, events) of the residual's pieces for a config."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
inp = config_inputs(cfg)
d = (D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D)(
    uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
t = {k: torch.from_numpy(inp[k]).to(d.device) for k in ("psi", "psi_prev", "u", "x")}
bu = torch.empty(d.ndof_u, dtype=torch.float64, device=d.device)
bp = torch.empty(d.ndof_psi, dtype=torch.float64, device=d.device)
y = torch.empty(d.ndof_psi, dtype=torch.float64, device=d.device)
fl = torch.zeros(1, dtype=torch.int32, device=d.device)


def timed(name, fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
        torch.cuda.synchronize()
    print(f"{name:40s} {e0.elapsed_time(e1) / reps * 1e3:9.2f} us", flush=True)


timed("residual (+cache)", lambda: d.residual_t(cfg.alphas[0], t["psi_prev"], t["u"], t["psi"], b_u=bu, b_psi=bp, flag=fl, wcache=True))
timed("residual (no cache)", lambda: d.residual_t(cfg.alphas[0], t["psi_prev"], t["u"], t["psi"], b_u=bu, b_psi=bp, flag=fl))
if cfg.kind == "obstacle":
    timed("psi-side moments (+cache)", lambda: d.exp_moments_t(t["psi"], out=bp, wcache=True, flag=fl))
    timed("psi-side moments (no cache)", lambda: d.exp_moments_t(t["psi"], out=bp, flag=fl))
timed("apply from psi", lambda: d.apply_D_t(t["psi"], t["x"], out=y))
timed("apply cached", lambda: d.apply_cached_t(t["x"], out=y))
timed("residual+apply (fused entry)", lambda: d.residual_apply_t(cfg.alphas[0], t["psi_prev"], t["u"], t["psi"], t["x"], b_u=bu, b_psi=bp, y=y, flag=fl))
timed("B^T u alone", lambda: d.BT_u_t(t["u"], out=bp))
