"""Interleaved A/B of the host-buffer D @ x transfer strategies on config 1
(same process, same box, alternating): slabs + page-locked results, whole
vector + page-locked results, whole vector + pageable results (round-2 start)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_13733_b200 import disc as D
from paper_2412_13733_b200.mesh import uniform_mesh_2d
from paper_2412_13733_b200.proximal import residual
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]; inp = config_inputs(cfg)
cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
d = cls(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
hp = {k: np.ascontiguousarray(inp[k]) for k in ("psi", "psi_prev", "u", "x")}
Dm = d.assemble_D(hp["psi"])
modes = {"slabs2+pinned": (2, False), "whole+pinned": (1, False), "whole+pageable": (1, True)}
res = {k: [] for k in modes}
for rep in range(7):
    for name, (slabs, nopin) in modes.items():
        d._SLABS = slabs
        if nopin:
            os.environ["HPG_NO_PINNED_OUT"] = "1"
        else:
            os.environ.pop("HPG_NO_PINNED_OUT", None)
        t0 = time.perf_counter()
        for _ in range(50):
            Dm @ hp["x"]
        torch.cuda.synchronize()
        if rep > 0:
            res[name].append((time.perf_counter() - t0) / 50 * 1e3)
os.environ.pop("HPG_NO_PINNED_OUT", None)
for name, v in res.items():
    print(f"{name:16s} per D @ x: min {min(v):.3f} median {np.median(v):.3f} max {max(v):.3f} ms")
ts = []
for _ in range(6):
    t0 = time.perf_counter(); residual(d, 1.0, hp["psi_prev"], hp["u"], hp["psi"]); ts.append(time.perf_counter() - t0)
print(f"residual (host buffers): min {min(ts)*1e3:.3f} median {np.median(ts)*1e3:.3f} ms")
