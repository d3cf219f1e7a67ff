"""Driver for ncu of the single-pass low-degree residual (+ apply): one
warm-up call, then a few fused residual_apply calls on a config-4 mesh."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4p6"]
inp = config_inputs(cfg)
d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
t = {k: torch.from_numpy(inp[k]).to(d.device) for k in ("psi", "psi_prev", "u", "x")}
for _ in range(4):
    d.residual_apply_t(cfg.alphas[0], t["psi_prev"], t["u"], t["psi"], t["x"])
torch.cuda.synchronize()
print("ok")
