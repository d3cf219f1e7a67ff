"""Warm-L2 driver for the cached Jacobian apply (the c1 dominant kernel): one
residual then several applies, so ncu can pick an apply launch by index."""
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
d.residual_t(1.0, t["psi_prev"], t["u"], t["psi"], wcache=True)
y = torch.empty_like(t["x"])
for _ in range(6):
    d.apply_cached_t(t["x"], out=y)
torch.cuda.synchronize()
print("ok")
