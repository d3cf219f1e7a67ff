"""Run a config's hot-path calls a few times (no graphs) for ncu launch lists.

    python tools/prof_step.py c1 [gauss|reference] [blocks]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
    rule = sys.argv[2] if len(sys.argv) > 2 else "gauss"
    blocks = len(sys.argv) > 3 and sys.argv[3] == "blocks"
    inp = config_inputs(cfg)
    mesh = uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p)
    cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
    d = cls(mesh, inp["f"], inp["phi"], rule=rule, nq=cfg.Q if rule == "gauss" else None)
    dev = d.device
    t = {k: torch.from_numpy(inp[k]).to(dev) for k in ("psi", "psi_prev", "u", "x")}
    torch.cuda.synchronize()
    for _ in range(3):
        d.residual_t(cfg.alphas[0], t["psi_prev"], t["u"], t["psi"], wcache=True)
        d.apply_cached_t(t["x"])
        d.apply_D_t(t["psi"], t["x"])
        if blocks:
            d.blocks_t()
    torch.cuda.synchronize()
    print("ok", d.plan.path, d.plan.splits)


if __name__ == "__main__":
    main()
