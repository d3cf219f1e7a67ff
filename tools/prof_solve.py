"""Time the whole penalty continuation (proximal.solve) on the GPU.

    python tools/prof_solve.py [cfg] [alpha_max]

Obstacle configs only (the reference's gradient continuation needs
problem-specific settings).  Prints per-step Newton/GMRES counts and the
wall time split (assembly = D(psi) weights, linsolve = preconditioner
factor + Schur GMRES), synchronised.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2412_13733_b200 import disc as D, proximal                 # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d                 # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs      # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    amax = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
    cfg = CONFIGS[name]
    inp = config_inputs(cfg)
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss",
                         nq=cfg.Q)
    sched = proximal.AlphaSchedule(alpha0=1.0, rate=2.0, alpha_max=amax)
    proximal.solve(d, proximal.AlphaSchedule(alpha0=1.0, nsteps=1), 1e-8)     # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = proximal.solve(d, sched, 1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"{name}: ndof_u={d.ndof_u} ndof_psi={d.ndof_psi} alphas={[s.alpha for s in rep.steps]} "
          f"converged={rep.converged}")
    print(f"  newton per step {[s.newton_iters for s in rep.steps]}  gmres per step "
          f"{[s.gmres_total for s in rep.steps]}")
    print(f"  total {t:.3f} s  ({rep.newton_total} Newton steps, {t / max(1, rep.newton_total) * 1e3:.1f} ms each; "
          f"assembly {rep.t_assembly_s:.3f} s, linsolve {rep.t_linsolve_s:.3f} s)")


if __name__ == "__main__":
    main()
