"""Small end-to-end pass over the library's entry points for compute-sanitizer
(memcheck / racecheck / synccheck): config 0 (both rules), config 4's p = 2 on
a 16 x 16 mesh, config 1's degree on 2 x 2 cells (warp path, generated U
passes), a gradient disc (CTA path), element blocks, the per-cell
preconditioner, the Schur operator and the device GMRES graph.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_13733_b200 import disc as D, schur  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.proximal import residual  # noqa: E402
from paper_2412_13733_b200.workloads import make_inputs, phi_bilinear, phi_sin  # noqa: E402


def run(kind, nc, p, rule, nq=None, blocks=True, solve=True):
    cls = D.ObstacleDisc2D if kind == "obstacle" else D.GradientDisc2D
    phi = phi_sin if kind == "obstacle" else phi_bilinear
    d = cls(uniform_mesh_2d(0.0, 1.0, nc, p), 1.0, phi, rule=rule, nq=nq)
    psi, u, x, _ = make_inputs(kind, nc, nc, p, seed=1)
    residual(d, 2.0, 0.5 * psi, u, psi)
    d.apply_D(psi, x)
    Dm = d.assemble_D(psi)
    Dm @ x
    t = lambda a: torch.from_numpy(a).cuda()
    d.residual_apply_t(2.0, t(0.5 * psi), t(u), t(psi), t(x))
    if blocks:
        Dm.blocks_t()
        Dm.matvec_blocks_t(t(x))
    if solve and d.ndof_u > 0:
        M = d.schur_preconditioner(Dm, 2.0, 1e-3)
        M.apply(x)
        Af = schur.DeviceStiffnessFactor(d)
        b_u, b_psi, _ = d.residual_t(2.0, t(0.5 * psi), t(u), t(psi), wcache=True)
        r = schur.schur_solve_t(d, d.assemble_D_t(t(psi)), 2.0, 1e-3, b_u, b_psi, Af, rtol=1e-10, maxiter=40)
        assert r.gmres.iterations > 0
    torch.cuda.synchronize()
    print(f"ok {kind} nc={nc} p={p} {rule} path={d.plan.path} splits={d.plan.splits}", flush=True)


if __name__ == "__main__":
    run("obstacle", 4, 8, "gauss", 12)          # config 0
    run("obstacle", 4, 8, "reference")
    run("obstacle", 16, 2, "gauss", 5)          # config 4, p = 2
    run("obstacle", 6, 4, "gauss", 7)           # config 4, p = 4 (k_lowp)
    run("obstacle", 2, 16, "gauss", 24)         # config 1 degree (k_warp)
    run("gradient", 2, 6, "gauss", 9)           # gradient, CTA path
    run("gradient", 3, 3, "reference")
    print("sanitize driver done")
