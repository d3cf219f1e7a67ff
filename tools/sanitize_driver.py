"""Small end-to-end pass over the library's entry points for compute-sanitizer
(memcheck / racecheck / synccheck): config 0 (both rules), config 4's p = 2 on
a 16 x 16 mesh, config 1's degree on 2 x 2 cells (warp path, generated U
passes), a gradient disc (CTA path), element blocks, the per-cell
preconditioner, the Schur operator, the device GMRES graph, and config 1's
degree on 60 x 60 cells (streaming apply, cell ranges, host slab pipeline,
row-per-thread LU and look-ahead solve).

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


def run_stream():
    """Config 1's degree on 60 x 60 cells: the persistent streaming apply
    (k_stream, split cells through shared memory + named barriers), the cell
    range entry, the host slab pipeline and page-locked inputs / results."""
    from paper_2412_13733_b200 import _lib
    from paper_2412_13733_b200.disc import pinned_array
    nc, p = 60, 16
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, nc, p), 1.0, phi_sin, rule="gauss", nq=24)
    psi, u, x, _ = make_inputs("obstacle", nc, nc, p, seed=2)
    Dm = d.assemble_D(psi)
    y = Dm @ x                                   # pageable x: two slabs (hpgApplyCachedHostSlab)
    xp = pinned_array(x.shape)
    xp[...] = x
    y2 = Dm @ xp                                 # page-locked x: one DMA, whole vector (k_stream)
    assert np.allclose(y, y2, rtol=1e-12, atol=1e-14)
    xt = torch.from_numpy(x).cuda()
    yt = torch.zeros_like(xt)
    for lo, hi in ((0, 40), (40, d.plan.ncells)):
        _lib.call("hpgApplyCachedRange", d.plan.handle, D._vp(Dm._w), D._vp(xt), D._vp(yt), lo, hi, D._stream())
    assert np.allclose(yt.cpu().numpy(), y, rtol=1e-12, atol=1e-14)
    M = D.DeviceCellBlockPreconditioner.from_blocks(
        d, torch.eye(d.n * d.n, dtype=torch.float64, device="cuda").repeat(d.plan.ncells, 1, 1)
        + 0.01 * torch.randn(d.plan.ncells, d.n * d.n, d.n * d.n, dtype=torch.float64, device="cuda"))
    M.apply_t(xt)                                # k_lu2 + look-ahead k_lu_solve
    torch.cuda.synchronize()
    print(f"ok stream nc={nc} p={p} path={d.plan.path}", flush=True)


if __name__ == "__main__":
    run("obstacle", 4, 8, "gauss", 12)          # config 0
    run("obstacle", 4, 8, "reference")
    run("obstacle", 16, 2, "gauss", 5)          # config 4, p = 2
    run("obstacle", 6, 4, "gauss", 7)           # config 4, p = 4 (k_lowp)
    run("obstacle", 2, 16, "gauss", 24)         # config 1 degree (k_warp)
    run("gradient", 2, 6, "gauss", 9)           # gradient, CTA path
    run("gradient", 3, 3, "reference")
    run_stream()
    print("sanitize driver done")
