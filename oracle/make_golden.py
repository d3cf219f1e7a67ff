"""Generate golden vectors from the UNMODIFIED reference package (test infrastructure).

Run here (the reference exists only in this container)::

    PYTHONPATH=/root/reference/pkg/src:. python oracle/make_golden.py

Writes ``tests/golden/*.npz``.  Each fixture holds the seeded inputs
(``paper_2412_13733_b200.workloads.make_inputs``), the quadrature tables the
reference used, and the reference's outputs:

* ``exp_moments`` / ``nl_moments`` (+ clamp flag),
* ``proximal.residual`` -> b_u, b_psi, clamped,
* ``apply_D(psi, x)`` and the assembled ``D @ x``,
* ``assemble_D`` blocks (all cells when small, else selected rows),
* ``phi_moments`` / ``phi_values`` and ``f_load``.

rule="gauss" fixtures substitute Gauss tables into the reference's own
``CellKernel1D`` objects and refresh the data
terms; the reference's unmodified methods then compute Gauss-rule results.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

from hpgalerkin import linalg, proximal                           # noqa: E402
from hpgalerkin.assembly import (GradientDisc2D, ObstacleDisc2D,   # noqa: E402
                                 _eval_data)
from hpgalerkin.mesh import Mesh1D, TensorMesh2D, uniform_mesh_2d  # noqa: E402

from paper_2412_13733_b200 import tables as tb                     # noqa: E402
from paper_2412_13733_b200.workloads import (make_inputs, phi_bilinear,  # noqa: E402
                                             phi_sin)

PREC_BETA = 0.25     # large enough that the E_beta term shows in the parity checks
SCHUR_RTOL = 1e-10
OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def substitute_gauss(disc, Q):
    """Replace every cell's tables by the Q-point Gauss rule (in place)."""
    p = int(disc.mesh.degrees_x[0])
    n = p - 1 if disc.kind == "obstacle" else p
    t = tb.Tables("gauss", p, n, Q)
    for k2 in disc.kernels.values():
        for k1 in (k2.kx, k2.ky):
            k1.nquad = Q
            k1.points = k1.midpoint + 0.5 * k1.h * t.xi
            k1.S = t.S
            k1.T = t.T
            k1.Su = t.Su
            k1.Tu = t.Tu
    return t


def build(kind, xpts, ypts, p, rule, Q, f, phi):
    mesh = TensorMesh2D(Mesh1D(xpts, np.full(len(xpts) - 1, p)),
                        Mesh1D(ypts, np.full(len(ypts) - 1, p)))
    cls = ObstacleDisc2D if kind == "obstacle" else GradientDisc2D
    disc = cls(mesh, f, phi)
    if rule == "gauss":
        t = substitute_gauss(disc, Q)
        disc.f_load = disc.load_vector(f)
        if kind == "obstacle":
            disc.phi_moments = disc.data_moments(phi)
        else:
            disc.phi_values = {c: _eval_data(phi, disc.kernels[c], "pointwise", 2)
                               for c in disc.cell_ids}
    else:
        n = p - 1 if kind == "obstacle" else p
        t = tb.Tables("reference", p, n)
        k = disc.kernels[disc.cell_ids[0]].kx
        assert np.array_equal(k.S, t.S) and np.array_equal(k.T, t.T)
    return disc, t


def case(name, kind, xpts, ypts, p, rule, Q=None, alpha=1.0, phi=phi_sin,
         seed=0, psi_scale=1.0, block_rows=None, psi_override=None, schur=True):
    xpts = np.asarray(xpts, dtype=float)
    ypts = np.asarray(ypts, dtype=float)
    disc, t = build(kind, xpts, ypts, p, rule, Q, 1.0, phi)
    psi, u, x, _ = make_inputs(kind, xpts.size - 1, ypts.size - 1, p, seed=seed)
    psi = psi * psi_scale
    if psi_override is not None:
        psi = psi_override(psi)
    psi_prev = np.zeros_like(psi)
    out = dict(kind=kind, xpts=xpts, ypts=ypts, p=p, rule=rule, nq=t.nq, alpha=alpha,
               S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi,
               psi=psi, u=u, x=x, psi_prev=psi_prev, f_load=disc.f_load)
    if kind == "obstacle":
        em, cl = disc.exp_moments(psi)
        out.update(moments=em, clamped=cl, phi_moments=disc.phi_moments)
    else:
        out.update(moments=disc.nl_moments(psi), clamped=False,
                   phi_values=np.stack([disc.phi_values[c] for c in disc.cell_ids]))
    b_u, b_psi, cl = proximal.residual(disc, alpha, psi_prev, u, psi)
    out.update(b_u=b_u, b_psi=b_psi, res_clamped=cl)
    out["apply_D"] = disc.apply_D(psi, x)
    D = disc.assemble_D(psi)
    out["Dx"] = D @ x
    out["D_clamped"] = bool(getattr(D, "clamped", False))
    blocks = np.stack(D.blocks)
    # per-cell Schur preconditioner (linalg.py:262-264) at PREC_BETA
    pb = np.stack(disc.precond_blocks(D, alpha, PREC_BETA))
    out["prec_beta"] = PREC_BETA
    try:
        out["precond_apply"] = linalg.schur_preconditioner(disc, D, alpha, PREC_BETA).apply(x)
    except ValueError:          # scipy lu_factor rejects non-finite blocks
        out["precond_error"] = True
    # Schur-reduced Newton step (linalg.py:213-287) with SuperLU on A
    if schur and not np.isnan(psi).any():
        A_factor = linalg.factor_stiffness(disc.A, "splu", 2)
        E = disc.E_matrix(PREC_BETA)
        out["stiff_solve"] = A_factor.solve(u)
        out["schur_mv"] = linalg.SchurOperator(disc, D, E, alpha, A_factor).matvec(x)
        r = linalg.schur_solve(disc, D, alpha, PREC_BETA, out["b_u"], out["b_psi"], A_factor,
                               rtol=SCHUR_RTOL, maxiter=150, E=E)
        out.update(schur_du=r.du, schur_dpsi=r.dpsi, schur_iters=r.gmres.iterations,
                   schur_res=np.asarray(r.gmres.residuals))
    if block_rows is None:
        out["blocks"] = blocks
        out["precond_blocks"] = pb
    else:
        rows = np.asarray(block_rows)
        out["block_rows"] = rows
        out["blocks_sel"] = blocks[:, rows, :]
        out["precond_sel"] = pb[:, rows, :]
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB  ndof_psi={psi.size} "
          f"ndof_u={u.size} nq={t.nq} clamped={out['clamped']}")


def solve_case(name, kind, nc, p, rule, Q=None, phi=phi_sin, beta=1e-3, alpha_max=8.0,
               line_search=False, linear_solver="schur"):
    """The reference's whole penalty continuation (proximal.solve) from zero."""
    pts = np.linspace(0.0, 1.0, nc + 1)
    disc, t = build(kind, pts, pts, p, rule, Q, 1.0, phi)
    sched = proximal.AlphaSchedule(alpha0=1.0, rate=2.0, alpha_max=alpha_max)
    opts = proximal.SolverOptions(line_search=line_search, linear_solver=linear_solver)
    rep = proximal.solve(disc, sched, beta, opts)
    out = dict(kind=kind, xpts=pts, ypts=pts, p=p, rule=rule, nq=t.nq, alpha=1.0, beta=beta,
               alpha_max=alpha_max, line_search=line_search, linear_solver=linear_solver,
               S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi,
               u=rep.u, psi=rep.psi, multiplier=rep.multiplier,
               outer_increment=rep.outer_increment, converged=rep.converged,
               newton_iters=np.array([s.newton_iters for s in rep.steps]),
               gmres_iters=np.array([sum(s.gmres_iters) for s in rep.steps]),
               alphas=np.array([s.alpha for s in rep.steps]))
    path = os.path.join(OUT, "solve", f"{name}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **out)
    print(f"solve/{name}: newton {out['newton_iters'].tolist()} gmres {out['gmres_iters'].tolist()}")


def qvi_case(name, nc, p, rule, Q=None, load=100.0, scale=0.05):
    """QVI temperature pieces (qvi.py:35-127) from the reference's own code."""
    from hpgalerkin import qvi
    from hpgalerkin.problems import ThermoformingData
    data = ThermoformingData(load=load)
    pts = np.linspace(0.0, 1.0, nc + 1)
    disc, t = build("obstacle", pts, pts, p, rule, Q, data.f, 0.0)
    solver = qvi.TemperatureSolver(disc, data)
    rng = np.random.default_rng(11)
    nf = solver.H.shape[0]
    vfull = rng.standard_normal(nf)
    rvals = rng.standard_normal((len(disc.cell_ids), t.nq, t.nq))
    _, u, _, _ = make_inputs("obstacle", nc, nc, p, seed=3)
    u_full = disc.u_space.extend_interior(scale * u)
    T, newton, gmres_its = solver.solve(u_full)
    out = dict(xpts=pts, ypts=pts, p=p, rule=rule, nq=t.nq, load=load, gamma=data.gamma,
               S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi,
               vfull=vfull, vals=np.stack(qvi._cell_grid_values(disc, vfull)),
               rvals=rvals, load_full=qvi._load_full(disc, list(rvals)), Hv=solver.H @ vfull,
               u_full=u_full, temp=T, newton=newton, gmres=np.array(gmres_its))
    path = os.path.join(OUT, "qvi", f"{name}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **out)
    print(f"qvi/{name}: nfull={nf} newton={newton} gmres={gmres_its}")


def solve_cases_r02():
    """Round-2 continuations: the monolithic solver and the gradient constraint,
    for the drop-in tests (tests/test_gpu_dropin.py)."""
    solve_case("obst_p4_mono_ref", "obstacle", 4, 4, "reference", linear_solver="monolithic")
    solve_case("obst_p5_mono_gauss", "obstacle", 3, 5, "gauss", Q=8, linear_solver="monolithic")
    grad_solve_case("grad_p2_ref", 4, 2, "reference")
    grad_solve_case("grad_p3_mono_gauss", 4, 3, "gauss", Q=6, linear_solver="monolithic")


def grad_solve_case(name, nc, p, rule, Q=None, linear_solver="schur"):
    """The reference CLI's gradient2d study settings (cli.py:321-360): the
    GradientFrame2D data with cellwise phi, alpha 2^-7 * sqrt(2)^k up to 4,
    Newton rtol 3e-5, GMRES rtol 1e-3, beta = 10^(-p + log2 h)."""
    import math

    from hpgalerkin.problems import GradientFrame2D
    prob = GradientFrame2D()
    pts = np.linspace(0.0, 1.0, nc + 1)
    mesh = TensorMesh2D(Mesh1D(pts, np.full(nc, p)), Mesh1D(pts, np.full(nc, p)))
    disc = GradientDisc2D(mesh, prob.f, prob.phi, phi_mode="cellwise")
    if rule == "gauss":
        t = substitute_gauss(disc, Q)
        disc.f_load = disc.load_vector(prob.f)
        disc.phi_values = {c: _eval_data(prob.phi, disc.kernels[c], "cellwise", 2)
                           for c in disc.cell_ids}
    else:
        t = tb.Tables("reference", p, p)
    sched = proximal.AlphaSchedule(alpha0=2.0 ** -7, rate=math.sqrt(2.0), alpha_max=4.0)
    opts = proximal.SolverOptions(newton_rtol=3e-5, newton_atol=1e-13, gmres_rtol=1e-3,
                                  linear_solver=linear_solver)
    beta = 10.0 ** (-p + math.log2(1.0 / nc))
    rep = proximal.solve(disc, sched, beta, opts)
    out = dict(kind="gradient", xpts=pts, ypts=pts, p=p, rule=rule, nq=t.nq, alpha=2.0 ** -7,
               beta=beta, alpha_max=4.0, line_search=False, linear_solver=linear_solver,
               S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi,
               u=rep.u, psi=rep.psi, multiplier=rep.multiplier,
               outer_increment=rep.outer_increment, converged=rep.converged,
               newton_iters=np.array([s.newton_iters for s in rep.steps]),
               gmres_iters=np.array([sum(s.gmres_iters) for s in rep.steps]),
               alphas=np.array([s.alpha for s in rep.steps]))
    path = os.path.join(OUT, "solve", f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"solve/{name}: newton {out['newton_iters'].tolist()} gmres {out['gmres_iters'].tolist()}")


def main():
    if "--r02" in sys.argv:
        solve_cases_r02()
        return
    os.makedirs(OUT, exist_ok=True)
    u4 = np.linspace(0.0, 1.0, 5)
    u2 = np.linspace(0.0, 1.0, 3)
    u1 = np.linspace(0.0, 1.0, 2)
    # config 0 (full size), both rules
    case("c0_ref", "obstacle", u4, u4, 8, "reference")
    case("c0_gauss", "obstacle", u4, u4, 8, "gauss", Q=12)
    # config 4 degrees on a 4x4 mesh (per-cell work identical to 256x256)
    for p in (2, 4, 6):
        case(f"c4p{p}_ref", "obstacle", u4, u4, p, "reference", alpha=4.0)
        case(f"c4p{p}_gauss", "obstacle", u4, u4, p, "gauss", Q=p + 3, alpha=4.0)
    # config 1 degree on a 2x2 mesh
    case("c1_ref", "obstacle", u2, u2, 16, "reference", alpha=4.0)
    case("c1_gauss", "obstacle", u2, u2, 16, "gauss", Q=24, alpha=16.0)
    # config 2 degree (gradient) on one and two cells; blocks as selected rows
    case("c2_ref", "gradient", u2, u1, 24, "reference", phi=phi_bilinear,
         block_rows=np.arange(0, 1152, 97))
    case("c2_gauss", "gradient", u2, u1, 24, "gauss", Q=36, phi=phi_bilinear,
         block_rows=np.arange(0, 1152, 97))
    # small gradient with full blocks
    case("grad_p6_ref", "gradient", u2, u2, 6, "reference", phi=phi_bilinear)
    case("grad_p6_gauss", "gradient", u2, u2, 6, "gauss", Q=9, phi=phi_bilinear)
    # config 3 degree on one cell, blocks as selected rows
    case("c3_ref", "obstacle", u1, u1, 82, "reference",
         block_rows=np.array([0, 1, 80, 81, 3280, 6560]), schur=False)
    case("c3_gauss", "obstacle", u1, u1, 82, "gauss", Q=128,
         block_rows=np.array([0, 1, 80, 81, 3280, 6560]), schur=False)
    # non-uniform widths, rectangular mesh
    xs = np.array([0.0, 0.15, 0.5, 1.0])
    ys = np.array([0.0, 0.3, 1.0])
    case("nonuni_ref", "obstacle", xs, ys, 5, "reference", alpha=2.0)
    case("nonuni_grad_gauss", "gradient", xs, ys, 4, "gauss", Q=7, phi=phi_bilinear)
    # clamp: overflow side must flag; NaN must flag
    case("clamp_ref", "obstacle", u2, u2, 3, "reference", psi_scale=-2000.0, schur=False)

    def nan_one(psi):
        psi = psi.copy()
        psi[5] = np.nan
        return psi

    case("nan_ref", "obstacle", u2, u2, 3, "reference", psi_override=nan_one)
    # QVI temperature solve pieces
    qvi_case("qvi_p4_gauss", 4, 4, "gauss", Q=7)
    qvi_case("qvi_p6_ref", 3, 6, "reference")
    qvi_case("qvi_p8_gauss", 4, 8, "gauss", Q=12, scale=0.2)
    # whole continuations (proximal.solve)
    solve_case("obst_p6_gauss", "obstacle", 4, 6, "gauss", Q=9)
    solve_case("obst_p8_ref", "obstacle", 4, 8, "reference")
    solve_case("obst_p4_ls", "obstacle", 6, 4, "gauss", Q=7, line_search=True)


if __name__ == "__main__":
    main()
