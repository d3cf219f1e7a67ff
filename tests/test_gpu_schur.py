"""GPU parity of the device Schur solve against the
reference's SuperLU-based SchurOperator / schur_solve (golden fixtures).

Stiffness solve and Schur matvec: 1e-12 global max-norm relative.  The GMRES
solve: same iteration count, residual history and solution to the GMRES
tolerance scale (rtol 1e-10 in the fixtures; the operators differ from the
reference's only by fp64 rounding).
"""
import numpy as np
import pytest

from golden_util import load, names
from oracle import hpg_oracle as orc
from test_gpu_fullsize import build
from test_gpu_parity import make_disc

pytestmark = pytest.mark.gpu
TOL = 1e-12
SMALL = [n for n in names() if not n.startswith("c3") and n not in ("clamp_ref", "nan_ref")]


@pytest.mark.parametrize("name", SMALL)
def test_schur_golden(name):
    from paper_2412_13733_b200 import schur
    g = load(name)
    d = make_disc(g)
    beta = float(g["prec_beta"])
    Af = schur.DeviceStiffnessFactor(d)
    assert orc.rel_err(Af.solve(g["u"]), g["stiff_solve"]) < TOL
    D = d.assemble_D(g["psi"])
    S = schur.DeviceSchurOperator(d, D, beta, g["alpha"], Af)
    assert orc.rel_err(S @ g["x"], g["schur_mv"]) < TOL
    r = schur.schur_solve(d, D, g["alpha"], beta, g["b_u"], g["b_psi"], Af, rtol=1e-10)
    assert r.gmres.iterations == int(g["schur_iters"])
    assert r.gmres.converged
    res, rres = np.asarray(r.gmres.residuals), g["schur_res"]
    assert np.allclose(res, rres, rtol=1e-6, atol=1e-9 * rres[0])
    assert orc.rel_err(r.dpsi, g["schur_dpsi"]) < 1e-8
    assert orc.rel_err(r.du, g["schur_du"]) < 1e-8


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c4p4"])
def test_full_size_stiffness_and_schur(cfg_name):
    """BASELINE sizes: A x == b through the exact A u kernel (backward error),
    and the one-call Schur apply == its composition from the pieces."""
    import torch
    from paper_2412_13733_b200 import schur
    cfg, d, P, inp, dev = build(cfg_name)
    alpha, beta = cfg.alphas[-1], 1e-3
    Af = schur.DeviceStiffnessFactor(d)
    x = Af.solve_t(dev["u"])
    xh = x.cpu().numpy()
    # normwise backward error through the exact A u kernel:
    # ||A x - b|| / (||A|| ||x|| + ||b||), ||A||_inf <= |Kx||My| + |Mx||Ky| (kron norms)
    import scipy.linalg as sla
    Kx, Mx = schur.u_matrices_1d(d.hx, cfg.p)
    nA = 2 * np.abs(Kx).sum(1).max() * np.abs(Mx).sum(1).max()
    r = d.A_u_t(x).cpu().numpy() - inp["u"]
    assert np.abs(r).max() / (nA * np.abs(xh).max() + np.abs(inp["u"]).max()) < 1e-14   # ~90 eps
    # forward: the same fast diagonalisation restated in NumPy
    lx, Vx = sla.eigh(Kx, Mx)
    B = inp["u"].reshape(Kx.shape[0], Kx.shape[0])
    X = Vx @ ((Vx.T @ B @ Vx) / (lx[:, None] + lx[None, :])) @ Vx.T
    assert orc.rel_err(xh, X.ravel()) < TOL
    d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
    D = d.assemble_D_t(dev["psi"])
    S = schur.DeviceSchurOperator(d, D, beta, alpha, Af)
    y = S.matvec_t(dev["x"]).cpu().numpy()
    Dx = d.apply_cached_t(dev["x"], wcache=D._w).cpu().numpy()
    z = d.BT_u_t(Af.solve_t(d.B_psi_t(dev["x"]))).cpu().numpy()
    if cfg.kind == "obstacle":
        Ex = beta * d.mass_psi * inp["x"]
    else:
        Ex = beta * _grad_E_apply(d, inp["x"])
    ref = -((Dx + Ex) + z / alpha)
    assert orc.rel_err(y, ref) < TOL
    torch.cuda.synchronize()


def _grad_E_apply(d, x):
    """E_unit blocks (assembly.py:753-759) applied per cell and component."""
    n = d.n
    out = np.zeros_like(x)
    for (cx, cy), idx in zip(d.cell_ids, d.cell_psi_indices):
        _, kx, mx = orc.spectral_1d(n, d.hx[cx])
        _, ky, my = orc.spectral_1d(n, d.hy[cy])
        E = np.kron(np.diag(kx), my) + np.kron(mx, np.diag(ky))
        m2 = n * n
        out[idx[:m2]] = E @ x[idx[:m2]]
        out[idx[m2:]] = E @ x[idx[m2:]]
    return out


def test_schur_needs_factor():
    from paper_2412_13733_b200 import _lib
    g = load("c0_gauss")
    d = make_disc(g)
    D = d.assemble_D(g["psi"])
    import torch
    xt = torch.from_numpy(g["x"]).cuda()
    out = torch.empty_like(xt)
    with pytest.raises(ValueError):
        _lib.call("hpgSchurApply", d.plan.handle, _lib.ctypes.c_void_p(D._w.data_ptr()), 1.0, 0.0,
                  _lib.ctypes.c_void_p(xt.data_ptr()), _lib.ctypes.c_void_p(out.data_ptr()), None)


def test_device_gmres_matches_reference_gmres_edge_cases():
    """schur.DeviceGmres vs the reference algorithm (linalg.py:134-207, restated
    here on the host) on a small nonsymmetric system: right and left
    preconditioning, a nonzero x0, the zero right-hand side (0 iterations,
    converged), maxiter exhaustion (not converged), and reuse of one workspace."""
    import torch
    from paper_2412_13733_b200 import schur
    rng = np.random.default_rng(3)
    n = 300
    Am = np.eye(n) * 4.0 + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
    Mm = np.diag(1.0 / np.diag(Am))
    b = rng.standard_normal(n)
    x0 = 0.1 * rng.standard_normal(n)
    At = torch.from_numpy(Am).cuda()
    Mt = torch.from_numpy(Mm).cuda()

    def amul(x, out):
        torch.mv(At, x, out=out)

    def pmul(x, out):
        torch.mv(Mt, x, out=out)

    def host_gmres(side, xs, rtol, maxiter):
        # the reference's algorithm, linalg.py:134-207
        x = np.zeros(n) if xs is None else xs.copy()
        r = b - Am @ x if np.any(x) else b.copy()
        if side == "left":
            r = Mm @ r
        beta = np.linalg.norm(r)
        if beta == 0.0:
            return x, 0, True
        V = [r / beta]
        H = np.zeros((maxiter + 1, maxiter)); cs = np.zeros(maxiter); sn = np.zeros(maxiter)
        g = np.zeros(maxiter + 1); g[0] = beta
        k, conv = 0, False
        for j in range(maxiter):
            w = Mm @ (Am @ V[j]) if side == "left" else Am @ (Mm @ V[j])
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (H[j, j] / d, H[j + 1, j] / d)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            g[j + 1] = -sn[j] * g[j]; g[j] = cs[j] * g[j]; H[j + 1, j] = 0.0
            k = j + 1
            if abs(g[j + 1]) <= rtol * beta:
                conv = True
                break
            V.append(w / np.linalg.norm(w))
        import scipy.linalg as sla
        y = sla.solve_triangular(H[:k, :k], g[:k], lower=False)
        dx = sum(y[i] * V[i] for i in range(k))
        if side == "right":
            dx = Mm @ dx
        return x + dx, k, conv

    G = schur.DeviceGmres(n, 40, torch.device("cuda"))
    bt = torch.from_numpy(b).cuda()
    tmp = torch.empty_like(bt)
    amul(bt, tmp)                     # library handles set up before any graph capture
    pmul(bt, tmp)
    torch.cuda.synchronize()
    for side in ("right", "left"):
        for xs in (None, x0):
            res = G.solve(amul, bt, M=pmul, side=side, x0=None if xs is None else torch.from_numpy(xs).cuda(),
                          rtol=1e-10)
            xr, kr, cr = host_gmres(side, xs, 1e-10, 40)
            assert abs(res.iterations - kr) <= 1 and res.converged == cr
            assert orc.rel_err(res.x.cpu().numpy(), xr) < 1e-9
            assert orc.rel_err(res.x.cpu().numpy(), np.linalg.solve(Am, b)) < 1e-8
    # zero right-hand side: 0 iterations, converged, x = 0
    z = G.solve(amul, torch.zeros(n, dtype=torch.float64, device="cuda"), M=pmul)
    assert z.iterations == 0 and z.converged and float(z.x.abs().max()) == 0.0
    # maxiter exhaustion: not converged after exactly maxiter iterations
    G3 = schur.DeviceGmres(n, 3, torch.device("cuda"))
    r3 = G3.solve(amul, bt, M=pmul, rtol=1e-14)
    xr, kr, cr = host_gmres("right", None, 1e-14, 3)
    assert r3.iterations == 3 and not r3.converged and kr == 3 and not cr
    assert orc.rel_err(r3.x.cpu().numpy(), xr) < 1e-10
    assert len(r3.residuals) == 4 and r3.residuals[0] == pytest.approx(np.linalg.norm(b))
