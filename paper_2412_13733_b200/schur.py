"""The Schur-reduced Newton solve on the device.

Mirrors ``hpgalerkin/linalg.py``:

* ``DeviceStiffnessFactor``  -- ``factor_stiffness`` / ``SpluFactor``
  (``linalg.py:100-117``): ``.solve(b)`` with the interior stiffness
  ``A = Kx (x) My + Mx (x) Ky`` (``assembly.py:42-78,470-474``).  Instead of a
  sparse LU, the tensor structure is diagonalised once on the host (1D
  generalized eigenproblems, ``u_matrices_1d``) and every solve is four dense
  GEMMs on the device (``hpgStiffnessSolve``).
* ``DeviceSchurOperator``    -- ``SchurOperator`` (``linalg.py:213-243``):
  ``-(D + E + B^T (alpha A)^{-1} B) x`` in one C-ABI call (``hpgSchurApply``).
* ``gmres_t``                -- ``gmres`` (``linalg.py:134-207``): unrestarted
  GMRES with modified Gram-Schmidt and Givens rotations, same algorithm and
  stopping rule, vectors resident on the device.
* ``schur_solve``            -- ``schur_solve`` (``linalg.py:269-287``).
"""

import ctypes
from collections import namedtuple

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib
from .disc import F64, DeviceCellBlockMatrix, _stream, _vp

GmresResult = namedtuple("GmresResult", "x iterations residuals converged")
SchurSolveResult = namedtuple("SchurSolveResult", "du dpsi gmres")


def legendre_map(p):
    """U dof -> Legendre coefficients on a cell (``spaces.py:45-57``): (p+1) x (p+1)."""
    m = p + 1
    r = np.zeros((m, m))
    r[0, 0], r[1, 0], r[0, 1], r[1, 1] = 0.5, -0.5, 0.5, 0.5
    for q in range(p - 1):
        r[q, 2 + q] = 1.0 / (2 * q + 3)
        r[q + 2, 2 + q] = -1.0 / (2 * q + 3)
    return r


def u_matrices_1d(widths, p):
    """Dense 1D stiffness and mass on the interior U dofs (``assembly.py:42-78``).

    Interior order: vertex hats 1..nc-1, then the p-1 bubbles of each cell
    (``spaces.py:25-43``); boundary hats are dropped (``restrict``).
    """
    widths = np.asarray(widths, dtype=float)
    nc, m = widths.size, p + 1
    nix = nc * p - 1
    R = legendre_map(p)
    K = np.zeros((nix, nix))
    M = np.zeros((nix, nix))
    for i, h in enumerate(widths):
        dofs = np.array([i - 1 if i >= 1 else -1, i if i <= nc - 2 else -1]
                        + [nc - 1 + i * (p - 1) + k for k in range(p - 1)])
        Kl = np.zeros((m, m))
        Kl[0, 0] = Kl[1, 1] = 1.0 / h
        Kl[0, 1] = Kl[1, 0] = -1.0 / h
        for k in range(p - 1):
            Kl[2 + k, 2 + k] = 4.0 / (h * (2 * k + 3))
        w = h / (2.0 * np.arange(m) + 1.0)
        Ml = R.T @ (w[:, None] * R)
        keep = dofs >= 0
        d = dofs[keep]
        K[np.ix_(d, d)] += Kl[np.ix_(keep, keep)]
        M[np.ix_(d, d)] += Ml[np.ix_(keep, keep)]
    return K, M


class DeviceStiffnessFactor:
    """``SpluFactor`` (``linalg.py:98-105``) for the 2D interior stiffness, on the GPU."""

    def __init__(self, disc):
        self.disc = disc
        p = disc.p
        Kx, Mx = u_matrices_1d(disc.hx, p)
        lx, Vx = sla.eigh(Kx, Mx)
        if np.array_equal(disc.hx, disc.hy):
            ly, Vy = lx, Vx
        else:
            Ky, My = u_matrices_1d(disc.hy, p)
            ly, Vy = sla.eigh(Ky, My)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (Vx, lx, Vy, ly)]
        _lib.call("hpgStiffnessFactor", disc.plan.handle,
                  *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs], _stream())
        self.n = disc.ndof_u

    def solve_t(self, b_t, out=None):
        d = self.disc
        d._check_len(b_t, self.n, "b")
        out = torch.empty(self.n, dtype=F64, device=d.device) if out is None else out
        _lib.call("hpgStiffnessSolve", d.plan.handle, _vp(b_t), _vp(out), _stream())
        return out

    def solve(self, b):
        d = self.disc
        x = self.solve_t(d.h2d(b, "stiff_b"), out=d._dev("stiff_x", self.n))
        return d.d2h(x, "stiff_x")


def factor_stiffness(disc):
    """``linalg.factor_stiffness(disc.A, ...)`` for a device discretisation."""
    return DeviceStiffnessFactor(disc)


class DeviceSchurOperator:
    """``SchurOperator`` (``linalg.py:213-229``): x -> -(D + E_beta + B^T (alpha A)^{-1} B) x.

    ``E`` is given as ``beta`` (``E_matrix(beta)``: diag(beta mass_psi) for the
    obstacle, beta x the per-cell spectral blocks for the gradient).
    """

    def __init__(self, disc, D, beta, alpha, A_factor=None):
        if not isinstance(D, DeviceCellBlockMatrix):
            raise TypeError("DeviceSchurOperator needs a device-backed D (disc.assemble_D)")
        if beta < 0:
            raise ValueError("beta must be >= 0")
        self.disc = disc
        self.D = D
        self.beta = float(beta)
        self.alpha = float(alpha)
        self.A_factor = A_factor if A_factor is not None else DeviceStiffnessFactor(disc)
        self.n = disc.ndof_psi

    def matvec_t(self, x_t, out=None):
        d = self.disc
        d._check_len(x_t, self.n, "x")
        out = torch.empty(self.n, dtype=F64, device=d.device) if out is None else out
        _lib.call("hpgSchurApply", d.plan.handle, _vp(self.D._w), self.alpha, self.beta, _vp(x_t),
                  _vp(out), _stream())
        return out

    def matvec(self, x):
        d = self.disc
        y = self.matvec_t(d.h2d(x, "schur_x"), out=d._dev("schur_y", self.n))
        return d.d2h(y, "schur_y")

    def __matmul__(self, x):
        return self.matvec(x)


def gmres_t(amul, b, M=None, side="right", x0=None, rtol=1e-8, atol=0.0, maxiter=150):
    """``linalg.gmres`` (``linalg.py:134-207``) on device vectors.

    ``amul`` / ``M``: callables on device tensors.  The Hessenberg matrix,
    rotations and the small triangular solve stay on the host (as in the
    reference); the Krylov basis, matvecs and orthogonalisation run on the
    GPU.  Returns ``GmresResult(x_t, iterations, residuals, converged)``.
    """
    pmul = (lambda v: v) if M is None else M
    n = b.numel()
    x = torch.zeros(n, dtype=F64, device=b.device) if x0 is None else x0.clone()
    if side not in ("left", "right"):
        raise ValueError("side must be 'left' or 'right'")
    r = b - amul(x) if bool(torch.any(x != 0)) else b.clone()
    if side == "left":
        r = pmul(r)
    beta = float(torch.linalg.vector_norm(r))
    residuals = [beta]
    if beta == 0.0:
        return GmresResult(x, 0, residuals, True)
    target = max(rtol * beta, atol)
    V = torch.empty((maxiter + 1, n), dtype=F64, device=b.device)
    V[0] = r / beta
    H = np.zeros((maxiter + 1, maxiter))
    cs = np.zeros(maxiter)
    sn = np.zeros(maxiter)
    g = np.zeros(maxiter + 1)
    g[0] = beta
    converged = False
    k = 0
    for j in range(maxiter):
        w = pmul(amul(V[j])) if side == "left" else amul(pmul(V[j]))
        hs = []
        for i in range(j + 1):                    # modified Gram-Schmidt
            h = torch.dot(V[i], w)
            w = w - h * V[i]
            hs.append(h)
        hs.append(torch.linalg.vector_norm(w))
        col = torch.stack(hs).cpu().numpy()
        H[: j + 2, j] = col
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        denom = np.hypot(H[j, j], H[j + 1, j])
        if denom == 0.0:
            cs[j], sn[j] = 1.0, 0.0
        else:
            cs[j] = H[j, j] / denom
            sn[j] = H[j + 1, j] / denom
        happy = H[j + 1, j] <= 1e-14 * max(1.0, abs(H[j, j]))
        H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        H[j + 1, j] = 0.0
        k = j + 1
        residuals.append(abs(g[j + 1]))
        if residuals[-1] <= target or happy:
            converged = True
            break
        V[j + 1] = w / col[-1]
    y = sla.solve_triangular(H[:k, :k], g[:k], lower=False)
    dx = torch.from_numpy(y).to(b.device) @ V[:k]
    if side == "right":
        dx = pmul(dx)
    x = x + dx
    if not converged and residuals[-1] <= target:
        converged = True
    return GmresResult(x, k, residuals, converged)


def schur_solve_t(disc, D, alpha, beta, b_u, b_psi, A_factor=None, rtol=1e-8, atol=0.0, maxiter=150,
                  side="right", precond=None):
    """``linalg.schur_solve`` (``linalg.py:269-287``) on device tensors."""
    A_factor = A_factor if A_factor is not None else DeviceStiffnessFactor(disc)
    S = DeviceSchurOperator(disc, D, beta, alpha, A_factor)
    y = b_psi - disc.BT_u_t(A_factor.solve_t(b_u)) / alpha
    if precond is None:
        precond = disc.schur_preconditioner(D, alpha, beta)
    res = gmres_t(S.matvec_t, y, M=precond.apply_t, side=side, rtol=rtol, atol=atol, maxiter=maxiter)
    dpsi = res.x
    du = A_factor.solve_t(b_u - disc.B_psi_t(dpsi)) / alpha
    return SchurSolveResult(du, dpsi, res)


def schur_solve(disc, D, alpha, beta, b_u, b_psi, A_factor=None, rtol=1e-8, atol=0.0, maxiter=150,
                side="right", precond=None):
    """NumPy in / NumPy out ``schur_solve``; ``gmres`` carries host residuals."""
    bu = torch.from_numpy(np.ascontiguousarray(b_u, dtype=np.float64)).to(disc.device)
    bp = torch.from_numpy(np.ascontiguousarray(b_psi, dtype=np.float64)).to(disc.device)
    r = schur_solve_t(disc, D, alpha, beta, bu, bp, A_factor, rtol, atol, maxiter, side, precond)
    g = GmresResult(r.gmres.x.cpu().numpy(), r.gmres.iterations, r.gmres.residuals, r.gmres.converged)
    return SchurSolveResult(r.du.cpu().numpy(), r.dpsi.cpu().numpy(), g)
