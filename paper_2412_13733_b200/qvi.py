"""QVI temperature solve on the device (``hpgalerkin/qvi.py:35-127``).

``DeviceTemperatureSolver`` mirrors ``TemperatureSolver``: Newton on
``(grad T, grad q) + gamma (T, q) = (g(q_gap), q)`` over the FULL U space
(no Dirichlet condition), Jacobian actions matrix-free
(``H v - (g'(gap) xi v, q)``), GMRES left-preconditioned with ``H^{-1}``.
The per-cell U synthesis / analysis run as strided-batched DGEMMs with a
deterministic scatter (``hpgUFullOperator``), ``H^{-1}`` is a fast
diagonalisation (``hpgUFullSolve``) instead of SuperLU.  The problem data
(``data.g``, ``g_deriv``, ``mould``, ``xi``) are host callables, evaluated
on host copies of the point samples exactly as the reference does.
"""

import ctypes

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib
from .disc import F64, _stream, _vp
from .schur import DeviceGmres, legendre_map


def u_matrices_full_1d(widths, p):
    """Dense 1D stiffness and mass over ALL U dofs (``assembly.py:42-78``):
    hats 0..nc (vertex order), then the p-1 bubbles of each cell."""
    widths = np.asarray(widths, dtype=float)
    nc, m = widths.size, p + 1
    nf = nc * p + 1
    R = legendre_map(p)
    K = np.zeros((nf, nf))
    M = np.zeros((nf, nf))
    for i, h in enumerate(widths):
        d = np.array([i, i + 1] + [nc + 1 + i * (p - 1) + k for k in range(p - 1)])
        Kl = np.zeros((m, m))
        Kl[0, 0] = Kl[1, 1] = 1.0 / h
        Kl[0, 1] = Kl[1, 0] = -1.0 / h
        for k in range(p - 1):
            Kl[2 + k, 2 + k] = 4.0 / (h * (2 * k + 3))
        w = h / (2.0 * np.arange(m) + 1.0)
        K[np.ix_(d, d)] += Kl
        M[np.ix_(d, d)] += R.T @ (w[:, None] * R)
    return K, M


class DeviceTemperatureSolver:
    """``TemperatureSolver`` (``qvi.py:63-127``) on the GPU."""

    def __init__(self, disc, data, gmres_rtol=1.5e-8, newton_rtol=1e-9, newton_maxit=30):
        self.disc = disc
        self.data = data
        self.gmres_rtol = gmres_rtol
        self.newton_rtol = newton_rtol
        self.newton_maxit = newton_maxit
        self.gamma = float(data.gamma)
        p, t = disc.p, disc.tables
        R = legendre_map(p)
        inv = 1.0 / (2.0 * np.arange(p + 1) + 1.0)
        SR = t.Su @ R
        TR = R.T @ (inv[:, None] * t.Tu)
        Kh = np.zeros((p + 1, p + 1))
        Kh[0, 0] = Kh[1, 1] = 1.0
        Kh[0, 1] = Kh[1, 0] = -1.0
        for k in range(p - 1):
            Kh[2 + k, 2 + k] = 4.0 / (2 * k + 3)
        Mh = R.T @ (inv[:, None] * R)
        Kx, Mx = u_matrices_full_1d(disc.hx, p)
        lx, Vx = sla.eigh(Kx, Mx)
        if np.array_equal(disc.hx, disc.hy):
            ly, Vy = lx, Vx
        else:
            Ky, My = u_matrices_full_1d(disc.hy, p)
            ly, Vy = sla.eigh(Ky, My)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (SR, TR, Kh, Mh, Vx, lx, Vy, ly)]
        _lib.call("hpgUFullSetup", disc.plan.handle, self.gamma,
                  *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs], _stream())
        self.nfull = (disc.ncx * p + 1) * (disc.ncy * p + 1)
        self.nq = t.nq
        dev = disc.device
        grids = disc.quad_grids()
        phi0, xi = [], []
        for X, Y in grids:
            XX, YY = np.meshgrid(X, Y, indexing="ij")
            phi0.append(data.mould(XX, YY))
            xi.append(data.xi(XX, YY))
        self.phi0_vals = torch.from_numpy(np.ascontiguousarray(np.stack(phi0), dtype=np.float64)).to(dev)
        self.xi_vals = torch.from_numpy(np.ascontiguousarray(np.stack(xi), dtype=np.float64)).to(dev)

    # -- the reference's module helpers (qvi.py:35-60) on device vectors
    def values_t(self, full_t):
        """``_cell_grid_values``: (ncells, nq, nq) samples of a full U vector."""
        d = self.disc
        out = torch.empty((d.plan.ncells, self.nq, self.nq), dtype=F64, device=d.device)
        _lib.call("hpgUFullValues", d.plan.handle, _vp(full_t), _vp(out), _stream())
        return out

    def load_t(self, vals_t):
        """``_load_full``: moments against every U basis function."""
        d = self.disc
        out = torch.empty(self.nfull, dtype=F64, device=d.device)
        _lib.call("hpgUFullOperator", d.plan.handle, self.gamma, None, None, _vp(vals_t), _vp(out), _stream())
        return -out

    def operator_t(self, v_t, w_t=None, rhs_t=None, out=None):
        """``H v - load(w .* values(v) + rhs)``."""
        d = self.disc
        out = torch.empty(self.nfull, dtype=F64, device=d.device) if out is None else out
        _lib.call("hpgUFullOperator", d.plan.handle, self.gamma, _vp(v_t), _vp(w_t), _vp(rhs_t), _vp(out),
                  _stream())
        return out

    def precond_t(self, b_t, out=None):
        """``H^{-1} b`` (the reference's ``splu(H).solve``)."""
        d = self.disc
        out = torch.empty(self.nfull, dtype=F64, device=d.device) if out is None else out
        _lib.call("hpgUFullSolve", d.plan.handle, _vp(b_t), _vp(out), _stream())
        return out

    def _host_map(self, fn, vals_t):
        return torch.from_numpy(np.ascontiguousarray(fn(vals_t.cpu().numpy()), dtype=np.float64)).to(vals_t.device)

    def _gmres(self):
        """One device GMRES workspace per solver (the reference's default maxiter, linalg.py:135)."""
        if getattr(self, "_gm", None) is None:
            self._gm = DeviceGmres(self.nfull, 150, self.disc.device)
        return self._gm

    def _residual_t(self, T, u_vals):
        gap = self.phi0_vals + self.xi_vals * self.values_t(T) - u_vals
        r = self.operator_t(T, None, self._host_map(self.data.g, gap))
        return r, gap

    def solve(self, u_full, T0=None):
        """Returns (T, newton_iters, gmres_iters_list) as the reference."""
        d = self.disc
        u_t = torch.from_numpy(np.ascontiguousarray(u_full, dtype=np.float64)).to(d.device)
        u_vals = self.values_t(u_t)
        T = (torch.zeros(self.nfull, dtype=F64, device=d.device) if T0 is None
             else torch.from_numpy(np.array(T0, dtype=np.float64)).to(d.device))
        r, gap = self._residual_t(T, u_vals)
        norm0 = float(torch.linalg.vector_norm(r))
        target = max(self.newton_rtol * norm0, 1e-14)
        gmres_its = []
        newton = 0
        while float(torch.linalg.vector_norm(r)) > target and newton < self.newton_maxit:
            gp = self._host_map(self.data.g_deriv, gap) * self.xi_vals

            def jmul(v, out, gp=gp):
                return self.operator_t(v, gp, out=out)

            res = self._gmres().solve(jmul, r, M=self.precond_t, side="left", rtol=self.gmres_rtol, atol=0.0)
            T = T - res.x
            gmres_its.append(res.iterations)
            newton += 1
            r, gap = self._residual_t(T, u_vals)
        return T.cpu().numpy(), newton, gmres_its
