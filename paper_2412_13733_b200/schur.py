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
* ``DeviceGmres`` / ``gmres_t`` -- ``gmres`` (``linalg.py:134-207``): the
  whole unrestarted, Givens-rotated iteration on the GPU as ONE CUDA graph
  with a device-side while loop (``hpgGmresSolve``, ``csrc/hpg_krylov.cu``):
  CGS2 Arnoldi, rotations, residual and stopping test on the device, the
  caller's operator kernels captured into the loop body; the reference's
  stopping rule and result fields.
* ``schur_solve``            -- ``schur_solve`` (``linalg.py:269-287``).

Every vector operation of the solve runs in the library's own kernels
(``hpgAxpby``, the stiffness solve's DMMA GEMMs): no cuBLAS, no ATen kernels.
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


def axpby_t(a, x, b, y, out):
    """out = a x + b y on device vectors (``hpgAxpby``)."""
    _lib.call("hpgAxpby", out.numel(), float(a), _vp(x), float(b), _vp(y), _vp(out), _stream())
    return out


class DeviceGmres:
    """``linalg.gmres`` (``linalg.py:134-207``) on the GPU for vectors of length n.

    ``solve(amul, b, M, side, x0, rtol, atol)``: ``amul(x, out)`` and
    ``M(x, out)`` enqueue device kernels writing ``out`` (no synchronisation,
    no allocation: they are captured into the loop body).  Returns the
    reference's ``GmresResult(x, iterations, residuals, converged)`` with x a
    device tensor; one host synchronisation per solve (the status read).
    """

    def __init__(self, n, maxiter, device):
        self.n, self.maxiter, self.device = int(n), int(maxiter), device
        h = ctypes.c_void_p()
        _lib.call("hpgGmresCreate", ctypes.byref(h), self.n, self.maxiter)
        self.handle = h
        mk = lambda: torch.zeros(self.n, dtype=F64, device=device)
        self.r, self.vin, self.z, self.w, self.dx = mk(), mk(), mk(), mk(), mk()
        _lib.call("hpgGmresBind", h, _vp(self.r), _vp(self.vin), _vp(self.w))
        self.stream = torch.cuda.Stream(device=device)     # captured: never the legacy stream
        self._lib = _lib.load()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.hpgGmresDestroy(h)
            except Exception:
                pass
            self.handle = None

    def solve(self, amul, b, M=None, side="right", x0=None, rtol=1e-8, atol=0.0):
        if side not in ("left", "right"):
            raise ValueError("side must be 'left' or 'right'")
        if b.numel() != self.n:
            raise ValueError(f"b has {b.numel()} entries, expected {self.n}")
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            # initial residual (linalg.py:149-152); A 0 = 0, so x0 = 0 gives r = b exactly
            if x0 is None:
                axpby_t(1.0, b, 0.0, None, self.r)
            else:
                amul(x0, self.w)
                axpby_t(1.0, b, -1.0, self.w, self.r)
            if side == "left" and M is not None:
                M(self.r, self.z)
                axpby_t(1.0, self.z, 0.0, None, self.r)
            s = _stream()
            _lib.call("hpgGmresCaptureBegin", self.handle, s)
            try:
                if M is None:
                    amul(self.vin, self.w)
                elif side == "right":
                    M(self.vin, self.z)
                    amul(self.z, self.w)
                else:
                    amul(self.vin, self.z)
                    M(self.z, self.w)
            finally:
                _lib.call("hpgGmresCaptureEnd", self.handle, s)
            _lib.call("hpgGmresSolve", self.handle, float(rtol), float(atol), _vp(self.dx), s)
            it, conv = ctypes.c_int(), ctypes.c_int()
            res = np.empty(self.maxiter + 1)
            _lib.call("hpgGmresStatus", self.handle, ctypes.byref(it), ctypes.byref(conv),
                      res.ctypes.data_as(ctypes.c_void_p), s)
            k = it.value
            x = torch.empty(self.n, dtype=F64, device=self.device)
            dx = self.dx
            if side == "right" and M is not None and k > 0:
                M(self.dx, self.z)
                dx = self.z
            if x0 is None:
                axpby_t(1.0, dx, 0.0, None, x)
            else:
                axpby_t(1.0, x0, 1.0, dx, x)
        cur.wait_stream(self.stream)
        return GmresResult(x, k, res[:k + 1].tolist(), bool(conv.value))


def gmres_t(amul, b, M=None, side="right", x0=None, rtol=1e-8, atol=0.0, maxiter=150):
    """One-shot ``DeviceGmres(...).solve`` (``linalg.gmres`` signature, device vectors)."""
    return DeviceGmres(b.numel(), maxiter, b.device).solve(amul, b, M, side, x0, rtol, atol)


def schur_solve_t(disc, D, alpha, beta, b_u, b_psi, A_factor=None, rtol=1e-8, atol=0.0, maxiter=150,
                  side="right", precond=None, gmres=None):
    """``linalg.schur_solve`` (``linalg.py:269-287``) on device tensors.

    ``gmres``: a reusable ``DeviceGmres`` for ``disc.ndof_psi`` unknowns."""
    A_factor = A_factor if A_factor is not None else DeviceStiffnessFactor(disc)
    S = DeviceSchurOperator(disc, D, beta, alpha, A_factor)
    # y = b_psi - B^T A^{-1} b_u / alpha
    y = disc.BT_u_t(A_factor.solve_t(b_u))
    axpby_t(1.0, b_psi, -1.0 / alpha, y, y)
    if precond is None:
        precond = disc.schur_preconditioner(D, alpha, beta)
    g = gmres if gmres is not None else DeviceGmres(disc.ndof_psi, maxiter, disc.device)
    if g.maxiter != maxiter:
        raise ValueError("gmres workspace was built for another maxiter")
    res = g.solve(lambda x, out: S.matvec_t(x, out=out), y, M=lambda x, out: precond.apply_t(x, out=out),
                  side=side, rtol=rtol, atol=atol)
    dpsi = res.x
    # du = A^{-1} (b_u - B dpsi) / alpha
    t = disc.B_psi_t(dpsi)
    axpby_t(1.0, b_u, -1.0, t, t)
    du = A_factor.solve_t(t)
    axpby_t(1.0 / alpha, du, 0.0, None, du)
    return SchurSolveResult(du, dpsi, res)


def schur_solve(disc, D, alpha, beta, b_u, b_psi, A_factor=None, rtol=1e-8, atol=0.0, maxiter=150,
                side="right", precond=None):
    """NumPy in / NumPy out ``schur_solve``; ``gmres`` carries host residuals."""
    bu = torch.from_numpy(np.ascontiguousarray(b_u, dtype=np.float64)).to(disc.device)
    bp = torch.from_numpy(np.ascontiguousarray(b_psi, dtype=np.float64)).to(disc.device)
    r = schur_solve_t(disc, D, alpha, beta, bu, bp, A_factor, rtol, atol, maxiter, side, precond)
    g = GmresResult(r.gmres.x.cpu().numpy(), r.gmres.iterations, r.gmres.residuals, r.gmres.converged)
    return SchurSolveResult(r.du.cpu().numpy(), r.dpsi.cpu().numpy(), g)
