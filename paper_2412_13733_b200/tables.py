"""Per-direction quadrature tables (host side, built once per discretisation).

Every device kernel is table-driven: a synthesis table ``S`` (nq x n, the
Legendre polynomials P_0..P_{n-1} evaluated at the nq reference points), a
truncated analysis table ``T`` (n x nq) and, for the U side, the same pair
with p+1 columns (``Su``, ``Tu``).  The per-cell mass weights
``w_i = h / (2 i + 1)`` are formed on the device from the cell width.

Two rules are provided:

* ``rule="reference"`` -- the reference's projection quadrature on
  ``nq = 2 (p + 1)`` Chebyshev-Lobatto points
  (``hpgalerkin/assembly.py:198-207``, ``transforms.py:30-36,137-168``).
  The tables are produced by the same sequence of floating-point operations
  as the reference (DCT-I of the reversed identity, Gauss-Legendre
  connection matrix, three-term Legendre recurrence), so they are
  bit-for-bit the reference's arrays; ``tests/test_tables.py`` pins that
  against golden copies.  Bitwise identity matters: a different but equally
  valid analysis matrix moves p=82 moments by ~1e-12 (SURVEY.md finding 9).
* ``rule="gauss"`` -- Q-point Gauss-Legendre quadrature (BASELINE.json's
  configs): ``S[g, j] = P_j(xi_g)``, ``T[i, g] = (2i+1)/2 * omega_g * P_i(xi_g)``.
"""

from functools import lru_cache

import numpy as np
from numpy.polynomial import chebyshev as npcheb
from numpy.polynomial import legendre as npleg
from scipy.fft import dct


def legendre_table(nmax, x):
    """P_0..P_nmax at x (shape (nmax+1,) + x.shape), zero outside [-1, 1].

    Same recurrence and operation order as ``hpgalerkin/basis.py:29-45``.
    """
    x = np.asarray(x, dtype=float)
    inside = (x >= -1.0) & (x <= 1.0)
    out = np.zeros((nmax + 1,) + x.shape)
    out[0] = np.where(inside, 1.0, 0.0)
    if nmax >= 1:
        out[1] = np.where(inside, x, 0.0)
    for k in range(1, nmax):
        out[k + 1] = ((2 * k + 1) * x * out[k] - k * out[k - 1]) / (k + 1)
    if nmax >= 1:
        out[1:, ~inside] = 0.0
    return out


def lobatto_points(q):
    """Chebyshev points of the second kind, ascending (``transforms.py:30-36``)."""
    if q < 1:
        raise ValueError("need at least one point")
    if q == 1:
        return np.zeros(1)
    return -np.cos(np.pi * np.arange(q) / (q - 1))


def _values_to_chebyshev(v):
    """Chebyshev interpolation coefficients via DCT-I (``transforms.py:39-53``)."""
    q = v.shape[0]
    if q == 1:
        return v.copy()
    c = dct(v[::-1], type=1, axis=0) / (q - 1)
    c[0] *= 0.5
    c[-1] *= 0.5
    return c


@lru_cache(maxsize=None)
def _chebyshev_to_legendre(q):
    """(2j+1)/2 * int P_j T_k by (q+1)-point Gauss rule (``transforms.py:68-82``)."""
    nodes, weights = npleg.leggauss(q + 1)
    P = legendre_table(q - 1, nodes)
    Tch = npcheb.chebvander(nodes, q - 1).T
    M = (P * weights) @ Tch.T
    M *= ((2.0 * np.arange(q) + 1.0) / 2.0)[:, None]
    return M


@lru_cache(maxsize=None)
def lobatto_analysis(q):
    """Full (q, q) interpolation->Legendre analysis matrix (``transforms.py:137-160``)."""
    eye = np.eye(q)
    c = _values_to_chebyshev(eye)
    A = _chebyshev_to_legendre(q) @ c.reshape(q, -1)
    A = A.reshape(eye.shape)
    A.flags.writeable = False
    return A


@lru_cache(maxsize=None)
def lobatto_synthesis(q, ncoeff):
    S = legendre_table(ncoeff - 1, lobatto_points(q)).T.copy()
    S.flags.writeable = False
    return S


@lru_cache(maxsize=None)
def gauss_rule(q):
    xi, om = npleg.leggauss(q)
    xi.flags.writeable = False
    om.flags.writeable = False
    return xi, om


def gauss_synthesis(q, ncoeff):
    xi, _ = gauss_rule(q)
    return legendre_table(ncoeff - 1, xi).T.copy()


def gauss_analysis(q, ncoeff):
    xi, om = gauss_rule(q)
    P = legendre_table(ncoeff - 1, xi)
    return ((2.0 * np.arange(ncoeff) + 1.0) / 2.0)[:, None] * P * om[None, :]


@lru_cache(maxsize=None)
def schur_triple_factors(n):
    """Reference-cell factors of the Schur hat triple (``assembly.py:577-595``).

    On a cell the triple is ``Bhat^T Ahat^{-1} Bhat`` with ``Bhat = gx (x) gy``
    and ``Ahat = Kx (x) My + Mx (x) Ky`` (spectral Gram ``assembly.py:156-170``,
    stiffness diagonal ``:147-153``, pentadiagonal mass ``:128-144``; n modes
    per direction).  With ``g = h ghat``, ``K = khat / h``, ``M = h mhat`` and
    ``khat^{-1/2} mhat khat^{-1/2} = V diag(lam) V^T``:

        T[(a,b),(c,d)] = (hx hy)^3 sum_ij Z[a,i] Z[b,j] Z[c,i] Z[d,j]
                                       / (hx^2 lam_i + hy^2 lam_j),
        Z = ghat^T khat^{-1/2} V.

    Returns ``(Z, lam)`` (n x n row-major, n); the device forms T per width key.
    Agrees with the reference's dense ``np.linalg.solve`` to <= 8e-16 relative
    for n <= 81 (tests/test_precond_host.py).
    """
    g = np.zeros((n, n))
    k = np.zeros(n)
    m = np.zeros((n, n))
    for a in range(n):
        g[a, a] = 1.0 / (2 * a + 1)
        k[a] = 4.0 * (2 * a + 3)
        m[a, a] = 1.0 / (2 * a + 1) + 1.0 / (2 * a + 5)
        if a + 2 < n:
            g[a, a + 2] = -1.0 / (2 * a + 5)
            m[a, a + 2] = m[a + 2, a] = -1.0 / (2 * a + 5)
    ki = 1.0 / np.sqrt(k)
    lam, v = np.linalg.eigh(ki[:, None] * m * ki[None, :])
    z = g.T @ (ki[:, None] * v)
    return np.ascontiguousarray(z), np.ascontiguousarray(lam)


class Tables:
    """The per-direction tables of one uniform-degree discretisation.

    ``p`` is the U degree, ``n`` the psi tile side (p-1 obstacle, p gradient).
    Arrays are C-contiguous float64 and shared by every cell of the mesh.
    """

    def __init__(self, rule, p, n, nq=None):
        if rule not in ("reference", "gauss"):
            raise ValueError(f"unknown quadrature rule {rule!r}")
        if n < 1:
            raise ValueError("psi tile side must be >= 1")
        self.rule = rule
        self.p = int(p)
        self.n = int(n)
        self.m = int(p) + 1
        if rule == "reference":
            nq_ref = 2 * (self.p + 1)
            if nq is not None and int(nq) != nq_ref:
                raise ValueError(f"reference rule fixes nq = 2(p+1) = {nq_ref}")
            self.nq = nq_ref
            A = lobatto_analysis(self.nq)
            self.S = np.ascontiguousarray(lobatto_synthesis(self.nq, self.n))
            self.T = np.ascontiguousarray(A[:self.n])
            self.Su = np.ascontiguousarray(lobatto_synthesis(self.nq, self.m))
            self.Tu = np.ascontiguousarray(A[:self.m])
            self.xi = lobatto_points(self.nq)
        else:
            if nq is None:
                raise ValueError("gauss rule needs the number of points nq")
            self.nq = int(nq)
            if self.nq < 1:
                raise ValueError("need at least one quadrature point")
            self.S = gauss_synthesis(self.nq, self.n)
            self.T = np.ascontiguousarray(gauss_analysis(self.nq, self.n))
            self.Su = gauss_synthesis(self.nq, self.m)
            self.Tu = np.ascontiguousarray(gauss_analysis(self.nq, self.m))
            self.xi = np.array(gauss_rule(self.nq)[0])

    def points(self, x0, x1):
        """Physical points of a cell [x0, x1] (``assembly.py:207``)."""
        return 0.5 * (x0 + x1) + 0.5 * (x1 - x0) * self.xi

    def __repr__(self):
        return f"Tables(rule={self.rule!r}, p={self.p}, n={self.n}, nq={self.nq})"
