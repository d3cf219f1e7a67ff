"""BASELINE.json configurations and their seeded synthetic inputs.

There is no public dataset for this path; BASELINE.json's five configs define
synthetic inputs.  One ``np.random.default_rng(seed)`` stream is drawn in the
order psi (component x, then y), u, x (direction), then config 3's obstacle
coefficients:

* psi: per cell and component, the n x n Legendre tile c_ij ~ N(0,1)/(1+i+j)^2
  with (i, j) the local Legendre indices, stored in the global x-major tensor
  order of ``PsiSpace2D`` (``hpgalerkin/spaces.py:212-214``);
* u: interior U dof (gx, gy) ~ N(0,1)/(1+lx+ly)^2 with l the 1D polynomial
  degree of the dof (hat -> 1, bubble W_k -> k+2);
* x: N(0,1) per psi dof; psi_prev = 0 (LVPP psi_0 = 0); f = 1.
"""

from dataclasses import dataclass, field

import numpy as np

from .tables import legendre_table


def phi_sin(x, y):
    return 0.2 + 0.1 * np.sin(np.pi * x) * np.sin(np.pi * y)


def phi_bilinear(x, y):
    return 0.5 + 0.25 * x * y


class LegendreSeriesObstacle:
    """phi(x, y) = 1 + sum_{i,j<=deg} a_ij P_i(2x-1) P_j(2y-1) (config 3)."""

    def __init__(self, coeffs):
        self.a = np.asarray(coeffs, dtype=float)

    def __call__(self, x, y):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        d = self.a.shape[0] - 1
        Px = legendre_table(d, 2.0 * x - 1.0)
        Py = legendre_table(d, 2.0 * y - 1.0)
        return 1.0 + np.einsum("ij,i...,j...->...", self.a, Px, Py)


@dataclass
class Config:
    name: str
    kind: str            # "obstacle" | "gradient"
    ncells: int          # per direction
    p: int
    Q: int               # Gauss points per direction (BASELINE.json)
    alphas: tuple
    k_mv: int            # Jacobian matvecs per residual
    reps: int = 1
    phi: str = "sin"
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.p - 1 if self.kind == "obstacle" else self.p

    @property
    def ncomp(self):
        return 1 if self.kind == "obstacle" else 2

    @property
    def N(self):
        return self.ncells * self.ncells

    def nq(self, rule):
        return 2 * (self.p + 1) if rule == "reference" else self.Q


CONFIGS = {
    "c0": Config("c0", "obstacle", 4, 8, 12, (1.0,), 1),
    "c1": Config("c1", "obstacle", 64, 16, 24, (1.0, 4.0, 16.0), 50),
    "c2": Config("c2", "gradient", 16, 24, 36, (1.0,), 1, phi="bilinear"),
    "c3": Config("c3", "obstacle", 4, 82, 128, (1.0,), 1, phi="series"),
    "c4p2": Config("c4p2", "obstacle", 256, 2, 5, (4.0,), 1, reps=100),
    "c4p4": Config("c4p4", "obstacle", 256, 4, 7, (4.0,), 1, reps=100),
    "c4p6": Config("c4p6", "obstacle", 256, 6, 9, (4.0,), 1, reps=100),
}


def u_dof_degrees_1d(ncells, p):
    """1D polynomial degree of each *interior* U dof (hats first, then bubbles)."""
    hats = np.ones(ncells - 1)
    bub = np.tile(np.arange(p - 1) + 2.0, ncells)
    return np.concatenate([hats, bub])


def make_inputs(kind, ncells_x, ncells_y, p, seed=0, series_phi=False):
    """Seeded (psi, u, x, phi) for a uniform-degree mesh."""
    rng = np.random.default_rng(seed)
    n = p - 1 if kind == "obstacle" else p
    ncomp = 1 if kind == "obstacle" else 2
    ix = np.arange(ncells_x * n) % n
    iy = np.arange(ncells_y * n) % n
    decay = (1.0 / (1.0 + ix[:, None] + iy[None, :]) ** 2).ravel()
    comps = [rng.standard_normal(decay.size) * decay for _ in range(ncomp)]
    psi = np.concatenate(comps)
    lx = u_dof_degrees_1d(ncells_x, p)
    ly = u_dof_degrees_1d(ncells_y, p)
    udecay = (1.0 / (1.0 + lx[:, None] + ly[None, :]) ** 2).ravel()
    u = rng.standard_normal(udecay.size) * udecay
    x = rng.standard_normal(psi.size)
    phi = None
    if series_phi:
        phi = LegendreSeriesObstacle(rng.normal(0.0, 0.1, size=(11, 11)))
    return psi, u, x, phi


def config_inputs(cfg, seed=0, ncells=None):
    """Inputs and data callables for a named config (optionally on a smaller mesh)."""
    nc = cfg.ncells if ncells is None else ncells
    psi, u, x, series = make_inputs(cfg.kind, nc, nc, cfg.p, seed=seed,
                                    series_phi=(cfg.phi == "series"))
    if cfg.phi == "sin":
        phi = phi_sin
    elif cfg.phi == "bilinear":
        phi = phi_bilinear
    else:
        phi = series
    return dict(psi=psi, u=u, x=x, psi_prev=np.zeros_like(psi), phi=phi, f=1.0)
