"""CPU checks of the Schur solve's host pieces.

The 1D interior stiffness/mass (schur.u_matrices_1d) reproduce the
reference's A = kron(Ax, My) + kron(Mx, Ay) (assembly.py:42-78, 470-474):
a dense solve and the fast-diagonalisation solve (the device algorithm,
restated in NumPy) both match the reference's SuperLU solution stored in the
golden fixtures.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from golden_util import load, names
from oracle.hpg_oracle import rel_err
from paper_2412_13733_b200.schur import u_matrices_1d

SMALL = [n for n in names() if not n.startswith("c3") and n not in ("clamp_ref", "nan_ref")]


@pytest.mark.parametrize("name", SMALL)
def test_stiffness_matches_reference(name):
    g = load(name)
    p = g["p"]
    Kx, Mx = u_matrices_1d(np.diff(g["xpts"]), p)
    Ky, My = u_matrices_1d(np.diff(g["ypts"]), p)
    b = g["u"]
    ref = g["stiff_solve"]
    if Kx.shape[0] * Ky.shape[0] <= 3000:
        A = np.kron(Kx, My) + np.kron(Mx, Ky)
        assert rel_err(np.linalg.solve(A, b), ref) < 1e-12
    lx, Vx = sla.eigh(Kx, Mx)
    ly, Vy = sla.eigh(Ky, My)
    B = b.reshape(Kx.shape[0], Ky.shape[0])
    X = Vx @ ((Vx.T @ B @ Vy) / (lx[:, None] + ly[None, :])) @ Vy.T
    assert rel_err(X.ravel(), ref) < 1e-12
