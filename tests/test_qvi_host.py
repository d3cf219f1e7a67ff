"""CPU pin of the QVI full-space U matrices (qvi.py:76-81, assembly.py:42-78):
H = kron(Ax, My) + kron(Mx, Ay) + gamma kron(Mx, My) built from
qvi.u_matrices_full_1d reproduces the reference's H v (golden fixtures)."""
import numpy as np
import pytest

from golden_util import load_qvi, qvi_names
from oracle.hpg_oracle import rel_err
from paper_2412_13733_b200.qvi import u_matrices_full_1d


@pytest.mark.parametrize("name", qvi_names())
def test_full_space_H(name):
    g = load_qvi(name)
    Kx, Mx = u_matrices_full_1d(np.diff(g["xpts"]), g["p"])
    Ky, My = u_matrices_full_1d(np.diff(g["ypts"]), g["p"])
    H = np.kron(Kx, My) + np.kron(Mx, Ky) + g["gamma"] * np.kron(Mx, My)
    assert rel_err(H @ g["vfull"], g["Hv"]) < 1e-13
