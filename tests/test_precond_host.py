"""CPU checks of the per-cell Schur preconditioner's host pieces.

* The reference-cell eigen-factors (tables.schur_triple_factors) reproduce
  the reference's dense hat triple Bhat^T Ahat^{-1} Bhat (assembly.py:577-595).
* The oracle's precond_blocks / CellBlockPreconditioner restatement matches
  the golden outputs of the unmodified reference (oracle/make_golden.py).
"""
from types import SimpleNamespace

import numpy as np
import pytest

from golden_util import load, names
from oracle import hpg_oracle as orc
from paper_2412_13733_b200.tables import schur_triple_factors

TOL = 1e-13


def eigen_triple(n, hx, hy):
    z, lam = schur_triple_factors(n)
    d = 1.0 / (hx ** 2 * lam[:, None] + hy ** 2 * lam[None, :])
    zz = np.kron(z, z)
    return (hx * hy) ** 3 * (zz * d.ravel()[None, :]) @ zz.T


@pytest.mark.parametrize("n,hx,hy", [(1, 0.5, 0.5), (3, 0.25, 0.25), (7, 0.25, 0.25),
                                     (15, 1 / 64, 1 / 64), (5, 0.15, 0.7), (24, 1 / 16, 1 / 16),
                                     (40, 1.0, 1.0)])
def test_triple_factors_match_dense_reference(n, hx, hy):
    ref = orc.schur_hat_triple(n, hx, hy)
    assert orc.rel_err(eigen_triple(n, hx, hy), ref) < 1e-14


def _problem(g):
    t = SimpleNamespace(S=g["S"], T=g["T"], Su=g["Su"], Tu=g["Tu"], xi=g["xi"], nq=g["nq"])
    return orc.Problem(g["kind"], g["xpts"], g["ypts"], g["p"], t)


@pytest.mark.parametrize("name", [n for n in names() if not n.startswith("c3")])
def test_oracle_precond_matches_reference(name):
    g = load(name)
    P = _problem(g)
    beta = float(g["prec_beta"])
    if "blocks" in g:
        blocks = g["blocks"]
    elif g["kind"] == "gradient":
        blocks = P.gradient_blocks(g["psi"], g["phi_values"].reshape(P.ncx, P.ncy, P.t.nq, P.t.nq))
    else:
        blocks, _ = P.obstacle_blocks(g["psi"])
    pb = np.stack(orc.precond_blocks(P, blocks, g["alpha"], beta))
    if np.isnan(g["psi"]).any():
        assert np.array_equal(np.isnan(pb), np.isnan(g["precond_blocks"]))
        assert "precond_error" in g          # scipy rejects non-finite blocks
        return
    if "precond_blocks" in g:
        assert orc.rel_err(pb, g["precond_blocks"]) < TOL
    else:
        assert orc.rel_err(pb[:, g["block_rows"], :], g["precond_sel"]) < TOL
    if np.isfinite(g["precond_apply"]).all():
        idx = orc.cell_psi_indices(P.ncx, P.ncy, P.n)
        if g["kind"] == "gradient":
            idx = [np.concatenate([i, i + P.ncomp_dofs]) for i in idx]
        y = orc.lu_precond_apply(pb, idx, P.ndof_psi, g["x"])
        assert orc.rel_err(y, g["precond_apply"]) < 1e-12
