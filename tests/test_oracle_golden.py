"""Pin the CPU oracle (and the product's table provider) to the reference's outputs.

The golden fixtures come from the unmodified reference package
(``oracle/make_golden.py``); this file needs no GPU and no reference install.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from golden_util import load, names
from oracle import hpg_oracle as orc
from paper_2412_13733_b200.tables import Tables

TOL = 1e-13   # oracle vs reference: pure fp64 reordering noise (~1e-15 seen)


def problem(g):
    t = SimpleNamespace(S=g["S"], T=g["T"], Su=g["Su"], Tu=g["Tu"], xi=g["xi"], nq=g["nq"])
    return orc.Problem(g["kind"], g["xpts"], g["ypts"], g["p"], t)


@pytest.mark.parametrize("name", names())
def test_product_tables_bitwise(name):
    g = load(name)
    n = g["p"] - 1 if g["kind"] == "obstacle" else g["p"]
    t = Tables(g["rule"], g["p"], n, g["nq"])
    for k in ("S", "T", "Su", "Tu", "xi"):
        assert np.array_equal(getattr(t, k), g[k]), k


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference(name):
    g = load(name)
    P = problem(g)
    nan_case = np.isnan(g["psi"]).any()
    if g["kind"] == "obstacle":
        m, cl = P.exp_moments(g["psi"])
        assert cl == g["clamped"]
        phi_vals = None
        phi_mom = g["phi_moments"]
    else:
        phi_vals = g["phi_values"].reshape(P.ncx, P.ncy, P.t.nq, P.t.nq)
        m = P.nl_moments(g["psi"], phi_vals)
        phi_mom = None
    if nan_case:
        assert np.array_equal(np.isnan(m), np.isnan(g["moments"]))
        return
    assert orc.rel_err(m, g["moments"]) < TOL
    b_u, b_psi, cl = P.residual(g["alpha"], g["psi_prev"], g["u"], g["psi"],
                                g["f_load"], phi_moments=phi_mom, phi_vals=phi_vals)
    assert cl == g["res_clamped"]
    assert orc.rel_err(b_u, g["b_u"]) < TOL
    assert orc.rel_err(b_psi, g["b_psi"]) < TOL
    if g["kind"] == "obstacle":
        y = P.obstacle_apply_D(g["psi"], g["x"])
        blocks, bcl = P.obstacle_blocks(g["psi"])
        assert bcl == g["D_clamped"]
    else:
        y = P.gradient_apply_D(g["psi"], g["x"], phi_vals)
        blocks = P.gradient_blocks(g["psi"], phi_vals)
    assert orc.rel_err(y, g["apply_D"]) < TOL
    assert orc.rel_err(y, g["Dx"]) < TOL
    if "blocks" in g:
        assert orc.rel_err(blocks, g["blocks"]) < TOL
    else:
        assert orc.rel_err(blocks[:, g["block_rows"], :], g["blocks_sel"]) < TOL


@pytest.mark.parametrize("name", ["c0_ref", "c0_gauss", "nonuni_ref", "c4p4_gauss"])
def test_oracle_data_terms(name):
    """phi moments and f_load from point samples (assembly.py:492,502-519)."""
    from paper_2412_13733_b200.workloads import phi_sin
    g = load(name)
    P = problem(g)
    assert orc.rel_err(P.data_moments(P.sample(phi_sin)), g["phi_moments"]) < TOL
    assert orc.rel_err(P.load_vector(P.sample(1.0)), g["f_load"]) < TOL


def test_clamp_truth_table():
    """SURVEY.md §7 measured truth table of _clamped_exp_neg."""
    cases = [(-800.0, np.exp(700.0), True), (-700.0, np.exp(700.0), False),
             (-700.0000001, np.exp(700.0), True), (np.inf, 0.0, False),
             (-np.inf, np.exp(700.0), True)]
    for v, val, flag in cases:
        e, f = orc.clamped_exp_neg(np.array([v]))
        assert f == flag and e[0] == val
    e, f = orc.clamped_exp_neg(np.array([np.nan]))
    assert f and np.isnan(e[0])
