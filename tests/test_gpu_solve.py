"""The whole LVPP penalty continuation on the GPU vs the reference's
proximal.solve (golden fixtures in tests/golden/solve, oracle/make_golden.py).

Same alpha schedule, options and stopping rules: the Newton iteration count
of every continuation step and the GMRES totals must match, the final state
(u, psi, multiplier) agrees to the Newton tolerance scale.
"""
import numpy as np
import pytest

from golden_util import load_solve, solve_names
from oracle.hpg_oracle import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", solve_names())
def test_continuation_matches_reference(name):
    from paper_2412_13733_b200 import disc as D, proximal
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    from paper_2412_13733_b200.workloads import phi_sin
    g = load_solve(name)
    mesh = TensorMesh2D(Mesh1D(g["xpts"], np.full(g["xpts"].size - 1, g["p"])),
                        Mesh1D(g["ypts"], np.full(g["ypts"].size - 1, g["p"])))
    d = D.ObstacleDisc2D(mesh, 1.0, phi_sin, rule=g["rule"], nq=g["nq"] if g["rule"] == "gauss" else None)
    sched = proximal.AlphaSchedule(alpha0=1.0, rate=2.0, alpha_max=g["alpha_max"])
    rep = proximal.solve(d, sched, g["beta"], proximal.SolverOptions(line_search=g["line_search"]))
    assert rep.converged == g["converged"]
    assert [s.newton_iters for s in rep.steps] == g["newton_iters"].tolist()
    gm = np.array([s.gmres_total for s in rep.steps])
    assert np.abs(gm - g["gmres_iters"]).max() <= 1
    assert rel_err(rep.u, g["u"]) < 1e-9
    assert rel_err(rep.psi, g["psi"]) < 1e-9
    assert rel_err(rep.multiplier, g["multiplier"]) < 1e-8
