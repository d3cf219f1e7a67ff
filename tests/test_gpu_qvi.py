"""GPU parity of the QVI temperature operators and solve
against the reference's qvi.py (golden fixtures, oracle/make_golden.py)."""
import numpy as np
import pytest

from golden_util import load_qvi, qvi_names
from oracle.hpg_oracle import rel_err
from qvi_data import ThermoformingData

pytestmark = pytest.mark.gpu
TOL = 1e-12


def solver_for(g):
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    from paper_2412_13733_b200.qvi import DeviceTemperatureSolver
    data = ThermoformingData(load=g["load"])
    mesh = TensorMesh2D(Mesh1D(g["xpts"], np.full(g["xpts"].size - 1, g["p"])),
                        Mesh1D(g["ypts"], np.full(g["ypts"].size - 1, g["p"])))
    d = D.ObstacleDisc2D(mesh, data.f, 0.0, rule=g["rule"], nq=g["nq"] if g["rule"] == "gauss" else None)
    return DeviceTemperatureSolver(d, data)


@pytest.mark.parametrize("name", qvi_names())
def test_qvi_operators(name):
    import torch
    g = load_qvi(name)
    s = solver_for(g)
    v = torch.from_numpy(g["vfull"]).cuda()
    assert rel_err(s.values_t(v).cpu().numpy(), g["vals"]) < TOL
    assert rel_err(s.load_t(torch.from_numpy(g["rvals"]).cuda()).cpu().numpy(), g["load_full"]) < TOL
    Hv = s.operator_t(v).cpu().numpy()
    assert rel_err(Hv, g["Hv"]) < TOL
    # H^{-1} (fast diagonalisation) inverts H
    x = s.precond_t(torch.from_numpy(g["Hv"]).cuda()).cpu().numpy()
    assert rel_err(x, g["vfull"]) < 1e-10


@pytest.mark.parametrize("name", qvi_names())
def test_temperature_solve(name):
    g = load_qvi(name)
    s = solver_for(g)
    T, newton, gmres_its = s.solve(g["u_full"])
    assert newton == g["newton"]
    assert gmres_its == g["gmres"].tolist()
    assert rel_err(T, g["temp"]) < 1e-9
