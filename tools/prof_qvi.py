"""Time the device QVI temperature solve at the paper's setting (4x4 mesh,
high degree).

    python tools/prof_qvi.py [p] [Q]

Membrane displacement: a seeded interior field extended by zero to the
boundary (as qvi.thermoform_solve feeds the temperature step).
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_2412_13733_b200 import disc as D                    # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d           # noqa: E402
from paper_2412_13733_b200.qvi import DeviceTemperatureSolver    # noqa: E402
from qvi_data import ThermoformingData                           # noqa: E402


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 82
    Q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    data = ThermoformingData()
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, 4, p), data.f, 0.0, rule="gauss", nq=Q)
    t0 = time.perf_counter()
    s = DeviceTemperatureSolver(d, data)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    nf1 = 4 * p + 1
    rng = np.random.default_rng(3)
    U = np.zeros((nf1, nf1))
    U[1:4 * 1, :] = 0.0
    inner = 0.05 * rng.standard_normal((nf1, nf1)) / (1.0 + np.add.outer(np.arange(nf1), np.arange(nf1)))
    inner[[0, 4], :] = 0.0
    inner[:, [0, 4]] = 0.0
    s.solve(inner.ravel())                      # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T, newton, gm = s.solve(inner.ravel())
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    v = torch.from_numpy(inner.ravel()).cuda()
    w = torch.rand((d.plan.ncells, Q, Q), dtype=torch.float64, device="cuda")

    def per_call(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts)) * 1e3

    t_j = per_call(lambda: s.operator_t(v, w))
    t_p = per_call(lambda: s.precond_t(v))
    print(f"QVI temperature 4x4 p={p} Q={Q}: nfull={s.nfull}  setup {t_setup:.2f} s (host eigh)  "
          f"solve {t * 1e3:.1f} ms (newton {newton}, gmres {gm})  Jacobian apply {t_j:.3f} ms  "
          f"H^-1 {t_p:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
