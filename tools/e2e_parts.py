"""Host-API timing pieces of the c1 e2e step: D @ x (NumPy in/out) and the
residual with host buffers; transfer strategy comparison on the same vector."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.proximal import residual  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
inp = config_inputs(cfg)
d = (D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D)(
    uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
Dm = d.assemble_D(inp["psi"])
x = inp["x"]


def timeit(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:50s} {dt*1e3:8.3f} ms", flush=True)


timeit("D @ x (hpgApplyCachedHost)", lambda: Dm @ x)
timeit("h2d(x) + apply_cached_t + d2h (staged torch)", lambda: d.d2h(Dm.matvec_t(d.h2d(x, "x")), "y"))
timeit("h2d(x) only", lambda: d.h2d(x, "x"))
y = Dm.matvec_t(d.h2d(x, "x"))
timeit("d2h(y) only", lambda: d.d2h(y, "y"))
timeit("apply_cached_t only", lambda: Dm.matvec_t(y))
timeit("np.empty + fill (page faults)", lambda: np.empty(x.size).fill(1.0))
timeit("residual (host buffers)", lambda: residual(d, 1.0, inp["psi_prev"], inp["u"], inp["psi"]))
timeit("assemble_D (host psi)", lambda: d.assemble_D(inp["psi"]))
