import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2412_13733_b200 import disc as D
from paper_2412_13733_b200.mesh import uniform_mesh_2d
from paper_2412_13733_b200.proximal import residual
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs
cfg = CONFIGS["c1"]; inp = config_inputs(cfg)
d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
hp = {k: np.ascontiguousarray(inp[k]) for k in ("psi", "psi_prev", "u", "x")}
for s in range(4):
    t0 = time.perf_counter()
    residual(d, 1.0, hp["psi_prev"], hp["u"], hp["psi"]); t1 = time.perf_counter()
    Dm = d.assemble_D(hp["psi"]); t2 = time.perf_counter()
    for _ in range(50):
        Dm @ hp["x"]
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"residual {1e3*(t1-t0):.2f} assemble {1e3*(t2-t1):.2f} 50 matvec {1e3*(t3-t2):.2f} total {1e3*(t3-t0):.2f}")
ts = []
for _ in range(200):
    t0 = time.perf_counter(); y = Dm @ hp["x"]; ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e3
print("per-call ms: min %.3f median %.3f mean %.3f p90 %.3f max %.3f" % (ts.min(), np.median(ts), ts.mean(), np.percentile(ts, 90), ts.max()))
