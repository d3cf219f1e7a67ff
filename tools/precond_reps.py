import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2412_13733_b200 import disc as D
from paper_2412_13733_b200.disc import DeviceCellBlockPreconditioner
from paper_2412_13733_b200.mesh import uniform_mesh_2d
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs
cfg = CONFIGS["c1"]; inp = config_inputs(cfg)
d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
t = {k: torch.from_numpy(inp[k]).cuda() for k in ("psi", "psi_prev", "u", "x")}
alpha, beta = cfg.alphas[-1], 1e-8
d.residual_t(alpha, t["psi_prev"], t["u"], t["psi"], wcache=True)
Dm = d.assemble_D_t(t["psi"])
M = None
for rep in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    M = DeviceCellBlockPreconditioner.from_operator(d, Dm, alpha, beta)
    e1.record()
    torch.cuda.synchronize()
    print(rep, "gpu %.2f ms" % e0.elapsed_time(e1), "wall %.2f ms" % ((time.perf_counter() - t0) * 1e3), "reserved %.1f GB" % (torch.cuda.memory_reserved() / 1e9))
# the same after an e2e-like phase (host buffers, page-locked results) and a 1.7 GB scratch allocation
from paper_2412_13733_b200.proximal import residual
from paper_2412_13733_b200.disc import pinned_array
hp = {k: np.ascontiguousarray(inp[k]) for k in ("psi", "psi_prev", "u", "x")}
for s in range(3):
    residual(d, 1.0, hp["psi_prev"], hp["u"], hp["psi"])
    Dh = d.assemble_D(hp["psi"])
    for _ in range(50):
        Dh @ hp["x"]
blk = torch.empty(d.plan.ncells * d.plan.block_len, dtype=torch.float64, device="cuda")
d.blocks_t(out=blk)
torch.cuda.synchronize()
del blk
for rep in range(8):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    lu = d.precond_blocks_t(Dm, alpha, beta)
    e[1].record()
    M = DeviceCellBlockPreconditioner.from_operator(d, Dm, alpha, beta)
    e[2].record()
    torch.cuda.synchronize()
    print("after e2e", rep, "assemble %.2f ms" % e[0].elapsed_time(e[1]), "from_operator %.2f ms" % e[1].elapsed_time(e[2]),
          "reserved %.1f GB" % (torch.cuda.memory_reserved() / 1e9))
    del lu
