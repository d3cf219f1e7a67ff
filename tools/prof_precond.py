"""Time the per-cell Schur preconditioner on the device (factor + apply) per config.

    python tools/prof_precond.py [cfg ...]

Factor = hpgPrecondFactor on D's blocks (D -> P -> LU, in place), timed
without the blocks build; apply = hpgLUSolve on the global psi vector.
Prints algorithmic rates: getrf 2/3 nb^3 flops per block, blocks read +
factors written (16 nb^2 B); getrs reads the factors once (8 nb^2 B).
CPU reference: scipy lu_factor / lu_solve on a sample of cells.
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2412_13733_b200 import _lib, disc as D                 # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d             # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    import scipy.linalg as sla
    names = sys.argv[1:] or ["c0", "c4p4", "c4p6", "c1", "c2"]
    for name in names:
        cfg = CONFIGS[name]
        inp = config_inputs(cfg)
        cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
        d = cls(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
        dev = {k: torch.from_numpy(np.ascontiguousarray(inp[k])).cuda() for k in ("psi", "psi_prev", "u", "x")}
        alpha, beta = cfg.alphas[-1], 1e-8
        d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
        Dm = d.assemble_D_t(dev["psi"])
        d._precond_ready()
        N = d.plan.ncells
        nb = d.n * d.n * d.ncomp
        blocks = d.blocks_t(wcache=Dm._w).view(N, nb, nb)
        src = blocks.clone()
        piv = torch.empty((N, nb), dtype=torch.int32, device=d.device)
        perm = torch.empty((N, nb), dtype=torch.int32, device=d.device)
        info = torch.zeros(1, dtype=torch.int32, device=d.device)

        def factor():
            blocks.copy_(src)
            _lib.call("hpgPrecondFactor", d.plan.handle, D._vp(blocks), D._vp(piv), D._vp(perm), float(alpha),
                      float(beta), 0, N, D._vp(info), D._stream())

        def copy_only():
            blocks.copy_(src)

        reps = 3 if nb > 500 else 10
        if os.environ.get("HPG_LU_PROF") and nb > 32:
            prof = torch.zeros(8, dtype=torch.int64, device=d.device)
            _lib.call("hpgLUProfile", D._vp(prof))
            factor()
            torch.cuda.synchronize()
            _lib.call("hpgLUProfile", ctypes.c_void_p(0))
            v = prof.cpu().numpy().astype(float)
            names_ = ["panel-load", "writeback", "gather", "Linv", "chunks", "panel-end", "transform", "columns"]
            tot = v.sum()
            print("   phases: " + "  ".join(f"{n_}={x / tot * 100:.1f}%" for n_, x in zip(names_, v)),
                  f" total {tot / (N if N < 296 else 296) / 1.9e3:.0f} us per CTA-lifetime", flush=True)
        t_f = ev_time(factor, reps) - ev_time(copy_only, reps)
        pblk = torch.empty_like(blocks)

        def assemble():
            _lib.call("hpgPrecondAssemble", d.plan.handle, D._vp(Dm._w), float(alpha), float(beta),
                      D._vp(pblk), 0, N, D._stream())

        t_asm = ev_time(assemble, reps)
        psrc = pblk.clone()

        def lu_only():
            pblk.copy_(psrc)
            _lib.call("hpgLUFactor", d.plan.handle, D._vp(pblk), D._vp(piv), D._vp(perm), N, D._vp(info),
                      D._stream())

        t_lu = ev_time(lu_only, reps) - ev_time(lambda: pblk.copy_(psrc), reps)
        print(f"   fused path: assemble P {t_asm * 1e3:.3f} ms + LU {t_lu * 1e3:.3f} ms = "
              f"{(t_asm + t_lu) * 1e3:.3f} ms", flush=True)
        M = D.DeviceCellBlockPreconditioner(d, blocks, piv, info, perm_t=perm)
        y = torch.empty_like(dev["x"])
        t_s = ev_time(lambda: M.apply_t(dev["x"], out=y), 20)
        t_blk = ev_time(lambda: d.blocks_t(wcache=Dm._w, out=blocks.view(N, -1)), reps)
        # CPU reference on a sample of cells
        host = src.cpu().numpy()
        pb = -host[: min(N, 64)]
        ns = min(N, max(1, int(2.0 / max(1e-4, 4e-10 * nb ** 3)))) if nb > 200 else min(N, 256)
        ns = min(ns, pb.shape[0])
        t0 = time.perf_counter()
        facs = [sla.lu_factor(pb[i]) for i in range(ns)]
        t1 = time.perf_counter()
        for i in range(ns):
            sla.lu_solve(facs[i], np.ones(nb))
        t2 = time.perf_counter()
        cpu_f = (t1 - t0) / ns * N
        cpu_s = (t2 - t1) / ns * N
        fl = N * 2.0 / 3.0 * nb ** 3
        print(f"{name:5s} N={N:6d} nb={nb:5d}  factor {t_f * 1e3:8.3f} ms ({fl / t_f * 1e-12:6.2f} TF/s, "
              f"{16.0 * N * nb * nb / t_f * 1e-9:7.1f} GB/s)  solve {t_s * 1e6:8.1f} us "
              f"({8.0 * N * nb * nb / t_s * 1e-9:7.1f} GB/s)  blocks {t_blk * 1e3:7.3f} ms | "
              f"CPU scipy: factor {cpu_f:7.3f} s solve {cpu_s:7.3f} s (sample {ns})", flush=True)


if __name__ == "__main__":
    main()
