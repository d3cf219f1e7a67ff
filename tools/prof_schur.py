"""Time the device Schur-reduced Newton solve per config.

    python tools/prof_schur.py [cfg ...]

stiffness factor (host eigh + upload), hpgStiffnessSolve, hpgSchurApply and
one full schur_solve_t (RHS = the residual at the config's inputs, the
device per-cell preconditioner, GMRES rtol 1e-8), CUDA-event timed after a
warm-up.  CPU reference: scipy SuperLU of the same A (the reference's
factor_stiffness 'splu', linalg.py:98-117) on a 16x16 mesh of the config's
degree (the full c1 factor takes minutes on this CPU).
"""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2412_13733_b200 import disc as D, schur                 # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d             # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402


def ev(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    for name in sys.argv[1:] or ["c1", "c2", "c4p4"]:
        cfg = CONFIGS[name]
        inp = config_inputs(cfg)
        cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
        d = cls(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
        dev = {k: torch.from_numpy(np.ascontiguousarray(inp[k])).cuda() for k in ("psi", "psi_prev", "u", "x")}
        alpha, beta = cfg.alphas[-1], 1e-8
        t0 = time.perf_counter()
        Af = schur.DeviceStiffnessFactor(d)
        torch.cuda.synchronize()
        t_fac = time.perf_counter() - t0
        b_u, b_psi, _ = d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
        Dm = d.assemble_D_t(dev["psi"])
        S = schur.DeviceSchurOperator(d, Dm, beta, alpha, Af)
        xs = torch.empty_like(dev["u"])
        t_solve = ev(lambda: Af.solve_t(dev["u"], out=xs), 20)
        ys = torch.empty_like(dev["x"])
        t_apply = ev(lambda: S.matvec_t(dev["x"], out=ys), 20)
        M = d.schur_preconditioner(Dm, alpha, beta)
        t_pre = ev(lambda: d.schur_preconditioner(Dm, alpha, beta), 3)
        res = {}

        def full():
            res["r"] = schur.schur_solve_t(d, Dm, alpha, beta, b_u, b_psi, Af, rtol=1e-8, precond=M)

        t_full = ev(full, 3)
        r = res["r"]
        nix = d.plan.ndof_u
        fl = 4 * 2.0 * (cfg.ncells * cfg.p - 1) ** 3
        print(f"{name:5s} ndof_u={nix:8d} ndof_psi={d.ndof_psi:8d}  stiffness factor {t_fac:6.2f} s (host eigh)  "
              f"solve {t_solve * 1e6:8.1f} us ({fl / t_solve * 1e-12:5.1f} TF/s)  schur apply {t_apply * 1e6:8.1f} us  "
              f"precond {t_pre * 1e3:7.2f} ms  schur_solve {t_full * 1e3:7.2f} ms ({r.gmres.iterations} GMRES its, "
              f"excl. precond factor)", flush=True)
        # CPU reference: SuperLU of the same A on a 16x16 mesh of this degree
        nc = 16
        Kx, Mx = schur.u_matrices_1d(np.full(nc, 1.0 / nc), cfg.p)
        A = (sp.kron(sp.csr_matrix(Kx), sp.csr_matrix(Mx)) + sp.kron(sp.csr_matrix(Mx), sp.csr_matrix(Kx))).tocsc()
        A.eliminate_zeros()
        t0 = time.perf_counter()
        lu = spla.splu(A)
        t1 = time.perf_counter()
        lu.solve(np.ones(A.shape[0]))
        t2 = time.perf_counter()
        print(f"      CPU SuperLU (reference factor_stiffness) on 16x16 p={cfg.p}: n={A.shape[0]} factor {t1 - t0:.2f} s, "
              f"solve {(t2 - t1) * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
