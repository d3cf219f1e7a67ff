"""Cost split of the device GMRES (schur.DeviceGmres): capture + instantiate
vs the graph solve, on a config's Schur system (default c1, Gauss rule)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2412_13733_b200 import _lib, schur  # noqa: E402
from paper_2412_13733_b200 import disc as D  # noqa: E402
from paper_2412_13733_b200.disc import _stream, _vp  # noqa: E402
from paper_2412_13733_b200.mesh import uniform_mesh_2d  # noqa: E402
from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = CONFIGS[name]
inp = config_inputs(cfg)
cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
d = cls(uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p), inp["f"], inp["phi"], rule="gauss", nq=cfg.Q)
t = lambda a: torch.from_numpy(a).cuda()
psi, u, pp = t(inp["psi"]), t(inp["u"]), t(inp["psi_prev"])
alpha, beta = cfg.alphas[-1], 1e-8
bu, bp, _ = d.residual_t(alpha, pp, u, psi, wcache=True)
Dm = d.assemble_D_t(psi)
Af = schur.DeviceStiffnessFactor(d)
M = d.schur_preconditioner(Dm, alpha, beta)
S = schur.DeviceSchurOperator(d, Dm, beta, alpha, Af)
G = schur.DeviceGmres(d.ndof_psi, 150, d.device)
torch.cuda.synchronize()


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


am = lambda x, out: S.matvec_t(x, out=out)
pm = lambda x, out: M.apply_t(x, out=out)
print(f"{name}: schur apply {wall(lambda: S.matvec_t(psi, out=G.w)):.3f} ms, precond apply "
      f"{wall(lambda: M.apply_t(psi, out=G.w)):.3f} ms")
print(f"full G.solve (capture+instantiate+run) {wall(lambda: G.solve(am, bp, M=pm)):.3f} ms")
s = torch.cuda.Stream()


def capture_only():
    with torch.cuda.stream(s):
        st = _stream()
        _lib.call("hpgGmresCaptureBegin", G.handle, st)
        pm(G.vin, G.z)
        am(G.z, G.w)
        _lib.call("hpgGmresCaptureEnd", G.handle, st)


print(f"capture+instantiate {wall(capture_only):.3f} ms")


def run_only():
    with torch.cuda.stream(s):
        _lib.call("hpgGmresSolve", G.handle, 1e-8, 0.0, _vp(G.dx), _stream())


print(f"graph solve only {wall(run_only):.3f} ms")
r = schur.schur_solve_t(d, Dm, alpha, beta, bu, bp, Af, rtol=1e-8, precond=M, gmres=G)
print("iterations", r.gmres.iterations, "residuals", r.gmres.residuals)
print(f"schur_solve_t {wall(lambda: schur.schur_solve_t(d, Dm, alpha, beta, bu, bp, Af, rtol=1e-8, precond=M, gmres=G)):.3f} ms")
