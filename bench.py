#!/usr/bin/env python
"""Benchmark: fp64 element-quadrature-points/s for residual + Jacobian apply.

Metric (BASELINE.json): EQP/s = N * Q^2 * (1 + k_mv) / t for
one "step" = 1 LVPP residual (proximal.residual: b_u, b_psi, clamp flag) +
k_mv Jacobian matvecs D(psi) x, on synthetic seeded inputs with the config's
shapes (no public dataset exists for this path).  Default workload: config 1
(64x64 mesh, p=16, Q=24 Gauss, 1 residual + 50 matvecs, alpha cycling over
{1, 4, 16}) -- the largest single-GPU configuration BASELINE.json quotes.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl b200|reference]

Prints ONE JSON line on rank 0.  ``value`` is device-timed (CUDA events on the
launching stream, inputs resident in HBM, L2 flushed between timed steps);
``e2e`` is the same metric through the reference-facing NumPy API with host
buffers (H2D/D2H inside the timed region).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

METRIC = "fp64 element-quadrature-points/sec for residual+Jacobian apply"
UNIT = "EQP/s"
P_FP64_TFLOPS = 37.17       # measured DMMA peak, profiles/fp64_peaks_r01.json
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def peaks():
    hbm = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    return hbm


def syn_flops(n, Q):
    return 2.0 * Q * n * (n + Q)


def algorithmic(cfg, disc_n, nq, ndof_psi, ndof_u):
    """SURVEY.md §8d canonical flops/bytes per residual and per matvec."""
    N = cfg.N
    nc = cfg.ncomp
    F_res = N * 2 * nc * syn_flops(disc_n, nq)
    F_mv = N * nc * 2 * syn_flops(disc_n, nq)
    phi_in = N * disc_n * disc_n if cfg.kind == "obstacle" else N * nq * nq
    B_res = 8.0 * (ndof_u + 2 * ndof_psi + phi_in + ndof_psi + ndof_u + ndof_u)
    B_mv = 8.0 * 2 * ndof_psi
    return F_res, F_mv, B_res, B_mv


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region
    through NVML (nvidia-ml-py) every ~2 ms in a background thread; falls back
    to `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reason_mask = 0
        self.max_mhz = None
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self._stop = threading.Event()

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.reason_mask |= int(get_reasons(h))
                    except Exception:
                        pass
                    self._stop.wait(0.002)

            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
        except Exception:
            self._stop = None
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self):
        reasons = sorted(k for k, bit in self.REASONS.items() if self.reason_mask & bit)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML during the timed region"}


def cpu_reference_step(cfg, rule, cells_frac=None):
    """One bounded sample of the workload on the CPU oracle (numpy port of the
    reference's per-cell algorithm, oracle/hpg_oracle.py).  Returns
    (seconds, eqp_in_sample, sample description)."""
    from types import SimpleNamespace

    from oracle import hpg_oracle as orc
    from paper_2412_13733_b200.tables import Tables
    nc_full = cfg.ncells
    # bound the sample: at most ~4096 cells x 8 matvecs of c1 size
    ncells = nc_full
    kmv = cfg.k_mv
    if cfg.name == "c1":
        kmv = 5
    if cfg.name.startswith("c4"):
        ncells = 64
    t = Tables(rule, cfg.p, cfg.n, cfg.nq(rule))
    tt = SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq)
    x = np.linspace(0.0, 1.0, ncells + 1)
    P = orc.Problem(cfg.kind, x, x, cfg.p, tt)
    inp = config_inputs(cfg, ncells=ncells)
    phi_vals = P.sample(inp["phi"])
    f_load = P.load_vector(P.sample(1.0))
    if cfg.kind == "obstacle":
        phi_mom = P.data_moments(phi_vals)
    t0 = time.perf_counter()
    if cfg.kind == "obstacle":
        P.residual(cfg.alphas[0], inp["psi_prev"], inp["u"], inp["psi"], f_load, phi_moments=phi_mom)
        for _ in range(kmv):
            P.obstacle_apply_D(inp["psi"], inp["x"])
    else:
        P.residual(cfg.alphas[0], inp["psi_prev"], inp["u"], inp["psi"], f_load, phi_vals=phi_vals)
        for _ in range(kmv):
            P.gradient_apply_D(inp["psi"], inp["x"], phi_vals)
    dt = time.perf_counter() - t0
    eqp = ncells * ncells * t.nq ** 2 * (1 + kmv)
    desc = (f"oracle (numpy port of hpgalerkin per-cell quadrature, batched over cells) on "
            f"{ncells}x{ncells} cells of {cfg.name} (p={cfg.p}, {rule} rule nq={t.nq}): "
            f"1 residual + {kmv} apply_D")
    return dt, eqp, desc


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def config_dict(cfg, rule):
    """The workload description shared by both arms (same config => comparable)."""
    nq = cfg.nq(rule)
    cached = not cfg.name.startswith("c4")
    return {"workload": f"{cfg.name}: {cfg.kind} {cfg.ncells}x{cfg.ncells} cells, p={cfg.p}, "
                        f"{rule} rule nq={nq}, (1 residual + {cfg.k_mv} Jacobian matvecs)"
                        + (f" x {cfg.reps}" if cfg.reps > 1 else "")
                        + (f", alpha cycling {list(cfg.alphas)}" if len(cfg.alphas) > 1 else ""),
            "rule": rule, "ncells": cfg.N, "p": cfg.p, "nq": nq, "k_mv": cfg.k_mv, "reps": cfg.reps,
            "matvec": "cached point weights" if cached else "weights recomputed from psi (fused with the residual)",
            "l2": "flushed between timed steps (256 MB write)",
            "eqp_per_step": cfg.N * nq * nq * (1 + cfg.k_mv) * cfg.reps}


# dram bytes per launch of the dominant kernel from one `ncu --set full` capture
# (cold caches: ncu flushes L2 between replays), see profiles/
NCU_TRAFFIC = {("c1", "gauss"): (26275072.0, "profiles/r01e_ncu_full_c1_apply.txt"),
               ("c4p6", "gauss"): (90302464.0 + 22354176.0, "profiles/r01b_ncu_full_c4p6_lowp.txt")}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1 per worker; rank 0 alone does the CPU
    # work here, so give its BLAS / OpenMP pools every host core back
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:
        pass
    rule = args.rule
    for _ in range(args.warmup):
        cpu_reference_step(cfg, rule)
    times, eqps = [], []
    desc = ""
    for _ in range(args.steps):
        dt, eqp, desc = cpu_reference_step(cfg, rule)
        times.append(dt)
        eqps.append(eqp)
    value = sum(eqps) / sum(times)
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config_dict(cfg, rule),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def precond_timing(disc, cfg, psi_prev, u, psi, x, b_u, b_psi, flag, hbm):
    """Factor (P blocks + LU) and apply (per-cell solves) of the device
    CellBlockPreconditioner at beta = 1e-8 (the CLI default, cli.py:142)."""
    import torch
    from paper_2412_13733_b200.disc import DeviceCellBlockPreconditioner
    alpha, beta = cfg.alphas[-1], 1e-8
    disc.residual_t(alpha, psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
    D = disc.assemble_D_t(psi)
    M = DeviceCellBlockPreconditioner.from_operator(disc, D, alpha, beta)
    y = M.apply_t(x)
    torch.cuda.synchronize()
    N, nb = disc.plan.ncells, cfg.ncomp * disc.n * disc.n
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    reps_f, reps_a = 3, 20
    ev[0].record()
    for _ in range(reps_f):
        M = DeviceCellBlockPreconditioner.from_operator(disc, D, alpha, beta)
    ev[1].record()
    ev[2].record()
    for _ in range(reps_a):
        M.apply_t(x, out=y)
    ev[3].record()
    torch.cuda.synchronize()
    t_f = ev[0].elapsed_time(ev[1]) * 1e-3 / reps_f
    t_a = ev[2].elapsed_time(ev[3]) * 1e-3 / reps_a
    F_f = N * 2.0 / 3.0 * nb ** 3
    B_f = 16.0 * N * nb * nb            # P written by the assembly epilogue, LU read+written once
    B_a = 8.0 * N * nb * nb + 16.0 * disc.ndof_psi
    lb_f = max(F_f / (P_FP64_TFLOPS * 1e12), B_f / (hbm * 1e9))
    return {"beta": beta, "factor_ms": t_f * 1e3, "factor_tflops": F_f / t_f / 1e12,
            "factor_roofline_frac": lb_f / t_f, "apply_us": t_a * 1e6, "apply_gbs": B_a / t_a / 1e9,
            "apply_roofline_frac": (B_a / (hbm * 1e9)) / t_a, "nb": nb,
            "path": "hpgPrecondAssemble + hpgLUFactor (from_operator), hpgLUSolve (apply)"}


def schur_timing(disc, cfg, psi_prev, u, psi, b_u, b_psi, flag):
    """Stiffness solve (fast diagonalisation), one-call Schur apply and one
    full schur_solve (device preconditioner, GMRES rtol 1e-8) at beta = 1e-8."""
    import torch
    from paper_2412_13733_b200 import schur
    alpha, beta = cfg.alphas[-1], 1e-8
    Af = schur.DeviceStiffnessFactor(disc)
    bu, bp, _ = disc.residual_t(alpha, psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
    D = disc.assemble_D_t(psi)
    S = schur.DeviceSchurOperator(disc, D, beta, alpha, Af)
    M = disc.schur_preconditioner(D, alpha, beta)
    xs = torch.empty_like(u)
    ys = torch.empty_like(psi)
    out = {}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / reps

    t_solve = timed(lambda: Af.solve_t(u, out=xs), 10)
    t_apply = timed(lambda: S.matvec_t(psi, out=ys), 10)

    def full():
        out["r"] = schur.schur_solve_t(disc, D, alpha, beta, bu, bp, Af, rtol=1e-8, precond=M)

    t_full = timed(full, 2)
    nix = cfg.ncells * cfg.p - 1
    fl = 4 * 2.0 * nix ** 3
    return {"beta": beta, "stiffness_solve_us": t_solve * 1e6, "stiffness_solve_tflops": fl / t_solve / 1e12,
            "schur_apply_us": t_apply * 1e6, "schur_solve_ms": t_full * 1e3,
            "gmres_iterations": out["r"].gmres.iterations,
            "path": "hpgStiffnessSolve (fast diagonalisation, cuBLAS DGEMM), hpgSchurApply, "
                    "schur.schur_solve_t (device GMRES + hpgLUSolve), preconditioner factor excluded"}


def solve_timing(disc):
    """proximal.solve from zero with AlphaSchedule(1, 2, alpha_max=16), beta = 1e-8:
    wall time (synchronised) including the one-time stiffness eigen-factorisation."""
    import torch
    from paper_2412_13733_b200 import proximal
    proximal.solve(disc, proximal.AlphaSchedule(alpha0=1.0, nsteps=1), 1e-8)     # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = proximal.solve(disc, proximal.AlphaSchedule(alpha0=1.0, rate=2.0, alpha_max=16.0), 1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    return {"seconds": t, "converged": rep.converged, "alphas": [s.alpha for s in rep.steps],
            "newton_per_step": [s.newton_iters for s in rep.steps],
            "gmres_per_step": [s.gmres_total for s in rep.steps],
            "ms_per_newton_step": t / max(1, rep.newton_total) * 1e3,
            "t_assembly_s": rep.t_assembly_s, "t_linsolve_s": rep.t_linsolve_s,
            "path": "paper_2412_13733_b200.proximal.solve (device Newton + Schur GMRES)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--rule", default="gauss", choices=["gauss", "reference"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=6)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # the reference arm is a CPU run: rank 0 alone measures and prints, the
        # other ranks exit without work
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2412_13733_b200 import dist as hdist
    if world > 1:
        # torchrun pins one intra-op thread per worker; the e2e host staging
        # copies use a fair share of the host cores instead
        torch.set_num_threads(max(1, (os.cpu_count() or 1) // world))
    torch.cuda.set_device(local)
    hdist.init("nccl")   # one process per GPU; weak scaling: each rank owns a config-sized slab
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    from paper_2412_13733_b200.proximal import residual

    rule = args.rule
    nq = cfg.nq(rule)
    inp = config_inputs(cfg, seed=rank)       # each rank: its own slab of elements (weak scaling)
    mesh = uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p)
    cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
    disc = cls(mesh, inp["f"], inp["phi"], rule=rule, nq=nq if rule == "gauss" else None)
    dev = disc.device
    psi = torch.from_numpy(inp["psi"]).to(dev)
    psi_prev = torch.from_numpy(inp["psi_prev"]).to(dev)
    u = torch.from_numpy(inp["u"]).to(dev)
    x = torch.from_numpy(inp["x"]).to(dev)
    b_u = torch.empty(disc.ndof_u, dtype=torch.float64, device=dev)
    b_psi = torch.empty(disc.ndof_psi, dtype=torch.float64, device=dev)
    y = torch.empty(disc.ndof_psi, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    cached = not cfg.name.startswith("c4")      # c4: HBM-bound, recompute weights from psi
    kmv = cfg.k_mv
    reps = cfg.reps

    def step_residual(alpha):
        if cached:
            # residual + the point weights of D(psi) for the Krylov matvecs
            disc.residual_t(alpha, psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
        else:
            # residual + Jacobian apply at the same psi in one pass (hpgResidualApply)
            disc.residual_apply_t(alpha, psi_prev, u, psi, x, b_u=b_u, b_psi=b_psi, y=y, flag=flag)

    def step_matvecs():
        for _ in range(kmv):
            if cached:
                disc.apply_cached_t(x, out=y)
            else:
                disc.apply_D_t(psi, x, out=y)

    # per-alpha graphs: residual, then matvecs (captured once each)
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for a in cfg.alphas:
            step_residual(a)
        step_matvecs()
    torch.cuda.synchronize()
    g_res = {}
    for a in cfg.alphas:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps if not cached else 1):
                step_residual(a)
        g_res[a] = g
    g_mv = None
    if cached:
        g_mv = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_mv, stream=stream):
            step_matvecs()
    torch.cuda.synchronize()

    launches_per_residual = 3 + (1 if disc.plan.splits > 1 and disc.plan.path == 1 else 0)
    launches_per_step = (launches_per_residual + kmv) if cached else disc.plan.residual_apply_kernels * reps

    def run_steps(nsteps, timed):
        evs = []
        for s in range(nsteps):
            a = cfg.alphas[s % len(cfg.alphas)]
            flush.fill_(float(s))                  # evict L2 between steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g_res[a].replay()
            e1.record(stream)
            if g_mv is not None:
                g_mv.replay()
            e2.record(stream)
            evs.append((e0, e1, e2))
        return evs

    with torch.cuda.stream(stream):
        run_steps(args.warmup, False)
        torch.cuda.synchronize()
        hdist.barrier(dev)
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            evs = run_steps(args.steps, True)
            torch.cuda.synchronize()
        hdist.barrier(dev)
        torch.cuda.synchronize()
    step_ms = [e0.elapsed_time(e2) for e0, e1, e2 in evs]
    res_ms = [e0.elapsed_time(e1) for e0, e1, e2 in evs]
    mv_ms = [e1.elapsed_time(e2) for e0, e1, e2 in evs] if cached else None
    total_ms = hdist.max_over_ranks(sum(step_ms), dev)       # slowest rank
    eqp_step = cfg.N * nq * nq * (1 + kmv) * reps
    value = hdist.aggregate_throughput(eqp_step, args.steps, world, total_ms * 1e-3)

    # roofline of the dominant kernel
    F_res, F_mv, B_res, B_mv = algorithmic(cfg, disc.n, nq, disc.ndof_psi, disc.ndof_u)
    hbm = peaks()
    if cached:
        t_k = statistics.mean(mv_ms) / kmv * 1e-3
        achieved = F_mv / t_k / 1e12
        roof = {"kernel": "k_warp<NT,QT,M_OBST_CACHED> (Jacobian apply from cached weights)"
                if cfg.kind == "obstacle" else "Jacobian apply from cached weights (gradient)",
                "bound": "tensor", "achieved": achieved, "peak": P_FP64_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / P_FP64_TFLOPS,
                "traffic": NCU_TRAFFIC.get((cfg.name, rule), (None, None))[0],
                "traffic_source": NCU_TRAFFIC.get((cfg.name, rule), (None, "not captured for this config"))[1],
                "peak_source": "measured FP64 DMMA peak (profiles/fp64_peaks_r01.json)",
                "algorithmic_per_launch": {"flops": F_mv, "bytes": B_mv},
                "avg_launch_us": t_k * 1e6}
    else:
        t_k = statistics.mean(res_ms) / reps * 1e-3       # fused residual + apply per rep
        bytes_ = B_res + B_mv
        achieved = bytes_ / t_k / 1e9
        roof = {"kernel": "k_lowp<p,Q,apply> (single-pass residual + Jacobian apply, one launch per rep)",
                "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm,
                "traffic": NCU_TRAFFIC.get((cfg.name, rule), (None, None))[0],
                "traffic_source": NCU_TRAFFIC.get((cfg.name, rule), (None, "not captured for this config"))[1],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic_per_launch": {"flops": F_res + F_mv, "bytes": bytes_},
                "avg_launch_us": t_k * 1e6}
    # roofline-combined lower bound for the whole step
    t_lb = max((F_res + kmv * F_mv) / (P_FP64_TFLOPS * 1e12), (B_res + kmv * B_mv) / (hbm * 1e9)) * reps
    step_frac = t_lb / (statistics.mean(step_ms) * 1e-3)

    # e2e through the reference-facing NumPy API (host buffers)
    e2e = None
    if args.e2e_steps > 0:
        hp = {k: np.ascontiguousarray(inp[k]) for k in ("psi", "psi_prev", "u", "x")}
        torch.cuda.synchronize()
        t_e2e = []
        for s in range(args.e2e_steps + 1):
            t0 = time.perf_counter()
            for _ in range(reps):
                bu_h, bpsi_h, cl = residual(disc, cfg.alphas[s % len(cfg.alphas)], hp["psi_prev"],
                                            hp["u"], hp["psi"])
                Dm = disc.assemble_D(hp["psi"]) if cached else None
                for _ in range(kmv):
                    y_h = (Dm @ hp["x"]) if cached else disc.apply_D(hp["psi"], hp["x"])
            torch.cuda.synchronize()
            if s > 0:
                t_e2e.append(time.perf_counter() - t0)
        h2d = 8 * reps * (2 * disc.ndof_psi + disc.ndof_u + (disc.ndof_psi if cached else 0)
                          + kmv * disc.ndof_psi * (1 if cached else 2))
        d2h = 8 * reps * (disc.ndof_u + disc.ndof_psi + kmv * disc.ndof_psi) + 4 * reps
        e2e = {"value": eqp_step / statistics.mean(t_e2e) * world, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": 1e3 * statistics.mean(t_e2e),
               "ms_per_step_min_median_max": [1e3 * min(t_e2e), 1e3 * statistics.median(t_e2e), 1e3 * max(t_e2e)],
               "path": "paper_2412_13733_b200.proximal.residual + disc.assemble_D + (D @ x) x k_mv, NumPy in/out"}

    # element-block assembly (reported separately): configs whose
    # BASELINE workload includes it
    blocks = None
    if cfg.name in ("c0", "c2", "c3") and world == 1:
        disc.residual_t(cfg.alphas[0], psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
        nbl = disc.plan.block_len
        chunk = max(1, min(cfg.N, int((8 << 30) // (8 * nbl))))      # <= 8 GB of blocks per launch
        out_blk = torch.empty((chunk, nbl), dtype=torch.float64, device=dev)
        disc.blocks_t(out=out_blk, c0=0, count=chunk)
        torch.cuda.synchronize()
        eb0 = torch.cuda.Event(enable_timing=True)
        eb1 = torch.cuda.Event(enable_timing=True)
        eb0.record()
        for c0 in range(0, cfg.N, chunk):
            disc.blocks_t(out=out_blk, c0=c0, count=min(chunk, cfg.N - c0))
        eb1.record()
        torch.cuda.synchronize()
        t_blk = eb0.elapsed_time(eb1) * 1e-3
        nb_ = cfg.ncomp * disc.n * disc.n
        nbfield = 1 if cfg.kind == "obstacle" else 3
        F_blk = cfg.N * nbfield * (2.0 * disc.n ** 4 * nq + 2.0 * disc.n ** 2 * nq ** 2)
        B_blk = 8.0 * cfg.N * nb_ * nb_ + 8.0 * disc.ndof_psi
        t_lb = max(F_blk / (P_FP64_TFLOPS * 1e12), B_blk / (hbm * 1e9))
        blocks = {"ms": t_blk * 1e3, "tflops": F_blk / t_blk / 1e12, "gbs": B_blk / t_blk / 1e9,
                  "roofline_frac": t_lb / t_blk, "bytes": B_blk, "flops": F_blk}
        del out_blk

    # per-cell Schur preconditioner (not part of the
    # headline workload): P blocks from the cached weights, batched LU, solve
    from paper_2412_13733_b200 import _lib
    precond = None
    if world == 1 and cfg.ncomp * disc.n * disc.n <= _lib.load().hpgLUMaxBlock():
        precond = precond_timing(disc, cfg, psi_prev, u, psi, x, b_u, b_psi, flag, hbm)

    # Schur-reduced Newton linear solve on the device
    # (needs the per-cell preconditioner: config 3's 6561^2 blocks exceed the
    # per-CTA LU, hpgLUMaxBlock, and are reported as unsupported, not timed)
    lu_fits = cfg.ncomp * disc.n * disc.n <= _lib.load().hpgLUMaxBlock()
    schur_info = None
    if world == 1 and disc.plan.ndof_u > 0:
        schur_info = (schur_timing(disc, cfg, psi_prev, u, psi, b_u, b_psi, flag) if lu_fits else
                      {"unsupported": "per-cell LU block side exceeds hpgLUMaxBlock()"})

    # the whole penalty continuation (proximal.solve) on the device, obstacle configs
    solve_info = None
    if world == 1 and cfg.kind == "obstacle":
        solve_info = (solve_timing(disc) if lu_fits else
                      {"unsupported": "per-cell LU block side exceeds hpgLUMaxBlock()"})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            dt, eqp, desc = cpu_reference_step(cfg, rule)
            cpu = {"value": eqp / dt, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                   "sample": desc, "seconds": dt}
        except Exception as exc:      # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inputs with the config's shapes and value laws, SURVEY.md §8d)",
            "config": config_dict(cfg, rule),
            "roofline": roof,
            "step_roofline_frac": step_frac,
            "blocks": blocks,
            "precond": precond,
            "schur": schur_info,
            "solve": solve_info,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "res_ms_mean": statistics.mean(res_ms),
            "mv_ms_mean": statistics.mean(mv_ms) if mv_ms else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
