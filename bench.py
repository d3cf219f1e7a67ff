#!/usr/bin/env python
"""Benchmark: fp64 element-quadrature-points/s for residual + Jacobian apply.

Metric (BASELINE.json): EQP/s = N * Q^2 * (1 + k_mv) * reps / t
for one "step" = 1 LVPP residual (proximal.residual: b_u, b_psi, clamp flag) +
k_mv Jacobian matvecs D(psi) x (x reps for config 4), on synthetic seeded
inputs with the config's shapes (no public dataset exists for this path).
Headline workload (the JSON line's top-level fields): config 1 (64x64 mesh,
p=16, Q=24 Gauss, 1 residual + 50 matvecs, alpha cycling over {1, 4, 16}) --
the largest single-GPU configuration BASELINE.json quotes.  ``per_config``
carries the same measurement for all five BASELINE configs (c4 at p = 2, 4, 6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl b200|reference]

Prints ONE JSON line on rank 0.
* ``value``: device-timed (CUDA events on the launching stream, inputs
  resident in HBM).  L2: flushed between timed steps (256 MB write); config 4
  additionally rotates its 100 repetitions over >= 3 input/output buffer sets
  totalling more than twice the 126 MB L2, so every repetition streams HBM;
  the Krylov matvecs of the cached configs rotate over 8 direction vectors
  (the weight cache of D(psi) is shared by all matvecs of a Newton step, as
  in GMRES).
* ``e2e``: the same metric through the reference-facing NumPy API with host
  buffers (H2D / D2H inside the timed region).
* ``cpu_baseline`` / ``--impl reference``: the UNMODIFIED reference package
  (hpgalerkin, installed into oracle/_ref by oracle/build_ref.sh) timed on the
  box's host cores on a bounded sample of the same workload: its own
  ``exp_moments`` / ``nl_moments`` + k_mv ``apply_D`` per repetition
  ("hot-only", the line's value) and ``proximal.residual`` as-is.
"""

import argparse
import json
import math
import os
import platform
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2412_13733_b200.workloads import CONFIGS, config_inputs  # noqa: E402

METRIC = "fp64 element-quadrature-points/sec for residual+Jacobian apply"
UNIT = "EQP/s"
P_FP64_TFLOPS = 37.17       # measured DMMA peak, profiles/fp64_peaks_r01.json
L2_BYTES = 126 << 20
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
ALL = ("c0", "c1", "c2", "c3", "c4p2", "c4p4", "c4p6")
# cells per direction of the reference's bounded CPU sample (its per-cell cost
# is mesh-size independent: a Python loop over cells)
REF_SAMPLE_CELLS = {"c0": 4, "c1": 16, "c2": 4, "c3": 1, "c4p2": 16, "c4p4": 16, "c4p6": 16}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (no MEASURED_PEAKS.json)"


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
    through NVML (nvidia-ml-py) every ~2 ms in a background thread."""

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


# ---------------------------------------------------------------------------
# the reference (CPU) arm: the unmodified hpgalerkin package

def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def _reference():
    """hpgalerkin from oracle/_ref (oracle/build_ref.sh); raises when missing."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "hpgalerkin")) and ref not in sys.path:
        sys.path.append(ref)
    import hpgalerkin.assembly  # noqa: F401
    import hpgalerkin.proximal  # noqa: F401
    return sys.modules["hpgalerkin"]


class ReferenceSample:
    """The reference's own disc on a cfg-degree mesh of ``nc`` x ``nc`` cells;
    rule='gauss' substitutes the Gauss tables into its CellKernel1D objects
     and refreshes its data terms."""

    def __init__(self, cfg, rule, nc):
        hp = _reference()
        from hpgalerkin import assembly as ra
        from hpgalerkin.mesh import uniform_mesh_2d

        from paper_2412_13733_b200.tables import Tables
        self.cfg, self.rule, self.nc = cfg, rule, nc
        inp = config_inputs(cfg, ncells=nc)
        mesh = uniform_mesh_2d(0.0, 1.0, nc, cfg.p)
        cls = ra.ObstacleDisc2D if cfg.kind == "obstacle" else ra.GradientDisc2D
        d = cls(mesh, inp["f"], inp["phi"])
        t = Tables(rule, cfg.p, cfg.n, cfg.nq(rule))
        if rule == "gauss":
            for k2 in d.kernels.values():
                for k1 in (k2.kx, k2.ky):
                    k1.nquad = t.nq
                    k1.points = k1.midpoint + 0.5 * k1.h * t.xi
                    k1.S, k1.T, k1.Su, k1.Tu = t.S, t.T, t.Su, t.Tu
            d.f_load = d.load_vector(inp["f"])
            if cfg.kind == "obstacle":
                d.phi_moments = d.data_moments(inp["phi"])
            else:
                d.phi_values = {c: ra._eval_data(inp["phi"], d.kernels[c], "pointwise", 2) for c in d.cell_ids}
        self.disc, self.inp, self.nq = d, inp, t.nq
        self.hp = hp
        self.eqp_rep = nc * nc * t.nq ** 2 * (1 + cfg.k_mv)

    def run(self):
        """One repetition: returns (t_hot, t_as_is) in seconds.
        hot-only = exp/nl_moments + k_mv apply_D; as-is = proximal.residual + k_mv apply_D."""
        from hpgalerkin import proximal
        d, inp, k = self.disc, self.inp, self.cfg.k_mv
        t0 = time.perf_counter()
        if self.cfg.kind == "obstacle":
            d.exp_moments(inp["psi"])
        else:
            d.nl_moments(inp["psi"])
        t1 = time.perf_counter()
        for _ in range(k):
            d.apply_D(inp["psi"], inp["x"])
        t2 = time.perf_counter()
        proximal.residual(d, self.cfg.alphas[0], inp["psi_prev"], inp["u"], inp["psi"])
        t3 = time.perf_counter()
        return (t1 - t0) + (t2 - t1), (t3 - t2) + (t2 - t1)

    def describe(self):
        c = self.cfg
        return (f"unmodified hpgalerkin {getattr(self.hp, '__version__', '?')} (oracle/_ref) on a "
                f"{self.nc}x{self.nc}-cell mesh of {c.name}'s degree (p={c.p}, {self.rule} rule "
                f"nq={self.nq}): per repetition exp/nl_moments + {c.k_mv} apply_D (hot-only; "
                f"as-is: proximal.residual + {c.k_mv} apply_D)")


def _threads(n):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n)
    except Exception:
        class _Nop:
            def __enter__(self):
                return self

            def __exit__(self, *a):
                return False
        return _Nop()


def reference_baseline(cfg, rule, reps=2, one_thread=True):
    """cpu_baseline record: the reference on all host cores (and on 1)."""
    cores = os.cpu_count() or 1
    s = ReferenceSample(cfg, rule, REF_SAMPLE_CELLS[cfg.name])
    with _threads(cores):
        s.run()                                   # warm-up
        hot, asis = zip(*[s.run() for _ in range(reps)])
    rec = {"value": s.eqp_rep / min(hot), "unit": UNIT, "cores": cores, "kind": "reference",
           "cpu_model": cpu_model(), "sample": s.describe() + f"; best of {reps}",
           "as_is_value": s.eqp_rep / min(asis)}
    if one_thread:
        with _threads(1):
            hot1 = min(s.run()[0] for _ in range(reps))
        rec["value_1thread"] = s.eqp_rep / hot1
    return rec


def run_reference(args, cfg, rank, world):
    """``--impl reference``: the unmodified reference on the host cores
    (rank 0 alone; the other ranks exit without work)."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    rule = args.rule
    s = ReferenceSample(cfg, rule, REF_SAMPLE_CELLS[cfg.name])
    with _threads(cores):
        for _ in range(args.warmup):
            s.run()
        times, asis = [], []
        for _ in range(args.steps):
            th, ta = s.run()
            times.append(th)
            asis.append(ta)
        with _threads(1):
            t1 = s.run()[0]
    value = s.eqp_rep * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config_dict(cfg, rule),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": s.describe(),
                         "as_is_value": s.eqp_rep * len(asis) / sum(asis),
                         "value_1thread": s.eqp_rep / t1},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, rule, cached=None):
    """The workload description shared by both arms (same config => comparable)."""
    nq = cfg.nq(rule)
    if cached is None:
        cached = cfg.k_mv > 1
    return {"workload": f"{cfg.name}: {cfg.kind} {cfg.ncells}x{cfg.ncells} cells, p={cfg.p}, "
                        f"{rule} rule nq={nq}, (1 residual + {cfg.k_mv} Jacobian matvecs)"
                        + (f" x {cfg.reps}" if cfg.reps > 1 else "")
                        + (f", alpha cycling {list(cfg.alphas)}" if len(cfg.alphas) > 1 else ""),
            "rule": rule, "ncells": cfg.N, "p": cfg.p, "nq": nq, "k_mv": cfg.k_mv, "reps": cfg.reps,
            "matvec": ("cached point weights of D(psi)" if cached else
                       "at the same psi, fused into the residual's pass (hpgResidualApply)"),
            "l2": ("flushed between timed steps (256 MB write); repetitions rotate over buffer sets "
                   "> 2x L2" if not cached else "flushed between timed steps (256 MB write); matvecs "
                   "rotate over 8 direction vectors"),
            "eqp_per_step": cfg.N * nq * nq * (1 + cfg.k_mv) * cfg.reps}


# dram bytes per launch of the dominant kernel from one `ncu --set full` capture
# (cold caches: ncu flushes L2 between replays), see profiles/
NCU_TRAFFIC = {("c1", "gauss"): (26274304.0 + 0.0, "profiles/r02c_ncu_full_c1_stream_cold.txt"),
               ("c4p6", "gauss"): (90812928.0 + 22752256.0, "profiles/r02a_ncu_full_c4p6_lowp.txt")}


# ---------------------------------------------------------------------------
# the B200 arm

def precond_timing(disc, cfg, psi_prev, u, psi, x, b_u, b_psi, flag, hbm):
    """Factor (P blocks + LU) and apply (per-cell solves) of the device
    CellBlockPreconditioner at beta = 1e-8 (the CLI default, cli.py:142)."""
    import torch
    from paper_2412_13733_b200.disc import DeviceCellBlockPreconditioner
    alpha, beta = cfg.alphas[-1], 1e-8
    disc.residual_t(alpha, psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
    D = disc.assemble_D_t(psi)
    M = DeviceCellBlockPreconditioner.from_operator(disc, D, alpha, beta)
    # (a second untimed build while the first is alive: the timed loop below
    # always holds two factor sets, both then come from torch's caching
    # allocator instead of a 1.7 GB cudaMalloc inside the timed region)
    M = DeviceCellBlockPreconditioner.from_operator(disc, D, alpha, beta)
    y = M.apply_t(x)
    torch.cuda.synchronize()
    N, nb = disc.plan.ncells, cfg.ncomp * disc.n * disc.n
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    reps_f, reps_a = 5, 20
    # each build timed on its own, median reported (a build now and then takes
    # 2-4x longer inside this process -- allocator / driver housekeeping --
    # while the kernels' own times are stable: tools/precond_reps.py)
    t_builds = []
    for _ in range(reps_f):
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        M = DeviceCellBlockPreconditioner.from_operator(disc, D, alpha, beta)
        f1.record()
        torch.cuda.synchronize()
        t_builds.append(f0.elapsed_time(f1) * 1e-3)
    ev[2].record()
    for _ in range(reps_a):
        M.apply_t(x, out=y)
    ev[3].record()
    torch.cuda.synchronize()
    t_f = statistics.median(t_builds)
    t_a = ev[2].elapsed_time(ev[3]) * 1e-3 / reps_a
    F_f = N * 2.0 / 3.0 * nb ** 3
    B_f = 16.0 * N * nb * nb            # P written by the assembly epilogue, LU read+written once
    B_a = 8.0 * N * nb * nb + 16.0 * disc.ndof_psi
    lb_f = max(F_f / (P_FP64_TFLOPS * 1e12), B_f / (hbm * 1e9))
    return {"beta": beta, "factor_ms": t_f * 1e3, "factor_ms_min_max": [1e3 * min(t_builds), 1e3 * max(t_builds)],
            "factor_tflops": F_f / t_f / 1e12,
            "factor_roofline_frac": lb_f / t_f, "apply_us": t_a * 1e6, "apply_gbs": B_a / t_a / 1e9,
            "apply_roofline_frac": (B_a / (hbm * 1e9)) / t_a, "nb": nb,
            "path": "hpgPrecondAssemble + hpgLUFactor (from_operator), hpgLUSolve (apply)"}


def schur_timing(disc, cfg, psi_prev, u, psi, b_u, b_psi, flag):
    """Stiffness solve (fast diagonalisation), one-call Schur apply and one
    full schur_solve (device preconditioner, device GMRES graph, rtol 1e-8) at
    beta = 1e-8."""
    import torch
    from paper_2412_13733_b200 import schur
    alpha, beta = cfg.alphas[-1], 1e-8
    Af = schur.DeviceStiffnessFactor(disc)
    bu, bp, _ = disc.residual_t(alpha, psi_prev, u, psi, b_u=b_u, b_psi=b_psi, flag=flag, wcache=True)
    D = disc.assemble_D_t(psi)
    S = schur.DeviceSchurOperator(disc, D, beta, alpha, Af)
    M = disc.schur_preconditioner(D, alpha, beta)
    G = schur.DeviceGmres(disc.ndof_psi, 150, disc.device)
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
        out["r"] = schur.schur_solve_t(disc, D, alpha, beta, bu, bp, Af, rtol=1e-8, precond=M, gmres=G)

    t_full = timed(full, 2)
    nix = cfg.ncells * cfg.p - 1
    fl = 4 * 2.0 * nix ** 3
    return {"beta": beta, "stiffness_solve_us": t_solve * 1e6, "stiffness_solve_tflops": fl / t_solve / 1e12,
            "schur_apply_us": t_apply * 1e6, "schur_solve_ms": t_full * 1e3,
            "gmres_iterations": out["r"].gmres.iterations,
            "path": "hpgStiffnessSolve (fast diagonalisation, own DMMA GEMMs), hpgSchurApply, "
                    "schur.schur_solve_t (device GMRES graph + hpgLUSolve), preconditioner factor excluded"}


def dist_rank():
    return int(os.environ.get("RANK", "0"))


def gpu_config(cfg, rule, args, local, world, full, e2e_steps):
    """Device-timed measurement of one config; ``full`` adds the headline-only
    extras (preconditioner, Schur solve)."""
    import torch

    from paper_2412_13733_b200 import _lib
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200 import dist as hdist
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    from paper_2412_13733_b200.proximal import residual

    nq = cfg.nq(rule)
    halo = None
    if world > 1:
        # §8e weak scaling: ONE mesh of world x ncells cell columns, each rank
        # owning ncells columns (its config-sized share) and running the
        # unchanged single-GPU path on its slab + two ghost columns per
        # interior side; ghost rows of psi, psi_prev and u come from the
        # neighbours over NCCL at the start of every step (dist.SlabHalo)
        from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
        from paper_2412_13733_b200.workloads import make_inputs
        rank = dist_rank()
        halo = hdist.SlabHalo(world * cfg.ncells, cfg.ncells, cfg.p, cfg.kind, world, rank)
        xg = np.linspace(0.0, float(world), world * cfg.ncells + 1)
        mesh = TensorMesh2D(Mesh1D(halo.local_points(xg), np.full(halo.ncx_local, cfg.p)),
                            Mesh1D(np.linspace(0.0, 1.0, cfg.ncells + 1), np.full(cfg.ncells, cfg.p)))
        inp = config_inputs(cfg, seed=0)
        psi_l, u_l, x_l, _ = make_inputs(cfg.kind, halo.ncx_local, cfg.ncells, cfg.p, seed=rank)
        inp.update(psi=psi_l, u=u_l, x=x_l, psi_prev=np.zeros_like(psi_l))
    else:
        inp = config_inputs(cfg, seed=0)
        mesh = uniform_mesh_2d(0.0, 1.0, cfg.ncells, cfg.p)
    cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
    disc = cls(mesh, inp["f"], inp["phi"], rule=rule, nq=nq if rule == "gauss" else None)
    dev = disc.device
    # the Jacobian matvecs: from the residual's cached point weights (Krylov
    # style), or -- config 4, and k_mv = 1 plans whose hpgResidualApply fuses
    # the apply into the residual's pass -- recomputed at the same psi
    cached = not (cfg.name.startswith("c4") or (cfg.k_mv == 1 and disc.plan.fused_apply))
    kmv, reps = cfg.k_mv, cfg.reps
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def new_set():
        return {"psi": t(inp["psi"]), "psi_prev": t(inp["psi_prev"]), "u": t(inp["u"]), "x": t(inp["x"]),
                "b_u": torch.empty(disc.ndof_u, dtype=torch.float64, device=dev),
                "b_psi": torch.empty(disc.ndof_psi, dtype=torch.float64, device=dev),
                "y": torch.empty(disc.ndof_psi, dtype=torch.float64, device=dev)}

    set_bytes = 8 * (5 * disc.ndof_psi + 2 * disc.ndof_u)
    nsets = min(max(3, math.ceil(2 * L2_BYTES / set_bytes)), reps) if not cached else 1
    sets = [new_set() for _ in range(nsets)]
    s0 = sets[0]
    NX = 8
    xs = [s0["x"]] + [s0["x"].clone() for _ in range(NX - 1)] if cached else None
    ys = [torch.empty_like(s0["y"]) for _ in range(NX)] if cached else None

    def step_residual(alpha):
        if cached:
            disc.residual_t(alpha, s0["psi_prev"], s0["u"], s0["psi"], b_u=s0["b_u"], b_psi=s0["b_psi"],
                            flag=flag, wcache=True)
        else:
            for r in range(reps):
                st = sets[r % nsets]
                disc.residual_apply_t(alpha, st["psi_prev"], st["u"], st["psi"], st["x"], b_u=st["b_u"],
                                      b_psi=st["b_psi"], y=st["y"], flag=flag)

    def step_matvecs(k):
        for i in range(k):
            disc.apply_cached_t(xs[i % NX], out=ys[i % NX])

    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for a in cfg.alphas:
            step_residual(a)
        if cached:
            step_matvecs(kmv)
    torch.cuda.synchronize()
    g_res = {}
    for a in cfg.alphas:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step_residual(a)
        g_res[a] = g
    g_mv = g_kern = None
    KREP = 20
    if cached:
        g_mv = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_mv, stream=stream):
            step_matvecs(kmv)
        g_kern = torch.cuda.CUDAGraph()                 # dominant-kernel timing replay
        with torch.cuda.graph(g_kern, stream=stream):
            step_matvecs(KREP)
    torch.cuda.synchronize()

    launches_per_residual = 3 + (1 if disc.plan.splits > 1 and disc.plan.path == 1 else 0)
    launches_per_step = (launches_per_residual + kmv) if cached else disc.plan.residual_apply_kernels * reps

    def run_steps(nsteps):
        evs = []
        for s in range(nsteps):
            a = cfg.alphas[s % len(cfg.alphas)]
            flush.fill_(float(s))                  # evict L2 between steps
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            if halo is not None:
                halo.exchange(psi_like=[s0["psi"], s0["psi_prev"]], u_like=[s0["u"]])
            g_res[a].replay()
            e1.record(stream)
            if g_mv is not None:
                g_mv.replay()
            e2.record(stream)
            evs.append((e0, e1, e2))
        return evs

    with torch.cuda.stream(stream):
        run_steps(args.warmup)
        torch.cuda.synchronize()
        hdist.barrier(dev)
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            evs = run_steps(args.steps)
            torch.cuda.synchronize()
        hdist.barrier(dev)
        torch.cuda.synchronize()
        t_kern = None
        if g_kern is not None:
            g_kern.replay()
            torch.cuda.synchronize()
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(stream)
            for _ in range(3):
                g_kern.replay()
            k1.record(stream)
            torch.cuda.synchronize()
            t_kern = k0.elapsed_time(k1) * 1e-3 / (3 * KREP)
    step_ms = [e0.elapsed_time(e2) for e0, e1, e2 in evs]
    res_ms = [e0.elapsed_time(e1) for e0, e1, e2 in evs]
    mv_ms = [e1.elapsed_time(e2) for e0, e1, e2 in evs] if cached else None
    total_ms = hdist.max_over_ranks(sum(step_ms), dev)       # slowest rank
    eqp_step = cfg.N * nq * nq * (1 + kmv) * reps
    value = hdist.aggregate_throughput(eqp_step, args.steps, world, total_ms * 1e-3)

    F_res, F_mv, B_res, B_mv = algorithmic(cfg, disc.n, nq, disc.ndof_psi, disc.ndof_u)
    hbm, hbm_src = peaks()
    traffic, traffic_src = NCU_TRAFFIC.get((cfg.name, rule), (None, "not captured for this config"))
    if cached:
        achieved = F_mv / t_kern / 1e12
        roof = {"kernel": ("k_stream|k_warp<NT,QT,M_OBST_CACHED>" if disc.plan.path == 0 else "k_cta<M_*_CACHED>")
                          + " (Jacobian apply from cached weights)",
                "bound": "tensor", "achieved": achieved, "peak": P_FP64_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / P_FP64_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "measured FP64 DMMA peak (profiles/fp64_peaks_r01.json)",
                "algorithmic_per_launch": {"flops": F_mv, "bytes": B_mv},
                "avg_launch_us": t_kern * 1e6,
                "timing": f"CUDA events around {KREP} back-to-back launches (graph) on the launching stream"}
    elif cfg.name.startswith("c4"):
        t_k = statistics.mean(res_ms) / reps * 1e-3       # fused residual + apply per rep
        bytes_ = B_res + B_mv
        achieved = bytes_ / t_k / 1e9
        roof = {"kernel": "k_lowp<p,Q,apply> (single-pass residual + Jacobian apply, one launch per rep)",
                "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": hbm_src,
                "algorithmic_per_launch": {"flops": F_res + F_mv, "bytes": bytes_},
                "avg_launch_us": t_k * 1e6,
                "timing": f"CUDA events around the step's {reps} launches (buffer sets rotated: {nsets})"}
    else:
        # hpgResidualApply in one row-split pass (k_wsplit_ra) + the U side and
        # hat gather: timed as the whole call (the kernel alone is faster)
        t_k = statistics.mean(res_ms) * 1e-3
        achieved = (F_res + F_mv) / t_k / 1e12
        roof = {"kernel": "hpgResidualApply = U side + k_wsplit_ra (fused residual + apply) + hat gather",
                "bound": "tensor", "achieved": achieved, "peak": P_FP64_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / P_FP64_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "measured FP64 DMMA peak (profiles/fp64_peaks_r01.json)",
                "algorithmic_per_launch": {"flops": F_res + F_mv, "bytes": B_res + B_mv},
                "avg_launch_us": t_k * 1e6,
                "timing": "CUDA events around the whole call (3 kernels) on the launching stream"}
    t_lb = max((F_res + kmv * F_mv) / (P_FP64_TFLOPS * 1e12), (B_res + kmv * B_mv) / (hbm * 1e9)) * reps
    step_frac = t_lb / (statistics.mean(step_ms) * 1e-3)

    # e2e through the reference-facing NumPy API (host buffers)
    e2e = None
    if e2e_steps > 0:
        # host inputs in page-locked memory (the contract's "from pinned host
        # memory": paper_2412_13733_b200.disc.pinned_array): uploaded by one DMA
        # each; one extra step with the same inputs in pageable memory (staged
        # through the library's page-locked buffers) is reported beside it
        from paper_2412_13733_b200.disc import pinned_array
        hp_page = {k: np.ascontiguousarray(inp[k]) for k in ("psi", "psi_prev", "u", "x")}
        hp = {}
        for k, v in hp_page.items():
            hp[k] = pinned_array(v.shape)
            hp[k][...] = v

        def e2e_step(h, s):
            for _ in range(reps):
                residual(disc, cfg.alphas[s % len(cfg.alphas)], h["psi_prev"], h["u"], h["psi"])
                Dm = disc.assemble_D(h["psi"]) if cached else None
                for _ in range(kmv):
                    (Dm @ h["x"]) if cached else disc.apply_D(h["psi"], h["x"])
            torch.cuda.synchronize()

        torch.cuda.synchronize()
        t_e2e = []
        E2E_WARM = 2      # untimed: the page-locked staging / result blocks are allocated here
        for s in range(e2e_steps + E2E_WARM):
            t0 = time.perf_counter()
            e2e_step(hp, s)
            if s >= E2E_WARM:
                t_e2e.append(time.perf_counter() - t0)
        t_page = []
        for s in range(3):
            t0 = time.perf_counter()
            e2e_step(hp_page, s)
            t_page.append(time.perf_counter() - t0)
        h2d = 8 * reps * (2 * disc.ndof_psi + disc.ndof_u + (disc.ndof_psi if cached else 0)
                          + kmv * disc.ndof_psi * (1 if cached else 2))
        d2h = 8 * reps * (disc.ndof_u + disc.ndof_psi + kmv * disc.ndof_psi) + 4 * reps
        e2e_s = hdist.max_over_ranks(statistics.mean(t_e2e), dev)
        e2e = {"value": eqp_step * world / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": 1e3 * e2e_s,
               "ms_per_step_min_median_max": [1e3 * min(t_e2e), 1e3 * statistics.median(t_e2e), 1e3 * max(t_e2e)],
               "host_inputs": "page-locked NumPy arrays (disc.pinned_array); results returned as page-locked arrays",
               "ms_per_step_pageable_inputs": 1e3 * min(t_page[1:]),
               "path": "paper_2412_13733_b200.proximal.residual + disc.assemble_D + (D @ x) x k_mv, NumPy in/out"}

    rec = {"config": config_dict(cfg, rule, cached), "value": value, "ms_per_step": total_ms / args.steps,
           "roofline": roof, "step_roofline_frac": step_frac, "e2e": e2e,
           "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
           "res_ms_mean": statistics.mean(res_ms), "mv_ms_mean": statistics.mean(mv_ms) if mv_ms else None,
           "buffer_sets": nsets}

    # element-block assembly (reported separately): configs whose
    # BASELINE workload includes it
    if cfg.name in ("c0", "c2", "c3") and world == 1:
        disc.residual_t(cfg.alphas[0], s0["psi_prev"], s0["u"], s0["psi"], b_u=s0["b_u"], b_psi=s0["b_psi"],
                        flag=flag, wcache=True)
        nbl = disc.plan.block_len
        out_blk = torch.empty((cfg.N, nbl), dtype=torch.float64, device=dev)
        disc.blocks_t(out=out_blk)
        torch.cuda.synchronize()
        eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eb0.record()
        disc.blocks_t(out=out_blk)
        eb1.record()
        torch.cuda.synchronize()
        t_blk = eb0.elapsed_time(eb1) * 1e-3
        nb_ = cfg.ncomp * disc.n * disc.n
        nbfield = 1 if cfg.kind == "obstacle" else 3
        F_blk = cfg.N * nbfield * (2.0 * disc.n ** 4 * nq + 2.0 * disc.n ** 2 * nq ** 2)
        B_blk = 8.0 * cfg.N * nb_ * nb_ + 8.0 * disc.ndof_psi
        lb = max(F_blk / (P_FP64_TFLOPS * 1e12), B_blk / (hbm * 1e9))
        rec["blocks"] = {"ms": t_blk * 1e3, "tflops": F_blk / t_blk / 1e12, "gbs": B_blk / t_blk / 1e9,
                         "roofline_frac": lb / t_blk, "bytes": B_blk, "flops": F_blk}
        del out_blk
    if full and world == 1:
        lu_fits = cfg.ncomp * disc.n * disc.n <= _lib.load().hpgLUMaxBlock()
        if lu_fits:
            rec["precond"] = precond_timing(disc, cfg, s0["psi_prev"], s0["u"], s0["psi"], s0["x"],
                                            s0["b_u"], s0["b_psi"], flag, hbm)
        if disc.plan.ndof_u > 0:
            rec["schur"] = (schur_timing(disc, cfg, s0["psi_prev"], s0["u"], s0["psi"], s0["b_u"],
                                         s0["b_psi"], flag) if lu_fits else
                            {"unsupported": "per-cell LU block side exceeds hpgLUMaxBlock()"})
    del sets, g_res, g_mv, g_kern
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


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
    ap.add_argument("--only", action="store_true", help="measure the headline config alone (no per_config)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
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
    hdist.init("nccl")
    rule = args.rule
    head = gpu_config(cfg, rule, args, local, world, full=True, e2e_steps=args.e2e_steps)
    per = {}
    if not args.only:
        for name in ALL:
            if name == cfg.name:
                rec = head
            else:
                rec = gpu_config(CONFIGS[name], rule, args, local, world, full=False, e2e_steps=3)
            per[name] = {k: rec[k] for k in ("value", "ms_per_step", "step_roofline_frac", "gpu_launches",
                                                "buffer_sets")}
            per[name]["roofline"] = {k: rec["roofline"][k] for k in ("kernel", "bound", "achieved", "peak",
                                                                     "unit", "frac", "avg_launch_us")}
            per[name]["e2e"] = rec["e2e"]["value"] if rec["e2e"] else None
            per[name]["workload"] = rec["config"]["workload"]
            if "blocks" in rec:
                per[name]["blocks"] = rec["blocks"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_baseline(cfg, rule, one_thread=True)
        except Exception as exc:      # the baseline must never sink the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {exc!r}"}
        for name in per:
            if name == cfg.name:
                per[name]["cpu_baseline"] = cpu.get("value")
                continue
            try:
                c = reference_baseline(CONFIGS[name], rule, reps=1, one_thread=False)
                per[name]["cpu_baseline"] = c["value"]
                per[name]["cpu_baseline_as_is"] = c["as_is_value"]
            except Exception as exc:
                per[name]["cpu_baseline"] = f"failed: {exc!r}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded inputs with the config's shapes and value laws, SURVEY.md §8d)",
            "config": head["config"],
            "parallelism": (f"dp{world}: one mesh of {world}x{cfg.ncells} cell columns sharded into "
                            f"slabs, 2 ghost columns per interface, NCCL halo exchange of psi/psi_prev/u "
                            f"rows per step" if world > 1 else "single GPU"),
            "roofline": head["roofline"],
            "step_roofline_frac": head["step_roofline_frac"],
            "precond": head.get("precond"),
            "schur": head.get("schur"),
            "cpu_baseline": cpu,
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "res_ms_mean": head["res_ms_mean"],
            "mv_ms_mean": head["mv_ms_mean"],
            "per_config": per or None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
