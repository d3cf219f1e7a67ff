"""Load the golden fixtures written by oracle/make_golden.py."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    for k in ("kind", "rule"):
        d[k] = str(d[k])
    for k in ("p", "nq"):
        d[k] = int(d[k])
    d["alpha"] = float(d["alpha"])
    for k in ("clamped", "res_clamped", "D_clamped"):
        d[k] = bool(d[k])
    return d


def solve_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "solve", "*.npz")))


def load_solve(name):
    with np.load(os.path.join(GOLDEN, "solve", name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    for k in ("kind", "rule"):
        d[k] = str(d[k])
    for k in ("p", "nq"):
        d[k] = int(d[k])
    for k in ("beta", "alpha_max", "outer_increment"):
        d[k] = float(d[k])
    d["line_search"] = bool(d["line_search"])
    d["converged"] = bool(d["converged"])
    d["alpha0"] = float(d["alpha"])
    d["linear_solver"] = str(d["linear_solver"]) if "linear_solver" in d else "schur"
    return d


def qvi_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "qvi", "*.npz")))


def load_qvi(name):
    with np.load(os.path.join(GOLDEN, "qvi", name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    d["rule"] = str(d["rule"])
    for k in ("p", "nq", "newton"):
        d[k] = int(d[k])
    for k in ("load", "gamma"):
        d[k] = float(d[k])
    return d
