"""GPU: the alternative launch paths of one operation agree.

* CTA path with row-tile splits: the cluster (DSMEM) reduction and the
  separate reduction kernel sum the split partials in the same order, so
  residual moments and cached applies are bitwise identical; both match the
  oracle at 1e-12 (few cells -> splits <= 8 -> cluster launch).
* CTA path with / without the shared-memory table copies: identical.
* Low-degree single-pass residual (k_lowp) vs the three-kernel path
  (U side + psi side + hat gather): same results to 1e-12 (different
  summation order of the hat contributions)."""
import os

import numpy as np
import pytest

from oracle import hpg_oracle as orc
from test_gpu_fullsize import build  # noqa: E402  (tests/ is on sys.path under pytest)

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _with_env(var, fn):
    os.environ[var] = "1"
    try:
        return fn()
    finally:
        del os.environ[var]


@pytest.mark.parametrize("cfg_name,ncells", [("c2", 2), ("c2", 3), ("c3", 2)])
def test_cta_split_reduction_paths(cfg_name, ncells):
    cfg, d, P, inp, dev = build(cfg_name, ncells=ncells)
    alpha = cfg.alphas[0]

    def run():
        b_u, b_psi, _ = d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
        y = d.apply_cached_t(dev["x"])
        return b_psi.cpu().numpy(), y.cpu().numpy()

    a_psi, a_y = run()
    b_psi, b_y = _with_env("HPG_NO_CLUSTER", run)
    c_psi, c_y = _with_env("HPG_NO_SMEM_TABLES", run)
    assert np.array_equal(a_psi, b_psi) and np.array_equal(a_y, b_y)
    assert np.array_equal(a_psi, c_psi) and np.array_equal(a_y, c_y)
    ry = (P.obstacle_apply_D(inp["psi"], inp["x"]) if cfg.kind == "obstacle"
          else P.gradient_apply_D(inp["psi"], inp["x"], P.sample(inp["phi"])))
    assert orc.rel_err(a_y, ry) < TOL


@pytest.mark.parametrize("cfg_name", ["c4p2", "c4p4", "c4p6"])
def test_lowp_single_pass_vs_three_kernels(cfg_name):
    cfg, d, P, inp, dev = build(cfg_name, ncells=37)
    alpha = cfg.alphas[0]

    def run():
        b_u, b_psi, y, flag = d.residual_apply_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], dev["x"])
        return b_u.cpu().numpy(), b_psi.cpu().numpy(), y.cpu().numpy(), int(flag.item())

    one = run()
    three = _with_env("HPG_LOWP_OFF", run)
    for a, b in zip(one[:3], three[:3]):
        assert orc.rel_err(a, b) < TOL
    assert one[3] == three[3]


@pytest.mark.parametrize("n", [1000, 921600, 921601])
def test_host_transfers_roundtrip(n):
    """NumPy <-> device through the API's staging (direct below 1 MB, two
    pinned half buffers above): exact, repeated, interleaved with kernels."""
    import torch
    cfg, d, P, inp, dev = build("c4p2", ncells=4)
    rng = np.random.default_rng(n)
    for rep in range(3):
        a = rng.standard_normal(n)
        t = d.h2d(a, f"rt{rep % 2}")
        b = rng.standard_normal(n)
        t2 = d.h2d(b, "rt_other")
        s = (t * 2.0 + t2).clone()
        torch.cuda.synchronize()
        assert np.array_equal(d.d2h(t, "rt"), a)
        assert np.array_equal(d.d2h(s, "rt2"), a * 2.0 + b)


@pytest.mark.parametrize("cfg_name,ncells", [("c1", 64), ("c1", 3), ("c2", 5), ("c3", 2), ("c4p4", 33)])
def test_host_pipelined_matvec(cfg_name, ncells):
    """``D @ x`` with NumPy arrays (page-locked staging in, page-locked result
    out, slabs of cell columns on large meshes) equals the device apply,
    repeatedly: bitwise call to call, and to 1e-13 against the whole-vector
    device apply (a slab may run on the one-wave kernel where the whole mesh
    runs on the streaming kernel: split cells sum in a different order)."""
    cfg, d, P, inp, dev = build(cfg_name, ncells=ncells)
    D = d.assemble_D(inp["psi"])
    ref = d.apply_cached_t(dev["x"]).cpu().numpy()
    first = D @ inp["x"]
    assert orc.rel_err(first, ref) < 1e-13
    for _ in range(3):
        assert np.array_equal(D @ inp["x"], first)
    x2 = np.random.default_rng(1).standard_normal(d.ndof_psi)
    import torch
    ref2 = d.apply_cached_t(torch.from_numpy(x2).cuda()).cpu().numpy()
    assert orc.rel_err(D @ x2, ref2) < 1e-13
    assert np.array_equal(D @ inp["x"], first)


@pytest.mark.parametrize("cfg_name", ["c4p2", "c4p6"])
@pytest.mark.parametrize("bad", [np.nan, -800.0])
def test_lowp_flag_and_nan_semantics(cfg_name, bad):
    """Single-pass kernel vs three-kernel path on a psi with one NaN / one
    overflowing coefficient: same clamp flag, same NaN pattern, same finite
    values (reference semantics: assembly.py:187-192, NaN propagates)."""
    import torch
    cfg, d, P, inp, dev = build(cfg_name, ncells=9)
    psi = inp["psi"].copy()
    psi[len(psi) // 3] = bad
    tp = torch.from_numpy(psi).cuda()

    def run():
        b_u, b_psi, y, flag = d.residual_apply_t(cfg.alphas[0], dev["psi_prev"], dev["u"], tp, dev["x"])
        return b_u.cpu().numpy(), b_psi.cpu().numpy(), y.cpu().numpy(), int(flag.item())

    one = run()
    three = _with_env("HPG_LOWP_OFF", run)
    assert one[3] == three[3] == 1
    for a, b in zip(one[:3], three[:3]):
        assert np.array_equal(np.isnan(a), np.isnan(b))
        ok = ~np.isnan(a)
        assert orc.rel_err(a[ok], b[ok]) < TOL


@pytest.mark.parametrize("ncx,ncy,nq", [(64, 64, 24), (61, 63, 24), (59, 61, 24), (64, 62, 16), (63, 61, 10)])
def test_streaming_cached_apply(ncx, ncy, nq):
    """Config-1 shaped cached Jacobian apply on the persistent streaming
    kernel (k_stream: equal row-tile runs per warp, cells split between two
    warps summed through shared memory) vs the oracle and vs the one-wave
    warp-per-cell kernel, on non-uniform meshes whose cells per SM are not a
    multiple of the scheduler groups (every run-boundary case)."""
    import torch
    from types import SimpleNamespace
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    from paper_2412_13733_b200.workloads import phi_sin
    p = 16
    rng = np.random.default_rng(ncx * 100 + ncy)
    xs = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, ncx))]); xs /= xs[-1]
    ys = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, ncy))]); ys /= ys[-1]
    mesh = TensorMesh2D(Mesh1D(xs, np.full(ncx, p)), Mesh1D(ys, np.full(ncy, p)))
    d = D.ObstacleDisc2D(mesh, 1.0, phi_sin, rule="gauss", nq=nq)   # nq = 24 / 16: 3 / 2 point tiles
    t = d.tables
    P = orc.Problem("obstacle", d.xpts, d.ypts, p, SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    psi = 0.5 * rng.standard_normal(d.ndof_psi)
    x = rng.standard_normal(d.ndof_psi)
    tp, tx = torch.from_numpy(psi).cuda(), torch.from_numpy(x).cuda()
    d.exp_moments_t(tp, wcache=True)

    def run():
        return d.apply_cached_t(tx).cpu().numpy()

    y_stream = run()
    y_stream2 = run()
    y_wave = _with_env("HPG_NO_STREAM", run)
    ry = P.obstacle_apply_D(psi, x)
    assert np.array_equal(y_stream, y_stream2)          # deterministic
    assert orc.rel_err(y_stream, ry) < TOL
    assert orc.rel_err(y_wave, ry) < TOL
    assert orc.rel_err(y_stream, y_wave) < 1e-13


@pytest.mark.parametrize("ncx,ncy,slabs", [(64, 64, 2), (61, 63, 3), (8, 8, 2)])
def test_host_matvec_slab_pipeline(ncx, ncy, slabs):
    """D @ x with NumPy in/out: the slab-pipelined transfer path (upload of
    slab k overlapping apply + download of slab k - 1 through
    hpgApplyCachedRange) returns what the whole-vector path returns; small
    meshes take the whole-vector path.  Results are fresh arrays."""
    from types import SimpleNamespace
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    from paper_2412_13733_b200.workloads import phi_sin
    p = 16
    rng = np.random.default_rng(ncx + 7 * ncy)
    xs = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, ncx))]); xs /= xs[-1]
    ys = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, ncy))]); ys /= ys[-1]
    mesh = TensorMesh2D(Mesh1D(xs, np.full(ncx, p)), Mesh1D(ys, np.full(ncy, p)))
    d = D.ObstacleDisc2D(mesh, 1.0, phi_sin, rule="gauss", nq=24)
    t = d.tables
    P = orc.Problem("obstacle", d.xpts, d.ypts, p, SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    psi = 0.5 * rng.standard_normal(d.ndof_psi)
    Dm = d.assemble_D(psi)
    xa, xb = rng.standard_normal(d.ndof_psi), rng.standard_normal(d.ndof_psi)
    d._SLABS = slabs
    ya = Dm @ xa
    yb = Dm @ xb
    ya_copy = ya.copy()
    d._SLABS = 1
    ya1 = Dm @ xa
    assert np.array_equal(ya, ya_copy)            # a later call does not touch an earlier result
    assert orc.rel_err(ya, P.obstacle_apply_D(psi, xa)) < TOL
    assert orc.rel_err(yb, P.obstacle_apply_D(psi, xb)) < TOL
    assert orc.rel_err(ya, ya1) < 1e-13


@pytest.mark.parametrize("cfg_name,ncells", [("c1", 64), ("c3", 2), ("c4p4", 64)])
def test_page_locked_inputs(cfg_name, ncells):
    """Inputs kept in page-locked arrays (``disc.pinned_array``, or results of
    earlier calls) are uploaded straight from the caller's memory: same
    results as pageable inputs, and a caller may overwrite its array as soon
    as a call has returned (``assemble_D`` keeps no reference to psi's memory)."""
    from paper_2412_13733_b200.disc import pinned_array
    from paper_2412_13733_b200.proximal import residual
    cfg, d, P, inp, dev = build(cfg_name, ncells=ncells)
    pin = {}
    for k in ("psi", "psi_prev", "u", "x"):
        pin[k] = pinned_array(inp[k].shape)
        pin[k][...] = inp[k]
    alpha = cfg.alphas[0]
    a = residual(d, alpha, inp["psi_prev"], inp["u"], inp["psi"])
    b = residual(d, alpha, pin["psi_prev"], pin["u"], pin["psi"])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    Dm = d.assemble_D(pin["psi"])
    y_ref = d.assemble_D(inp["psi"]) @ inp["x"]
    pin["psi"][...] = 123.0                       # the call has returned: D must not change
    y = Dm @ pin["x"]
    # (1e-13: pageable vectors of a large mesh go through the slab pipeline,
    # whose slabs may run on the one-wave kernel -- another summation order
    # for the cells the streaming kernel splits between two warps)
    assert orc.rel_err(y, y_ref) < 1e-13
    # a result (page-locked) fed back as an input
    y2 = Dm @ y
    assert orc.rel_err(y2, Dm @ np.array(y, copy=True)) < 1e-13
    assert np.array_equal(d.apply_D(inp["psi"], pin["x"]), d.apply_D(inp["psi"], inp["x"]))


def test_host_matvec_slabs_gradient():
    """The slab pipeline on a gradient plan (two stacked components: a slab is
    two row ranges) with the warp-per-cell apply: 56 x 56 cells, p = 8."""
    from types import SimpleNamespace
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    p, nc = 8, 56
    rng = np.random.default_rng(5)
    d = D.GradientDisc2D(uniform_mesh_2d(0.0, 1.0, nc, p), 1.0, 0.7, rule="gauss", nq=12)
    assert d.plan.path == 0 and d.ndof_psi >= 2 * d._STAGE_MIN
    t = d.tables
    P = orc.Problem("gradient", d.xpts, d.ypts, p, SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    psi = 0.3 * rng.standard_normal(d.ndof_psi)
    x = rng.standard_normal(d.ndof_psi)
    Dm = d.assemble_D(psi)
    ry = P.gradient_apply_D(psi, x, P.sample(0.7))
    for slabs in (2, 3, 1):
        d._SLABS = slabs
        y = Dm @ x
        assert orc.rel_err(y, ry) < TOL, slabs


@pytest.mark.parametrize("ranges", [[(0, 4000), (4000, 4096)], [(0, 96), (96, 4096)], [(0, 1), (1, 2049), (2049, 4096)]])
def test_apply_cached_range(ranges):
    """hpgApplyCachedRange: disjoint cell ranges (streaming kernel with a
    non-zero first cell, one-wave kernel, a single cell) tile the full apply;
    cells outside a range are left untouched."""
    import torch
    from paper_2412_13733_b200 import _lib, disc as D
    cfg, d, P, inp, dev = build("c1")
    d.exp_moments_t(dev["psi"], wcache=True)
    full = d.apply_cached_t(dev["x"]).cpu().numpy()
    y = torch.full_like(dev["x"], -7.0)
    for lo, hi in ranges:
        _lib.call("hpgApplyCachedRange", d.plan.handle, D._vp(d._wcache), D._vp(dev["x"]), D._vp(y), lo, hi,
                  D._stream())
        got = y.cpu().numpy()
        n = d.n
        cells = np.arange(lo, hi)
        # x-major cell order: cell = cx * ncy + cy; its tile rows / columns
        tile = got.reshape(d.ncx * n, d.ncy * n)
        ref = full.reshape(d.ncx * n, d.ncy * n)
        cx, cy = cells[0] // d.ncy, cells[0] % d.ncy
        assert orc.rel_err(tile[cx * n:(cx + 1) * n, cy * n:(cy + 1) * n], ref[cx * n:(cx + 1) * n, cy * n:(cy + 1) * n]) < 1e-13
    assert orc.rel_err(y.cpu().numpy(), full) < 1e-13          # the ranges tiled everything
    with pytest.raises(ValueError):                            # HPG_ERR_ARG
        _lib.call("hpgApplyCachedRange", d.plan.handle, D._vp(d._wcache), D._vp(dev["x"]), D._vp(y), 10, 5000,
                  D._stream())
