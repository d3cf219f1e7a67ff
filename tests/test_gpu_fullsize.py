"""GPU parity at BASELINE.json's full sizes against the (golden-pinned) CPU
oracle, plus size-independent properties:
* all 14 (config, rule) pairs: residual, Jacobian apply from psi, cached
  apply and the fused residual + apply vs the oracle on the full meshes;
* element blocks on the full meshes (every cell assembled in one call, the
  multi-wave grids included), sampled cells vs the oracle's per-cell
  weighted blocks, and the dense-block matvec vs the matrix-free apply;
* D(psi) x three ways (matrix-free from psi, from cached weights, dense blocks);
* exact u-side couplings (B^T u, B psi, A u) on their own;
* linearity of the Jacobian apply in x;
* the residual's exact zero-state identity (tests/test_proximal.py:144-153)."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import hpg_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-12


def build(cfg_name, rule="gauss", ncells=None):
    import torch
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    from paper_2412_13733_b200.workloads import CONFIGS, config_inputs
    cfg = CONFIGS[cfg_name]
    nc = cfg.ncells if ncells is None else ncells
    inp = config_inputs(cfg, ncells=nc)
    cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
    d = cls(uniform_mesh_2d(0.0, 1.0, nc, cfg.p), inp["f"], inp["phi"], rule=rule,
            nq=cfg.Q if rule == "gauss" else None)
    t = d.tables
    P = orc.Problem(cfg.kind, d.xpts, d.ypts, cfg.p,
                    SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    dev = {k: torch.from_numpy(np.ascontiguousarray(inp[k])).cuda() for k in ("psi", "psi_prev", "u", "x")}
    return cfg, d, P, inp, dev


# every BASELINE.json config under both quadrature rules (14 pairs)
ALL_PAIRS = [(c, r) for c in ("c0", "c1", "c2", "c3", "c4p2", "c4p4", "c4p6") for r in ("gauss", "reference")]


@pytest.mark.parametrize("cfg_name,rule", ALL_PAIRS)
def test_full_size_residual_and_apply(cfg_name, rule):
    cfg, d, P, inp, dev = build(cfg_name, rule)
    alpha = cfg.alphas[-1]
    phi_vals = P.sample(inp["phi"])
    f_load = P.load_vector(P.sample(1.0))
    assert orc.rel_err(d.f_load, f_load) < TOL
    if cfg.kind == "obstacle":
        phi_mom = P.data_moments(phi_vals)
        assert orc.rel_err(d.phi_moments, phi_mom) < TOL
        rb_u, rb_psi, rcl = P.residual(alpha, inp["psi_prev"], inp["u"], inp["psi"], f_load,
                                       phi_moments=phi_mom)
        ry = P.obstacle_apply_D(inp["psi"], inp["x"])
    else:
        rb_u, rb_psi, rcl = P.residual(alpha, inp["psi_prev"], inp["u"], inp["psi"], f_load,
                                       phi_vals=phi_vals)
        ry = P.gradient_apply_D(inp["psi"], inp["x"], phi_vals)
    b_u, b_psi, flag = d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
    assert orc.rel_err(b_u.cpu().numpy(), rb_u) < TOL
    assert orc.rel_err(b_psi.cpu().numpy(), rb_psi) < TOL
    if cfg.kind == "obstacle":
        assert bool(flag.item()) == rcl
    y_cached = d.apply_cached_t(dev["x"]).cpu().numpy()
    y_psi = d.apply_D_t(dev["psi"], dev["x"]).cpu().numpy()
    assert orc.rel_err(y_cached, ry) < TOL
    assert orc.rel_err(y_psi, ry) < TOL
    b_u2, b_psi2, y2, _ = d.residual_apply_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], dev["x"])
    assert orc.rel_err(b_u2.cpu().numpy(), rb_u) < TOL
    assert orc.rel_err(b_psi2.cpu().numpy(), rb_psi) < TOL
    assert orc.rel_err(y2.cpu().numpy(), ry) < TOL
    # without the weight cache (the single-pass low-degree kernels at config 4)
    b_u3, b_psi3, flag3 = d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"])
    assert orc.rel_err(b_u3.cpu().numpy(), rb_u) < TOL
    assert orc.rel_err(b_psi3.cpu().numpy(), rb_psi) < TOL
    if cfg.kind == "obstacle":
        assert bool(flag3.item()) == rcl


@pytest.mark.parametrize("p", [2, 3, 4, 6])
@pytest.mark.parametrize("rule", ["gauss", "reference"])
def test_low_degree_ragged_tiles(p, rule):
    """Single-pass low-degree kernels (k_lowt tiles of 8 x 16 cells at p <= 3,
    k_lowp above) on a rectangular, non-uniform 19 x 37 mesh: several tiles,
    partial tiles on both edges, halo cells on every tile boundary, per-cell
    sizes; residual, fused residual + apply and the clamp flag vs the oracle."""
    import torch
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    from paper_2412_13733_b200.workloads import phi_sin
    rng = np.random.default_rng(100 + p)
    xs = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, 19))]); xs /= xs[-1]
    ys = np.concatenate([[0.0], np.cumsum(rng.uniform(0.5, 1.5, 37))]); ys /= ys[-1]
    mesh = TensorMesh2D(Mesh1D(xs, np.full(19, p)), Mesh1D(ys, np.full(37, p)))
    d = D.ObstacleDisc2D(mesh, 1.0, phi_sin, rule=rule, nq=p + 3 if rule == "gauss" else None)
    t = d.tables
    P = orc.Problem("obstacle", d.xpts, d.ypts, p, SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    psi = rng.standard_normal(d.ndof_psi)
    psi[::97] = -800.0                            # clamped points: the flag must be raised
    psi_prev = rng.standard_normal(d.ndof_psi)
    u = rng.standard_normal(d.ndof_u)
    x = rng.standard_normal(d.ndof_psi)
    alpha = 3.0
    phi_mom = P.data_moments(P.sample(phi_sin))
    f_load = P.load_vector(P.sample(1.0))
    rb_u, rb_psi, rcl = P.residual(alpha, psi_prev, u, psi, f_load, phi_moments=phi_mom)
    ry = P.obstacle_apply_D(psi, x)
    assert rcl
    dv = {k: torch.from_numpy(v).cuda() for k, v in (("psi", psi), ("pp", psi_prev), ("u", u), ("x", x))}
    b_u, b_psi, flag = d.residual_t(alpha, dv["pp"], dv["u"], dv["psi"])
    assert orc.rel_err(b_u.cpu().numpy(), rb_u) < TOL
    assert orc.rel_err(b_psi.cpu().numpy(), rb_psi) < TOL
    assert bool(flag.item())
    b_u2, b_psi2, y2, flag2 = d.residual_apply_t(alpha, dv["pp"], dv["u"], dv["psi"], dv["x"])
    assert orc.rel_err(b_u2.cpu().numpy(), rb_u) < TOL
    assert orc.rel_err(b_psi2.cpu().numpy(), rb_psi) < TOL
    assert orc.rel_err(y2.cpu().numpy(), ry) < TOL
    assert bool(flag2.item())


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c4p4"])
def test_u_side_couplings(cfg_name):
    cfg, d, P, inp, dev = build(cfg_name, ncells=8 if cfg_name != "c4p4" else 32)
    assert orc.rel_err(d.BT_u_t(dev["u"]).cpu().numpy(), P.BT_u(inp["u"])) < TOL
    assert orc.rel_err(d.B_psi_t(dev["psi"]).cpu().numpy(), P.B_psi(inp["psi"])) < TOL
    assert orc.rel_err(d.A_u_t(dev["u"]).cpu().numpy(), P.A_u(inp["u"])) < TOL


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3"])
def test_blocks_three_ways(cfg_name):
    """dense-block matvec == cached matrix-free apply == apply from psi."""
    import torch
    cfg, d, P, inp, dev = build(cfg_name, ncells=4 if cfg_name != "c3" else 2)
    D = d.assemble_D_t(dev["psi"])
    y1 = D.matvec_t(dev["x"]).cpu().numpy()
    y2 = D.matvec_blocks_t(dev["x"]).cpu().numpy()
    y3 = d.apply_D_t(dev["psi"], dev["x"]).cpu().numpy()
    assert orc.rel_err(y2, y1) < TOL
    assert orc.rel_err(y3, y1) < TOL
    # selected cells against the oracle's einsum blocks
    if cfg.kind == "obstacle":
        ref, _ = P.obstacle_blocks(inp["psi"])
    else:
        ref = P.gradient_blocks(inp["psi"], P.sample(inp["phi"]))
    got = D.blocks_t().cpu().numpy()
    assert orc.rel_err(got, ref) < TOL
    del torch


def test_apply_is_linear_in_x():
    import torch
    cfg, d, P, inp, dev = build("c1", ncells=16)
    x2 = torch.from_numpy(np.random.default_rng(7).standard_normal(d.ndof_psi)).cuda()
    d.residual_t(1.0, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
    a = d.apply_cached_t(dev["x"])
    b = d.apply_cached_t(x2)
    ab = d.apply_cached_t(2.5 * dev["x"] - 0.5 * x2)
    diff = (ab - (2.5 * a - 0.5 * b)).abs().max().item()
    assert diff / a.abs().max().item() < 1e-13


def test_residual_zero_state():
    """b_u == 0 exactly and b_psi == phi_moments - exp_moments(0) at the zero state
    with f = 0 (reference tests/test_proximal.py:144-153, here in 2D)."""
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    from paper_2412_13733_b200.proximal import residual
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, 4, 3), 0.0, 2.0)
    z_psi, z_u = np.zeros(d.ndof_psi), np.zeros(d.ndof_u)
    b_u, b_psi, cl = residual(d, 0.5, z_psi, z_u, z_psi)
    assert not cl
    assert np.abs(b_u).max() == 0.0
    em, _ = d.exp_moments(z_psi)
    np.testing.assert_allclose(b_psi, d.phi_moments - em, atol=1e-15)


def test_cellwise_data_and_moments_from_values():
    """phi_mode='cellwise' broadcast and moments_from_values (assembly.py:308-317,528-533)."""
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    phi = lambda x, y: np.sin(x) * (1 + y)
    d = D.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, 3, 4), 1.0, phi, phi_mode="cellwise")
    t = d.tables
    P = orc.Problem("obstacle", d.xpts, d.ypts, 4,
                    SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))
    mx = 0.5 * (d.xpts[:-1] + d.xpts[1:])
    my = 0.5 * (d.ypts[:-1] + d.ypts[1:])
    vals = np.broadcast_to(phi(mx[:, None], my[None, :])[:, :, None, None],
                           (3, 3, t.nq, t.nq)).copy()
    assert orc.rel_err(d.phi_moments, P.data_moments(vals)) < TOL
    grids = d.quad_grids()
    samples = [phi(*np.meshgrid(gx, gy, indexing="ij")) for gx, gy in grids]
    assert orc.rel_err(d.moments_from_values(samples), P.data_moments(P.sample(phi))) < TOL


def _sample_cells(N, seed=0):
    rng = np.random.default_rng(seed)
    pick = {0, N - 1, N // 2, N // 3}
    while len(pick) < min(N, 8):
        pick.add(int(rng.integers(N)))
    return sorted(pick)


def _oracle_cell_block(cfg, P, inp, phi_vals, e):
    """The oracle's weighted block(s) of cell e (assembly.py:257-263, 550-557, 804-815)."""
    cx, cy = divmod(e, P.ncy)
    sl = (slice(cx, cx + 1), slice(cy, cy + 1))
    args = (P.t.S, P.t.T, P.wx[cx:cx + 1], P.wy[cy:cy + 1])
    if cfg.kind == "obstacle":
        tiles = P._tiles(inp["psi"])[sl]
        W, _ = orc.clamped_exp_neg(orc.synthesize(P.t.S, tiles))
        return orc.weighted_blocks(*args, W)[0]
    vx = orc.synthesize(P.t.S, P._tiles(inp["psi"], 0)[sl])
    vy = orc.synthesize(P.t.S, P._tiles(inp["psi"], 1)[sl])
    ph = phi_vals[sl]
    r2 = 1.0 + vx * vx + vy * vy
    inv, inv3 = r2 ** -0.5, r2 ** -1.5
    kxx, kxy, kyy = ph * (inv - vx * vx * inv3), ph * (-vx * vy * inv3), ph * (inv - vy * vy * inv3)
    Wxx, Wxy, Wyy = (orc.weighted_blocks(*args, k)[0] for k in (kxx, kxy, kyy))
    return np.block([[Wxx, Wxy], [Wxy, Wyy]])


@pytest.mark.parametrize("cfg_name,rule", ALL_PAIRS)
def test_full_size_blocks_sampled(cfg_name, rule):
    """Every cell's block in ONE assembly call on the full BASELINE mesh (c1:
    4096 cells through the persistent multi-wave block-row grid; c3: the
    two-GEMM path), sampled cells vs the oracle at 1e-12, and the dense-block
    matvec == the matrix-free cached apply on the whole mesh."""
    import torch
    cfg, d, P, inp, dev = build(cfg_name, rule)
    phi_vals = P.sample(inp["phi"])
    D = d.assemble_D_t(dev["psi"])
    blocks = D.blocks_t()
    torch.cuda.synchronize()
    for e in _sample_cells(d.plan.ncells):
        got = blocks[e].cpu().numpy()
        ref = _oracle_cell_block(cfg, P, inp, phi_vals, e)
        assert orc.rel_err(got, ref) < TOL, f"cell {e}"
    y_blk = D.matvec_blocks_t(dev["x"]).cpu().numpy()
    y_mf = D.matvec_t(dev["x"]).cpu().numpy()
    assert orc.rel_err(y_blk, y_mf) < TOL
    del blocks, D
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg_name,nslab", [("c1", 2), ("c2", 3), ("c4p4", 4)])
def test_slab_sharded_residual_on_one_gpu(cfg_name, nslab):
    """§8e on one GPU: the mesh split into slabs, each slab (plus two ghost cell
    columns) an independent device disc, ghost rows filled by the same halo
    exchange the multi-GPU path runs over NCCL; the stitched owned rows equal
    the single-disc residual and Jacobian apply."""
    import torch
    from paper_2412_13733_b200 import dist as hd
    from paper_2412_13733_b200 import disc as D
    from paper_2412_13733_b200.mesh import Mesh1D, TensorMesh2D
    cfg, d, P, inp, dev = build(cfg_name)
    alpha = cfg.alphas[-1]
    gb_u, gb_psi, gflag = d.residual_t(alpha, dev["psi_prev"], dev["u"], dev["psi"], wcache=True)
    gy = d.apply_cached_t(dev["x"])
    hs = [hd.SlabHalo(cfg.ncells, cfg.ncells, cfg.p, cfg.kind, nslab, r) for r in range(nslab)]
    cls = D.ObstacleDisc2D if cfg.kind == "obstacle" else D.GradientDisc2D
    loc = {k: [] for k in ("psi", "psi_prev", "u", "x")}
    discs = []
    for h in hs:
        m = TensorMesh2D(Mesh1D(h.local_points(d.xpts), np.full(h.ncx_local, cfg.p)),
                         Mesh1D(d.ypts, np.full(cfg.ncells, cfg.p)))
        discs.append(cls(m, inp["f"], inp["phi"], rule="gauss", nq=cfg.Q))
        for k in ("psi", "psi_prev", "x"):
            t = torch.from_numpy(h.local_psi(inp[k]).copy()).cuda()
            loc[k].append(t)
        loc["u"].append(torch.from_numpy(h.local_u(inp["u"]).copy()).cuda())
    # ghost rows zeroed, then filled by the halo exchange
    for r, h in enumerate(hs):
        for k in ("psi", "psi_prev"):
            v = h.psi_view(loc[k][r])
            keep = v[:, h.own_psi_local].clone()
            v.zero_()
            v[:, h.own_psi_local] = keep
        uv = h.u_view(loc["u"][r])
        keep = uv[h.own_u_local].clone()
        uv.zero_()
        uv[h.own_u_local] = keep
    hd.exchange_in_process(hs, [loc["psi"], loc["psi_prev"]], [loc["u"]])
    bu = torch.full_like(gb_u, float("nan")).view(-1, hs[0].niy)
    bpsi = torch.full_like(gb_psi, float("nan")).view(cfg.ncomp, -1, hs[0].ld)
    y = torch.full_like(gy, float("nan")).view(cfg.ncomp, -1, hs[0].ld)
    for r, (h, dd) in enumerate(zip(hs, discs)):
        b_u, b_psi, _ = dd.residual_t(alpha, loc["psi_prev"][r], loc["u"][r], loc["psi"][r], wcache=True)
        yl = dd.apply_cached_t(loc["x"][r])
        bu[torch.from_numpy(h.own_u_rows).cuda()] = h.owned_u(b_u)
        bpsi[:, torch.from_numpy(h.own_psi_rows).cuda()] = h.owned_psi(b_psi)
        y[:, torch.from_numpy(h.own_psi_rows).cuda()] = h.owned_psi(yl)
    assert orc.rel_err(bu.reshape(-1).cpu().numpy(), gb_u.cpu().numpy()) < 1e-13
    assert orc.rel_err(bpsi.reshape(-1).cpu().numpy(), gb_psi.cpu().numpy()) < 1e-13
    assert orc.rel_err(y.reshape(-1).cpu().numpy(), gy.cpu().numpy()) < 1e-13
