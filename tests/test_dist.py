"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 path's host logic,
and the sharding claim behind it: the psi side of the path is element-local,
so slabs of cells computed independently reproduce the global result."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import torch.multiprocessing as mp

from oracle import hpg_oracle as orc
from paper_2412_13733_b200 import dist as D
from paper_2412_13733_b200.tables import Tables
from paper_2412_13733_b200.workloads import make_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    r, w, _ = D.init("gloo")
    D.barrier()
    mx = D.max_over_ranks(1.5 + r)
    x0, x1 = D.slab(10, w, r)
    out[r] = (r, w, mx, x0, x1, D.aggregate_throughput(100, 3, w, mx))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_gloo_world2_timing_and_slabs():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][2] == res[1][2] == 2.5           # max over ranks
    assert (res[0][3], res[0][4], res[1][3], res[1][4]) == (0, 5, 5, 10)
    assert res[0][5] == 100 * 3 * 2 / 2.5


def test_slab_partition_covers():
    for ncx in (1, 7, 64, 256):
        for world in (1, 2, 3, 8):
            spans = [D.slab(ncx, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == ncx
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_psi_side_is_element_local():
    """exp moments and D(psi) x of a 6x4 mesh == concatenation over x-slabs."""
    p, ncx, ncy = 5, 6, 4
    t = Tables("gauss", p, p - 1, 8)
    tt = SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq)
    xs = np.linspace(0.0, 1.0, ncx + 1)
    ys = np.linspace(0.0, 1.0, ncy + 1)
    psi, _, x, _ = make_inputs("obstacle", ncx, ncy, p, seed=3)
    G = orc.Problem("obstacle", xs, ys, p, tt)
    m_glob, _ = G.exp_moments(psi)
    y_glob = G.obstacle_apply_D(psi, x)
    n = p - 1
    rows = ncy * n
    parts_m, parts_y = [], []
    for r in range(3):
        x0, x1 = D.slab(ncx, 3, r)
        L = orc.Problem("obstacle", xs[x0:x1 + 1], ys, p, tt)
        sl = slice(x0 * n * rows, x1 * n * rows)
        parts_m.append(L.exp_moments(psi[sl])[0])
        parts_y.append(L.obstacle_apply_D(psi[sl], x[sl]))
    assert orc.rel_err(np.concatenate(parts_m), m_glob) < 1e-15
    assert orc.rel_err(np.concatenate(parts_y), y_glob) < 1e-15


# ---------------------------------------------------------------------------
# §8e: one mesh sharded over ranks (slabs + two ghost columns + halo exchange)

def _problem(kind, xs, ys, p, nq=None):
    n = p - 1 if kind == "obstacle" else p
    t = Tables("gauss", p, n, nq or p + 3)
    return orc.Problem(kind, xs, ys, p, SimpleNamespace(S=t.S, T=t.T, Su=t.Su, Tu=t.Tu, xi=t.xi, nq=t.nq))


def _phi(x, y):
    return 0.2 + 0.1 * np.sin(np.pi * x) * np.sin(np.pi * y)


def _local_residual(kind, h, xs, ys, p, alpha, psi_prev, u, psi):
    """The oracle's residual on the rank's extended slab (the computation each
    GPU runs with the unchanged single-GPU path)."""
    L = _problem(kind, h.local_points(xs), ys, p)
    f_load = L.load_vector(L.sample(1.0))
    if kind == "obstacle":
        return L.residual(alpha, psi_prev, u, psi, f_load, phi_moments=L.data_moments(L.sample(_phi)))
    return L.residual(alpha, psi_prev, u, psi, f_load, phi_vals=L.sample(_phi))


def _sharded_worker(rank, world, port, kind, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    D.init("gloo")
    p, ncx, ncy = 4, 7, 3
    xs, ys = np.linspace(0, 1, ncx + 1), np.linspace(0, 1, ncy + 1)
    psi, u, _, _ = make_inputs(kind, ncx, ncy, p, seed=2)
    psi_prev = 0.3 * np.roll(psi, 5)
    h = D.SlabHalo(ncx, ncy, p, kind, world, rank)
    loc = {}
    for name, g, like in (("psi", psi, "psi"), ("psi_prev", psi_prev, "psi"), ("u", u, "u")):
        t = torch.from_numpy((h.local_psi(g) if like == "psi" else h.local_u(g)).copy())
        # ghost rows hold garbage until the exchange fills them
        own = np.zeros(t.numel(), bool)
        if like == "psi":
            v = own.reshape(h.ncomp, -1, h.ld)
            v[:, h.own_psi_local] = True
        else:
            own.reshape(-1, h.niy)[h.own_u_local] = True
        t[torch.from_numpy(~own)] = float("nan")
        loc[name] = t
    h.exchange(psi_like=[loc["psi"], loc["psi_prev"]], u_like=[loc["u"]])
    b_u, b_psi, cl = _local_residual(kind, h, xs, ys, p, 1.7, loc["psi_prev"].numpy(), loc["u"].numpy(),
                                     loc["psi"].numpy())
    out[rank] = (h.own_u_rows, h.owned_u(b_u), h.own_psi_rows, h.owned_psi(b_psi), bool(cl))
    import torch.distributed as dist
    dist.destroy_process_group()


def _stitch(res, kind, ncx, ncy, p):
    n = p - 1 if kind == "obstacle" else p
    nc = 1 if kind == "obstacle" else 2
    niy = ncy * p - 1
    bu = np.full((ncx * p - 1, niy), np.nan)
    bpsi = np.full((nc, ncx * n, ncy * n), np.nan)
    for r in sorted(res):
        urows, uvals, prows, pvals, _ = res[r]
        bu[urows] = uvals
        bpsi[:, prows] = pvals
    return bu.ravel(), bpsi.ravel()


def test_gloo_world2_sharded_residual_equals_global():
    """Two ranks (gloo, CPU) each own a slab, exchange the ghost rows of psi,
    psi_prev and u, run the residual on their extended slab; the stitched
    owned rows equal the global residual (b_u across the shared hat line too)."""
    world = 2
    p, ncx, ncy = 4, 7, 3
    for kind in ("obstacle", "gradient"):
        port = _free_port()
        with mp.Manager() as mgr:
            out = mgr.dict()
            mp.spawn(_sharded_worker, args=(world, port, kind, out), nprocs=world, join=True)
            res = dict(out)
        xs, ys = np.linspace(0, 1, ncx + 1), np.linspace(0, 1, ncy + 1)
        psi, u, _, _ = make_inputs(kind, ncx, ncy, p, seed=2)
        psi_prev = 0.3 * np.roll(psi, 5)
        G = _problem(kind, xs, ys, p)
        f_load = G.load_vector(G.sample(1.0))
        if kind == "obstacle":
            gb_u, gb_psi, _ = G.residual(1.7, psi_prev, u, psi, f_load, phi_moments=G.data_moments(G.sample(_phi)))
        else:
            gb_u, gb_psi, _ = G.residual(1.7, psi_prev, u, psi, f_load, phi_vals=G.sample(_phi))
        bu, bpsi = _stitch(res, kind, ncx, ncy, p)
        assert not np.isnan(bu).any() and not np.isnan(bpsi).any()      # every row owned once
        assert orc.rel_err(bu, gb_u) < 1e-14, kind
        assert orc.rel_err(bpsi, gb_psi) < 1e-14, kind


def test_slab_halo_ownership_partition():
    """Owned rows of all ranks partition the global psi and u rows; every
    ghost row of a rank is owned by an adjacent rank."""
    for kind, p, ncx, ncy, world in (("obstacle", 2, 16, 4, 8), ("obstacle", 6, 9, 2, 4),
                                     ("gradient", 3, 8, 3, 3), ("obstacle", 16, 64, 64, 8)):
        hs = [D.SlabHalo(ncx, ncy, p, kind, world, r) for r in range(world)]
        n = p - 1 if kind == "obstacle" else p
        own_psi = np.concatenate([h.own_psi_rows for h in hs])
        own_u = np.concatenate([h.own_u_rows for h in hs])
        assert np.array_equal(np.sort(own_psi), np.arange(ncx * n))
        assert np.array_equal(np.sort(own_u), np.arange(ncx * p - 1))
        for h in hs:
            ghost_u = np.setdiff1d(h.u_rows, h.own_u_rows)
            recv_u = np.concatenate([h.u_rows[pl["recv_u"]] for pl in h.peers.values()] + [np.array([], int)])
            assert np.array_equal(np.sort(recv_u), ghost_u)
            ghost_p = np.setdiff1d(h.psi_rows, h.own_psi_rows)
            recv_p = np.concatenate([h.psi_rows[pl["recv_psi"]] for pl in h.peers.values()] + [np.array([], int)])
            assert np.array_equal(np.sort(recv_p), ghost_p)
