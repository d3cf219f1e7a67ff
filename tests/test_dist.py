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
