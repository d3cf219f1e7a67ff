"""Multi-GPU sharding of one mesh: one process per GPU.

Partition: contiguous slabs of cell columns ``cx in [x0, x1)`` per rank
(``slab``).  The psi side is element-local (Psi is cellwise discontinuous,
``spaces.py:89-108``); the u side shares hat dofs between neighbouring cells
(``spaces.py:25-43``), so ``b_u`` on the vertical hat line of a slab
interface sums contributions from cells on both ranks.

``SlabHalo`` makes every rank's share an ordinary single-GPU problem: the
rank runs the unchanged device path on its slab EXTENDED by two ghost cell
columns per interior side, ``[a, b) = [max(0, x0-2), min(ncx, x1+2))``.  The
first ghost column makes the interface hat line an interior dof of the local
mesh, so ``b_u`` there gets both cells' contributions locally; the second one
makes the ghost cell's own far hat line a local dof too (a local mesh treats
its boundary hat lines as Dirichlet zeros).  Before a residual the ghost rows
of the inputs (psi, psi_prev, u) are exchanged with the two neighbours
(NCCL send/recv over NVLink, or gloo on the CPU); afterwards each rank keeps
the rows it owns.  The Krylov matvecs D(psi) x need no exchange (element-
local).  Everything is expressed in GLOBAL row indices, so both sides of an
exchange derive the same ordered row lists independently:

* psi: x-major rows ``[c n, (c+1) n)`` of cell column c, per component
  (row length ``ncy n``);
* u: rows of the (nix x niy) interior array; the 1D x-interior numbering is
  hat lines 1..ncx-1 (row = line-1) then the p-1 bubbles of each cell
  (row = ncx-1 + c (p-1) + k) -- a local mesh of cells [a, b) uses exactly
  the ascending global rows of its interior lines and cells.

Ownership: a rank owns its cells' psi rows and bubble rows and the hat lines
``x0 .. x1-1`` (line 0 and line ncx are Dirichlet).
"""

import os

import numpy as np
import torch
import torch.distributed as dist

GHOST = 2


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend):
    """Initialise the default process group from the torchrun environment."""
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        kw = {}
        if backend == "nccl":
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


def slab(ncx, world, rank):
    """Contiguous cell-column range [x0, x1) of a rank (balanced to one column)."""
    base, extra = divmod(ncx, world)
    x0 = rank * base + min(rank, extra)
    return x0, x0 + base + (1 if rank < extra else 0)


def _u_rows(ncx, p, c0, c1, own_lines=None):
    """Ascending global u rows of the interior of cells [c0, c1) (or, with
    own_lines=(l0, l1), the hat lines l0..l1-1 instead of c0+1..c1-1)."""
    l0, l1 = own_lines if own_lines is not None else (c0 + 1, c1)
    lines = np.arange(max(l0, 1), min(l1, ncx))
    if p == 1:
        return lines - 1
    bub = (ncx - 1) + (np.arange(c0, c1)[:, None] * (p - 1) + np.arange(p - 1)[None, :]).ravel()
    return np.concatenate([lines - 1, bub]).astype(np.int64)


class SlabHalo:
    """Rank ``rank``'s extended slab of an ncx x ncy, degree-p mesh."""

    def __init__(self, ncx, ncy, p, kind, world, rank, ghost=GHOST):
        if world > 1 and ncx < 2 * world:
            raise ValueError("need at least two cell columns per rank")
        self.ncx, self.ncy, self.p, self.kind = ncx, ncy, p, kind
        self.world, self.rank = world, rank
        self.n = p - 1 if kind == "obstacle" else p
        self.ncomp = 1 if kind == "obstacle" else 2
        self.ld = ncy * self.n
        self.x0, self.x1 = slab(ncx, world, rank)
        self.a, self.b = max(0, self.x0 - ghost), min(ncx, self.x1 + ghost)
        self.niy = ncy * p - 1 if p > 1 else ncy - 1
        # global row lists of the local (extended) arrays and of the owned part
        self.psi_rows = np.arange(self.a * self.n, self.b * self.n)
        self.u_rows = _u_rows(ncx, p, self.a, self.b)
        self.own_psi_rows = np.arange(self.x0 * self.n, self.x1 * self.n)
        self.own_u_rows = _u_rows(ncx, p, self.x0, self.x1, own_lines=(self.x0, self.x1))
        self.own_psi_local = np.searchsorted(self.psi_rows, self.own_psi_rows)
        self.own_u_local = np.searchsorted(self.u_rows, self.own_u_rows)
        assert np.array_equal(self.u_rows[self.own_u_local], self.own_u_rows)
        # exchange plans with the neighbours (global rows, ascending)
        self.peers = {}
        for q in (rank - 1, rank + 1):
            if 0 <= q < world:
                other = SlabHalo.__new__(SlabHalo)
                other._rows_only(ncx, ncy, p, kind, world, q, ghost)
                send_psi = np.intersect1d(other.psi_rows, self.own_psi_rows)
                recv_psi = np.intersect1d(self.psi_rows, other.own_psi_rows)
                send_u = np.intersect1d(other.u_rows, self.own_u_rows)
                recv_u = np.intersect1d(self.u_rows, other.own_u_rows)
                self.peers[q] = {
                    "send_psi": np.searchsorted(self.psi_rows, send_psi),
                    "recv_psi": np.searchsorted(self.psi_rows, recv_psi),
                    "send_u": np.searchsorted(self.u_rows, send_u),
                    "recv_u": np.searchsorted(self.u_rows, recv_u),
                }
        self._dev_idx = {}

    def _rows_only(self, ncx, ncy, p, kind, world, rank, ghost):
        n = p - 1 if kind == "obstacle" else p
        x0, x1 = slab(ncx, world, rank)
        a, b = max(0, x0 - ghost), min(ncx, x1 + ghost)
        self.psi_rows = np.arange(a * n, b * n)
        self.u_rows = _u_rows(ncx, p, a, b)
        self.own_psi_rows = np.arange(x0 * n, x1 * n)
        self.own_u_rows = _u_rows(ncx, p, x0, x1, own_lines=(x0, x1))

    # ------------------------------------------------------------- layouts
    @property
    def ncx_local(self):
        return self.b - self.a

    def local_points(self, xpts):
        """Breakpoints of the extended slab from the global ones."""
        return np.asarray(xpts)[self.a:self.b + 1]

    def psi_view(self, vec):
        """(ncomp, rows, ld) view of a local psi vector."""
        return vec.reshape(self.ncomp, -1, self.ld)

    def u_view(self, vec):
        return vec.reshape(-1, self.niy)

    def local_psi(self, glob):
        """Global psi vector -> local (extended) psi vector (for setup and tests)."""
        g = glob.reshape(self.ncomp, self.ncx * self.n, self.ld)
        return g[:, self.psi_rows].reshape(-1)

    def local_u(self, glob):
        return glob.reshape(-1, self.niy)[self.u_rows].reshape(-1)

    def owned_psi(self, loc):
        """Owned rows of a local psi vector, (ncomp, own_rows, ld) flattened per component."""
        return self.psi_view(loc)[:, self.own_psi_local]

    def owned_u(self, loc):
        return self.u_view(loc)[self.own_u_local]

    # ------------------------------------------------------------- halo exchange
    def _idx(self, key, q, device):
        k = (key, q, str(device))
        t = self._dev_idx.get(k)
        if t is None:
            t = torch.from_numpy(self.peers[q][key]).to(device)
            self._dev_idx[k] = t
        return t

    def exchange(self, psi_like=(), u_like=(), group=None):
        """Fill the ghost rows of local psi-shaped and u-shaped tensors from
        the neighbours' owned rows (torch.distributed send/recv; NCCL on the
        GPU, gloo on the CPU).  Returns after the receives complete."""
        ops, recvs = [], []
        for q in sorted(self.peers):
            for kind, tensors in (("psi", psi_like), ("u", u_like)):
                for t in tensors:
                    view = self.psi_view(t) if kind == "psi" else self.u_view(t)
                    dim = 1 if kind == "psi" else 0
                    si = self._idx("send_" + kind, q, t.device)
                    ri = self._idx("recv_" + kind, q, t.device)
                    if si.numel():
                        ops.append(dist.P2POp(dist.isend, view.index_select(dim, si).contiguous(), q, group))
                    if ri.numel():
                        buf = torch.empty_like(view.index_select(dim, ri))
                        ops.append(dist.P2POp(dist.irecv, buf, q, group))
                        recvs.append((view, dim, ri, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for view, dim, ri, buf in recvs:
            view.index_copy_(dim, ri, buf)


def exchange_in_process(halos, psi_like, u_like):
    """The same exchange between SlabHalo objects of ONE process: ``psi_like``
    / ``u_like`` are lists of fields, each a list of the ranks' local tensors
    (single-GPU slab tests)."""
    for r, h in enumerate(halos):
        for q, plan in h.peers.items():
            src = halos[q]
            mine = src.peers[r]
            for kind, fields in (("psi", psi_like), ("u", u_like)):
                for per_rank in fields:
                    dst_t, src_t = per_rank[r], per_rank[q]
                    if kind == "psi":
                        dv, sv, dim = h.psi_view(dst_t), src.psi_view(src_t), 1
                    else:
                        dv, sv, dim = h.u_view(dst_t), src.u_view(src_t), 0
                    si = torch.as_tensor(mine["send_" + kind], device=sv.device)
                    ri = torch.as_tensor(plan["recv_" + kind], device=dv.device)
                    if ri.numel():
                        dv.index_copy_(dim, ri, sv.index_select(dim, si))


def barrier(device=None):
    if dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None and device.type == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (the timing rule: slowest rank wins)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank, steps, world, max_seconds):
    """Whole-job throughput: units all ranks processed / slowest rank's time."""
    return units_per_rank * steps * world / max_seconds
