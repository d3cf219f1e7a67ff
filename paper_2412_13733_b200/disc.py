"""Device-backed discretisations: the reference's solver-facing API on the B200 path.

``ObstacleDisc2D`` / ``GradientDisc2D`` mirror ``hpgalerkin/assembly.py:452-603``
and ``:699-860`` for the hot-path members: the same constructor arguments,
the same method names, the same argument meaning and the same returned arrays
(global x-major psi order, interior U order, cell order (cx, cy) cx-major).
Every computation runs in ``libhpg_b200.so`` (sm_100a CUDA kernels behind the
C ABI of ``include/hpg_b200.h``); there is no CPU fallback.

Two API levels:

* reference-facing (NumPy in / NumPy out, host buffers): ``exp_moments``,
  ``nl_moments``, ``apply_D``, ``assemble_D``, ``data_moments``,
  ``moments_from_values``, ``load_vector`` and ``proximal.residual`` -- the
  drop-in seam;
* device-resident (torch CUDA tensors, asynchronous on the current stream):
  the ``*_t`` methods, used by the benchmark and by callers that keep the
  Newton state on the GPU.
"""

import ctypes
import os
import weakref

import numpy as np
import torch

from . import _lib
from .tables import Tables, schur_triple_factors

F64 = torch.float64


def _vp(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def pinned_array(shape):
    """A float64 NumPy array in page-locked host memory.  Vectors a caller
    keeps in such arrays are uploaded by ONE DMA straight from the array (no
    staging copy: 0.14 ms instead of 0.22-0.33 ms for config 1's 7.4 MB
    vector); the NumPy-facing methods return their large results in arrays
    of this kind as well, so an iteration's vectors stay page-locked."""
    n = int(np.prod(shape))
    t = torch.empty(max(n, 1), dtype=F64, pin_memory=True)
    return t.numpy()[:n].reshape(shape)


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.HpgError("paper_2412_13733_b200 needs a CUDA device (no CPU fallback)")


class Plan:
    """Owns one ``hpgPlan`` (device tables + geometry + workspaces)."""

    def __init__(self, kind, ncx, ncy, p, tables, hx, hy):
        _require_cuda()
        lib = _lib.load()
        self._lib = lib
        arrs = [np.ascontiguousarray(a, dtype=np.float64)
                for a in (tables.S, tables.T, tables.Su, tables.Tu, hx, hy)]
        h = ctypes.c_void_p()
        _lib.call("hpgPlanCreate", ctypes.byref(h), kind, ncx, ncy, p, tables.nq,
                  *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs])
        self.handle = h
        info = (ctypes.c_longlong * 12)()
        _lib.call("hpgPlanInfo", h, info)
        (self.n, self.m, self.nq, self.ncells, self.ndof_psi, self.ndof_u,
         self.wcache_len, self.block_len, self.path, self.splits,
         self.residual_apply_kernels, self.fused_apply) = [int(v) for v in info]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.hpgPlanDestroy(h)
            except Exception:
                pass
            self.handle = None


class _DeviceDisc:
    dim = 2

    def __init__(self, mesh2d, f, phi, f_mode="pointwise", phi_mode="pointwise",
                 rule="reference", nq=None):
        _require_cuda()
        mx, my = mesh2d.mesh_x, mesh2d.mesh_y
        degs = np.unique(np.concatenate([np.asarray(mx.degrees), np.asarray(my.degrees)]))
        if self.kind == "obstacle" and np.any(degs < 2):
            raise ValueError("obstacle discretization requires p >= 2")
        if degs.size != 1:
            raise ValueError("the B200 path needs one polynomial degree on every cell "
                             f"(got degrees {degs.tolist()})")
        self.mesh = mesh2d
        self.p = int(degs[0])
        self.n = self.p - 1 if self.kind == "obstacle" else self.p
        self.m = self.p + 1
        self.rule = rule
        self.tables = Tables(rule, self.p, self.n, nq)
        self.xpts = np.asarray(mx.points, dtype=float)
        self.ypts = np.asarray(my.points, dtype=float)
        self.ncx = self.xpts.size - 1
        self.ncy = self.ypts.size - 1
        self.hx = np.diff(self.xpts)
        self.hy = np.diff(self.ypts)
        kind = _lib.HPG_OBSTACLE if self.kind == "obstacle" else _lib.HPG_GRADIENT
        self.plan = Plan(kind, self.ncx, self.ncy, self.p, self.tables, self.hx, self.hy)
        self.nquad = self.tables.nq
        self.ncomp_dofs = self.ncx * self.n * self.ncy * self.n
        self.ndof_psi = self.plan.ndof_psi
        self.ndof_u = self.plan.ndof_u
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._wcache = torch.empty(self.plan.wcache_len, dtype=F64, device=self.device)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._pinned = {}
        self._devbuf = {}
        self._events = {}
        self._cell_psi_indices = None
        wx = np.concatenate([h / (2.0 * np.arange(self.n) + 1.0) for h in self.hx])
        wy = np.concatenate([h / (2.0 * np.arange(self.n) + 1.0) for h in self.hy])
        mass = np.kron(wx, wy)
        self.mass_psi = mass if self.kind == "obstacle" else np.concatenate([mass, mass])
        self.f_load_t = self.load_vector_t(self.sample_t(f, f_mode))
        self.f_load = self.f_load_t.cpu().numpy()

    # ------------------------------------------------------------------ layout
    @property
    def cell_ids(self):
        return [(cx, cy) for cx in range(self.ncx) for cy in range(self.ncy)]

    def _scalar_cell_indices(self):
        n, ndof_y = self.n, self.ncy * self.n
        ax = np.arange(n)
        out = []
        for cx in range(self.ncx):
            ix = (cx * n + ax) * ndof_y
            for cy in range(self.ncy):
                out.append(np.add.outer(ix, cy * n + ax).ravel())
        return out

    @property
    def cell_psi_indices(self):
        """Global psi indices per cell, in cell order (``assembly.py:489,744``)."""
        if self._cell_psi_indices is None:
            sc = self._scalar_cell_indices()
            if self.kind == "obstacle":
                self._cell_psi_indices = sc
            else:
                self._cell_psi_indices = [np.concatenate([i, i + self.ncomp_dofs]) for i in sc]
        return self._cell_psi_indices

    def quad_grids(self):
        """Per-cell (x axis, y axis) quadrature points, in cell order (``assembly.py:524``)."""
        gx, gy = self._grids()
        return [(gx[cx], gy[cy]) for cx, cy in self.cell_ids]

    def _grids(self):
        t = self.tables
        gx = np.stack([t.points(self.xpts[i], self.xpts[i + 1]) for i in range(self.ncx)])
        gy = np.stack([t.points(self.ypts[i], self.ypts[i + 1]) for i in range(self.ncy)])
        return gx, gy

    # --------------------------------------------------------------- transfers
    def _pin(self, tag, n):
        b = self._pinned.get(tag)
        if b is None or b.numel() < n:
            b = torch.empty(max(n, 1), dtype=F64, pin_memory=True)
            self._pinned[tag] = b
        return b[:n]

    def _dev(self, tag, n):
        b = self._devbuf.get(tag)
        if b is None or b.numel() < n:
            b = torch.empty(max(n, 1), dtype=F64, device=self.device)
            self._devbuf[tag] = b
        return b[:n]

    # Host<->device transfers of the reference-facing API.  Measured on the
    # B200 boxes (tools/xfer_bench2.py, tools/e2e_slab_probe.py, 7.4 MB): a
    # direct pageable copy runs at 17.7 GB/s H2D / 14.5 GB/s D2H; one DMA from
    # / to page-locked memory at 54 GB/s (0.137 ms), both directions at once
    # at 0.153 ms.  The multi-threaded host copy (torch) into the page-locked
    # staging buffer runs at 53 GB/s when the source is not cache resident, so
    # uploads stage through two half-size buffers (the copy of one half
    # overlapping the DMA of the other: 0.22 ms; one chunk 0.28, four 0.27,
    # eight 0.44 -- every extra DMA / event costs ~20 us on these boxes).
    # Small vectors go direct.
    _STAGE_MIN = 1 << 17          # doubles (1 MB): uploads below go direct (pageable)
    _CHUNK_MIN = 1 << 19          # doubles (4 MB): uploads below stage as one chunk
    _PIN_OUT_MIN = 1 << 14        # doubles (128 KB): results below come back pageable
                                  # (c3's 0.84 MB vector: direct 0.086 ms, page-locked 0.048 ms)

    _H2D_CHUNKS = int(os.environ.get("HPG_H2D_CHUNKS", "2"))

    def _stage_buf(self, n, count=2):
        st = getattr(self, "_stage", None)
        if st is None or st["n"] < n or len(st["buf"]) < count:
            if st is not None:                       # both users keep fitting
                n, count = max(n, st["n"]), max(count, len(st["buf"]))
                torch.cuda.synchronize()
            st = {"n": n, "buf": [torch.empty(n, dtype=F64, pin_memory=True) for _ in range(count)],
                  "ev": [None] * count}
            self._stage = st
        return st

    def h2d(self, arr, tag, defer_sync=False):
        """Host array -> (reused) device tensor."""
        a = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1)
        dev = self._dev("in_" + tag, a.size)
        n = a.size
        if n >= self._PIN_OUT_MIN:
            at = torch.from_numpy(a)
            if at.is_pinned():
                # page-locked source (pinned_array, or one of our own results):
                # one DMA from the caller's memory; it must not change before
                # the copy is done, so the transfer is finished here unless the
                # caller synchronises before it returns anyway
                dev.copy_(at, non_blocking=True)
                if not defer_sync:
                    torch.cuda.current_stream().synchronize()
                return dev
        if n < self._STAGE_MIN:
            dev.copy_(torch.from_numpy(a))
            return dev
        # pipelined: the host copy of chunk i + 1 into its page-locked buffer
        # overlaps the DMA of chunk i
        nch = self._H2D_CHUNKS if n >= self._CHUNK_MIN else 1
        step = (n + nch - 1) // nch
        st = self._stage_buf(step, nch)
        at = torch.from_numpy(a)
        for i in range(nch):
            lo, hi = i * step, min(n, (i + 1) * step)
            if lo >= hi:
                break
            if st["ev"][i] is not None:
                st["ev"][i].synchronize()          # the buffer's previous DMA is done
            st["buf"][i][:hi - lo].copy_(at[lo:hi])
            dev[lo:hi].copy_(st["buf"][i][:hi - lo], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            st["ev"][i] = ev
        return dev

    # Large results come back in page-locked memory of their own: the DMA
    # writes the fresh array directly (no staging copy, no first-touch page
    # faults of a new pageable block: 30.7 -> ~50 GB/s).  The block belongs to
    # the returned array (its base keeps the tensor alive) and goes back to
    # torch's caching host allocator when the caller drops the array.  Page-
    # locked results still held by the caller are capped; beyond the cap the
    # staged pageable path is used.
    _PINNED_OUT_CAP = 4 << 30     # bytes
    _pinned_out_bytes = 0

    @classmethod
    def _pinned_out_release(cls, nbytes):
        cls._pinned_out_bytes -= nbytes

    def h2d_many(self, arrs, tags, defer_sync=False):
        """Several host arrays -> device tensors.  Small / mid-size arrays
        (each below the chunking threshold) are packed into one page-locked
        staging buffer and uploaded by ONE DMA into one device buffer (the
        results are 256-byte aligned views of it); large ones go one by one
        through the pipelined path."""
        flat = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in arrs]
        if all(a.size >= self._PIN_OUT_MIN and torch.from_numpy(a).is_pinned() for a in flat):
            return [self.h2d(a, t, defer_sync=defer_sync) for a, t in zip(flat, tags)]
        if any(a.size >= self._CHUNK_MIN for a in flat) or sum(a.size for a in flat) < 64:
            return [self.h2d(a, t) for a, t in zip(flat, tags)]
        offs, total = [], 0
        for a in flat:
            offs.append(total)
            total += (a.size + 31) // 32 * 32
        st = self._stage_buf(total, 1)
        if st["ev"][0] is not None:
            st["ev"][0].synchronize()
        pin = st["buf"][0]
        for a, o in zip(flat, offs):
            if a.size:
                pin[o:o + a.size].copy_(torch.from_numpy(a))
        dev = self._dev("in_many_" + "_".join(tags), total)
        dev.copy_(pin[:total], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        st["ev"][0] = ev
        return [dev[o:o + a.size] for a, o in zip(flat, offs)]

    def d2h_many(self, tensors, flag=None):
        """Several device tensors -> fresh host arrays with ONE stream
        synchronisation (page-locked results enqueued back to back); ``flag``
        (a device int tensor) comes back as a Python int the same way."""
        cls = _DeviceDisc
        outs, pend = [], []
        for t in tensors:
            t = t.reshape(-1)
            n = t.numel()
            if (n >= self._PIN_OUT_MIN and cls._pinned_out_bytes + 8 * n <= cls._PINNED_OUT_CAP
                    and os.environ.get("HPG_NO_PINNED_OUT") is None):
                buf = torch.empty(n, dtype=F64, pin_memory=True)
                buf.copy_(t, non_blocking=True)
                cls._pinned_out_bytes += 8 * n
                outs.append(None)
                pend.append((len(outs) - 1, buf, n))
            else:
                outs.append(self.d2h(t, "many"))
        fbuf = None
        if flag is not None:
            fbuf = self._pinned.get("flag_out")
            if fbuf is None:
                fbuf = self._pinned["flag_out"] = torch.empty(1, dtype=torch.int32, pin_memory=True)
            fbuf.copy_(flag.reshape(-1)[:1], non_blocking=True)
        if pend or fbuf is not None:
            torch.cuda.current_stream().synchronize()
        for i, buf, n in pend:
            arr = buf.numpy()
            weakref.finalize(arr, cls._pinned_out_release, 8 * n)
            outs[i] = arr
        return outs, (int(fbuf[0]) if fbuf is not None else None)

    def d2h(self, t, tag):
        """Device tensor -> fresh host array (the reference returns fresh arrays)."""
        t = t.reshape(-1)
        n = t.numel()
        if n < self._PIN_OUT_MIN:
            out = np.empty(n)
            torch.from_numpy(out).copy_(t)
            return out
        cls = _DeviceDisc
        if cls._pinned_out_bytes + 8 * n <= cls._PINNED_OUT_CAP and os.environ.get("HPG_NO_PINNED_OUT") is None:
            buf = torch.empty(n, dtype=F64, pin_memory=True)
            buf.copy_(t, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            out = buf.numpy()
            cls._pinned_out_bytes += 8 * n
            weakref.finalize(out, cls._pinned_out_release, 8 * n)
            return out
        out = np.empty(n)
        half = (n + 1) // 2
        st = self._stage_buf(half)
        ot = torch.from_numpy(out)
        parts = ((0, half), (half, n))
        evs = []
        for i, (lo, hi) in enumerate(parts):
            if st["ev"][i] is not None:
                st["ev"][i].synchronize()
            st["buf"][i][:hi - lo].copy_(t[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            evs.append(ev)
        for i, (lo, hi) in enumerate(parts):
            evs[i].synchronize()                   # half i landed; half i+1 still in flight
            ot[lo:hi].copy_(st["buf"][i][:hi - lo])
            st["ev"][i] = None
        return out

    # D @ x with host buffers, pipelined over slabs of cell columns.  D is
    # block diagonal over cells and a slab of whole cell columns is a
    # contiguous row range of the x-major vectors, so slab k uploads (copy
    # stream) while slab k - 1 is applied and downloaded (compute stream):
    # both PCIe directions are busy at once, and the result lands directly in
    # a page-locked array of its own (see d2h).
    _SLABS = int(os.environ.get("HPG_MATVEC_SLABS", "2"))   # c1, per D @ x: 2 slabs 0.41 ms, 1: 0.43, 3: 0.41, 4: 0.50

    def host_matvec_cached(self, x, wcache):
        a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        n = a.size
        self._check_len(torch.from_numpy(a), self.ndof_psi, "x")
        cls = _DeviceDisc
        S = min(self._SLABS, self.ncx)
        if n >= self._PIN_OUT_MIN and torch.from_numpy(a).is_pinned():
            # page-locked x: upload straight from it, no slabs (d2h synchronises)
            y = self.apply_cached_t(self.h2d(a, "x", defer_sync=True), out=self._dev("out_y", n), wcache=wcache)
            return self.d2h(y, "y")
        if (S < 2 or n < 2 * self._STAGE_MIN or self.plan.path != 0
                or cls._pinned_out_bytes + 8 * n > cls._PINNED_OUT_CAP
                or os.environ.get("HPG_NO_PINNED_OUT") is not None):
            y = self.apply_cached_t(self.h2d(a, "x"), out=self._dev("out_y", n), wcache=wcache)
            return self.d2h(y, "y")
        dev_x, dev_y = self._dev("in_x", n), self._dev("out_y", n)
        out = torch.empty(n, dtype=F64, pin_memory=True)
        cur = torch.cuda.current_stream()
        up = getattr(self, "_up_stream", None)
        if up is None:
            up = self._up_stream = torch.cuda.Stream()
        up.wait_stream(cur)                    # earlier readers of dev_x are done
        at = torch.from_numpy(a)
        rows = self.n * self.ncy * self.n      # doubles per cell column and component
        bounds = [self.ncx * k // S for k in range(S + 1)]
        st = self._stage_buf(max(bounds[k + 1] - bounds[k] for k in range(S)) * rows * self.ncomp, S)
        for k in range(S):
            cx0, cx1 = bounds[k], bounds[k + 1]
            ln = (cx1 - cx0) * rows
            # uploads of an earlier call of this method finished before it
            # returned; h2d() shares the buffers and leaves an event behind
            if st["ev"][k] is not None:
                st["ev"][k].synchronize()
                st["ev"][k] = None
            for c in range(self.ncomp):
                lo = c * self.ncomp_dofs + cx0 * rows
                st["buf"][k][c * ln:(c + 1) * ln].copy_(at[lo:lo + ln])
            _lib.call("hpgApplyCachedHostSlab", self.plan.handle, _vp(wcache), _vp(st["buf"][k]), _vp(dev_x),
                      _vp(dev_y), _vp(out), cx0, cx1, ctypes.c_void_p(up.cuda_stream), _stream())
        cur.synchronize()
        res = out.numpy()
        cls._pinned_out_bytes += 8 * n
        weakref.finalize(res, cls._pinned_out_release, 8 * n)
        return res

    def _check_len(self, v, n, what):
        if v.numel() != n:
            raise ValueError(f"{what} has {v.numel()} entries, expected {n}")

    # ------------------------------------------------------------- data terms
    def sample(self, g, mode="pointwise"):
        """Point samples (ncells, nq, nq) of scalar data (``assembly.py:301-317``)."""
        nq = self.nquad
        shape = (self.ncx, self.ncy, nq, nq)
        if np.isscalar(g):
            return np.full(shape, float(g))
        gx, gy = self._grids()
        if mode == "cellwise":
            mx = 0.5 * (self.xpts[:-1] + self.xpts[1:])
            my = 0.5 * (self.ypts[:-1] + self.ypts[1:])
            vals = np.asarray(g(mx[:, None], my[None, :]), dtype=float)
            return np.broadcast_to(vals[:, :, None, None], shape).copy()
        X = np.broadcast_to(gx[:, None, :, None], shape)
        Y = np.broadcast_to(gy[None, :, None, :], shape)
        return np.array(np.broadcast_to(np.asarray(g(X, Y), dtype=float), shape), copy=True)

    def sample_t(self, g, mode="pointwise"):
        vals = self.sample(g, mode)
        return torch.from_numpy(vals.reshape(-1)).to(self.device)

    def moments_from_values_t(self, vals_t, out=None):
        out = torch.empty(self.ncomp_dofs, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgMomentsFromValues", self.plan.handle, _vp(vals_t), _vp(out), _stream())
        return out

    def load_vector_t(self, vals_t, out=None):
        out = torch.empty(self.ndof_u, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgLoadVector", self.plan.handle, _vp(vals_t), _vp(out), _stream())
        return out

    def data_moments(self, g, mode="pointwise"):
        """(g, zeta_i) over psi dofs (``assembly.py:514-519``)."""
        return self.moments_from_values_t(self.sample_t(g, mode)).cpu().numpy()

    def moments_from_values(self, values):
        """From per-cell grid samples in cell order (``assembly.py:528-533``)."""
        vals = np.ascontiguousarray(np.stack([np.asarray(v, dtype=float) for v in values]))
        return self.moments_from_values_t(torch.from_numpy(vals.reshape(-1)).to(self.device)).cpu().numpy()

    def load_vector(self, f, mode="pointwise"):
        """(f, v_i) over interior U dofs (``assembly.py:502-512``)."""
        return self.load_vector_t(self.sample_t(f, mode)).cpu().numpy()

    # ---------------------------------------------------------- u-side pieces
    def BT_u_t(self, u_t, out=None):
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgBTu", self.plan.handle, _vp(u_t), _vp(out), _stream())
        return out

    def B_psi_t(self, psi_t, out=None):
        out = torch.empty(self.ndof_u, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgBPsi", self.plan.handle, _vp(psi_t), _vp(out), _stream())
        return out

    def A_u_t(self, u_t, out=None):
        out = torch.empty(self.ndof_u, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgAu", self.plan.handle, _vp(u_t), _vp(out), _stream())
        return out

    # --------------------------------------------------------------- Jacobian
    def apply_cached_t(self, x_t, out=None, wcache=None):
        """D x from the weights cached by the last moments/residual call."""
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        w = self._wcache if wcache is None else wcache
        _lib.call("hpgApplyCached", self.plan.handle, _vp(w), _vp(x_t), _vp(out), _stream())
        return out

    def blocks_t(self, wcache=None, out=None, c0=0, count=None):
        count = self.plan.ncells - c0 if count is None else count
        nb2 = self.plan.block_len
        out = torch.empty((count, nb2), dtype=F64, device=self.device) if out is None else out
        w = self._wcache if wcache is None else wcache
        _lib.call("hpgBlocks", self.plan.handle, _vp(w), _vp(out), c0, count, _stream())
        return out

    def blocks_matvec_t(self, blocks_t, x_t, out=None):
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgBlocksMatvec", self.plan.handle, _vp(blocks_t), _vp(x_t), _vp(out), _stream())
        return out

    def assemble_D(self, psi):
        """Element blocks of D as a device-backed CellBlockMatrix (``assembly.py:550-557``)."""
        psi_t = self.h2d(psi, "psi")
        clamped = self._weights_t(psi_t)
        w = self._wcache.clone()
        return DeviceCellBlockMatrix(self, w, bool(clamped.item()) if clamped is not None else False)

    def assemble_D_t(self, psi_t):
        clamped = self._weights_t(psi_t)
        # snapshots: later residual / moments calls overwrite the disc's
        # weight cache and clamp flag
        return DeviceCellBlockMatrix(self, self._wcache.clone(),
                                     clamped.clone() if clamped is not None else False)

    # ------------------------------------------------ per-cell Schur preconditioner
    def _precond_ready(self):
        """Hat triples per width key on the device (``schur_hat_triple``, assembly.py:577-595)."""
        if self.kind == "obstacle" and not getattr(self, "_triples_ready", False):
            z, lam = schur_triple_factors(self.n)
            _lib.call("hpgPrecondPrepare", self.plan.handle, z.ctypes.data_as(ctypes.c_void_p),
                      lam.ctypes.data_as(ctypes.c_void_p), _stream())
            self._triples_ready = True

    def _blocks_of(self, D):
        """Fresh device copy of D's element blocks (device-backed or host CellBlockMatrix)."""
        nb = self.n * self.n * self.ncomp
        if isinstance(D, DeviceCellBlockMatrix):
            return self.blocks_t(wcache=D._w).view(-1, nb, nb)
        arr = np.ascontiguousarray(np.stack(D.blocks), dtype=np.float64)
        if arr.shape != (self.plan.ncells, nb, nb):
            raise ValueError("D.blocks has the wrong shape")
        return torch.from_numpy(arr).to(self.device)

    def precond_blocks_t(self, D, alpha, beta):
        """Device blocks (ncells, nb, nb) of ``precond_blocks(D, alpha, beta)``."""
        if beta < 0:
            raise ValueError("beta must be >= 0")
        self._precond_ready()
        nb = self.n * self.n * self.ncomp
        if isinstance(D, DeviceCellBlockMatrix):
            # fused: the blocks kernel writes P_e directly from D's point weights
            out = torch.empty((self.plan.ncells, nb, nb), dtype=F64, device=self.device)
            _lib.call("hpgPrecondAssemble", self.plan.handle, _vp(D._w), float(alpha), float(beta),
                      _vp(out), 0, self.plan.ncells, _stream())
            return out
        out = self._blocks_of(D)
        _lib.call("hpgPrecondBlocks", self.plan.handle, _vp(out), float(alpha), float(beta), 0,
                  self.plan.ncells, _stream())
        return out

    def precond_blocks(self, D, alpha, beta):
        """Dense blocks of -(D + E_beta + Bhat^T Ahat_alpha^{-1} Bhat) (obstacle,
        ``assembly.py:597-603``) or -(D + E_beta) (gradient, ``:851-860``), one
        host array per cell in ``cell_ids`` order."""
        arr = self.precond_blocks_t(D, alpha, beta).cpu().numpy()
        return [arr[i] for i in range(arr.shape[0])]

    def schur_preconditioner(self, D, alpha, beta):
        """``linalg.schur_preconditioner`` (linalg.py:262-264) with the per-cell LU on the GPU."""
        return DeviceCellBlockPreconditioner.from_operator(self, D, alpha, beta)

    def _residual_t(self, alpha, psi_prev_t, u_t, psi_t, phi_t, b_u=None, b_psi=None, wcache=None,
                    flag=None):
        for v, n, what in ((psi_prev_t, self.ndof_psi, "psi_prev"), (u_t, self.ndof_u, "u"),
                           (psi_t, self.ndof_psi, "psi")):
            self._check_len(v, n, what)
        b_u = torch.empty(self.ndof_u, dtype=F64, device=self.device) if b_u is None else b_u
        b_psi = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if b_psi is None else b_psi
        flag = self._flag if flag is None else flag
        flag.zero_()
        if wcache is True:
            wcache = self._wcache
        _lib.call("hpgResidual", self.plan.handle, float(alpha), _vp(psi_prev_t), _vp(u_t),
                  _vp(psi_t), _vp(phi_t), _vp(self.f_load_t), _vp(b_u), _vp(b_psi), _vp(flag),
                  _vp(wcache), _stream())
        return b_u, b_psi, flag

    def _residual_apply_t(self, alpha, psi_prev_t, u_t, psi_t, x_t, phi_t, b_u=None, b_psi=None,
                          y=None, flag=None):
        for v, n, what in ((psi_prev_t, self.ndof_psi, "psi_prev"), (u_t, self.ndof_u, "u"),
                           (psi_t, self.ndof_psi, "psi"), (x_t, self.ndof_psi, "x")):
            self._check_len(v, n, what)
        b_u = torch.empty(self.ndof_u, dtype=F64, device=self.device) if b_u is None else b_u
        b_psi = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if b_psi is None else b_psi
        y = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if y is None else y
        flag = self._flag if flag is None else flag
        flag.zero_()
        _lib.call("hpgResidualApply", self.plan.handle, float(alpha), _vp(psi_prev_t), _vp(u_t),
                  _vp(psi_t), _vp(phi_t), _vp(self.f_load_t), _vp(x_t), _vp(b_u), _vp(b_psi), _vp(y),
                  _vp(flag), _stream())
        return b_u, b_psi, y, flag


class ObstacleDisc2D(_DeviceDisc):
    """Device-backed ``hpgalerkin.assembly.ObstacleDisc2D`` (``assembly.py:452-603``).

    Extra keyword arguments: ``rule`` ("reference" = 2(p+1) Chebyshev-Lobatto
    projection quadrature as the reference; "gauss" = ``nq``-point Gauss).
    """

    kind = "obstacle"
    ncomp = 1

    def __init__(self, mesh2d, f, phi, f_mode="pointwise", phi_mode="pointwise",
                 rule="reference", nq=None):
        super().__init__(mesh2d, f, phi, f_mode, phi_mode, rule, nq)
        self.phi_moments_t = self.moments_from_values_t(self.sample_t(phi, phi_mode))

    @property
    def phi_moments(self):
        return self.phi_moments_t.cpu().numpy()

    @phi_moments.setter
    def phi_moments(self, value):
        # QVI overwrites the obstacle moments between solves (qvi.py:205)
        v = np.ascontiguousarray(value, dtype=np.float64).reshape(-1)
        if v.size != self.ndof_psi:
            raise ValueError("phi_moments has the wrong length")
        self.phi_moments_t = torch.from_numpy(v).to(self.device)

    # device-resident API
    def exp_moments_t(self, psi_t, out=None, wcache=None, flag=None):
        """Returns (moments, device clamp flag); also refreshes the weight cache."""
        self._check_len(psi_t, self.ndof_psi, "psi")
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        flag = self._flag if flag is None else flag
        flag.zero_()
        if wcache is True:
            wcache = self._wcache
        _lib.call("hpgObstacleMoments", self.plan.handle, _vp(psi_t), _vp(out), _vp(flag),
                  _vp(wcache), _stream())
        return out, flag

    def apply_D_t(self, psi_t, x_t, out=None):
        self._check_len(psi_t, self.ndof_psi, "psi")
        self._check_len(x_t, self.ndof_psi, "x")
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgObstacleApplyD", self.plan.handle, _vp(psi_t), _vp(x_t), _vp(out), _stream())
        return out

    def residual_t(self, alpha, psi_prev_t, u_t, psi_t, **kw):
        """``proximal.residual`` on device; ``wcache=True`` also caches D(psi)'s weights."""
        return self._residual_t(alpha, psi_prev_t, u_t, psi_t, self.phi_moments_t, **kw)

    def residual_apply_t(self, alpha, psi_prev_t, u_t, psi_t, x_t, **kw):
        """Residual and y = D(psi) x in one launch sequence (hpgResidualApply)."""
        return self._residual_apply_t(alpha, psi_prev_t, u_t, psi_t, x_t, self.phi_moments_t, **kw)

    def _weights_t(self, psi_t):
        tmp = self._dev("moments_scratch", self.ndof_psi)
        _, flag = self.exp_moments_t(psi_t, out=tmp, wcache=True)
        return flag

    # reference-facing API
    def exp_moments(self, psi):
        """((e^{-psi}, zeta_i), clamped) -- ``assembly.py:541-548``."""
        out, flag = self.exp_moments_t(self.h2d(psi, "psi"), out=self._dev("out_moments", self.ndof_psi))
        (res,), fl = self.d2h_many([out], flag=flag)
        return res, bool(fl)

    def apply_D(self, psi, x):
        """``assembly.py:559-567``."""
        psi_t, x_t = self.h2d_many([psi, x], ["psi", "x"])
        y = self.apply_D_t(psi_t, x_t, out=self._dev("out_y", self.ndof_psi))
        return self.d2h(y, "y")


class GradientDisc2D(_DeviceDisc):
    """Device-backed ``hpgalerkin.assembly.GradientDisc2D`` (``assembly.py:699-860``)."""

    kind = "gradient"
    ncomp = 2

    def __init__(self, mesh2d, f, phi, f_mode="pointwise", phi_mode="pointwise",
                 rule="reference", nq=None):
        super().__init__(mesh2d, f, phi, f_mode, phi_mode, rule, nq)
        self.phi_values_t = self.sample_t(phi, phi_mode)

    @property
    def cell_scalar_indices(self):
        return self._scalar_cell_indices()

    @property
    def phi_values(self):
        """dict cell -> (nq, nq) samples, as ``assembly.py:747-748``."""
        v = self.phi_values_t.cpu().numpy().reshape(self.plan.ncells, self.nquad, self.nquad)
        return {c: v[i] for i, c in enumerate(self.cell_ids)}

    def nl_moments_t(self, psi_t, out=None, wcache=None):
        self._check_len(psi_t, self.ndof_psi, "psi")
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        if wcache is True:
            wcache = self._wcache
        _lib.call("hpgGradientMoments", self.plan.handle, _vp(psi_t), _vp(self.phi_values_t),
                  _vp(out), _vp(wcache), _stream())
        return out

    def apply_D_t(self, psi_t, x_t, out=None):
        self._check_len(psi_t, self.ndof_psi, "psi")
        self._check_len(x_t, self.ndof_psi, "x")
        out = torch.empty(self.ndof_psi, dtype=F64, device=self.device) if out is None else out
        _lib.call("hpgGradientApplyD", self.plan.handle, _vp(psi_t), _vp(self.phi_values_t),
                  _vp(x_t), _vp(out), _stream())
        return out

    def residual_t(self, alpha, psi_prev_t, u_t, psi_t, **kw):
        return self._residual_t(alpha, psi_prev_t, u_t, psi_t, self.phi_values_t, **kw)

    def residual_apply_t(self, alpha, psi_prev_t, u_t, psi_t, x_t, **kw):
        return self._residual_apply_t(alpha, psi_prev_t, u_t, psi_t, x_t, self.phi_values_t, **kw)

    def _weights_t(self, psi_t):
        tmp = self._dev("moments_scratch", self.ndof_psi)
        self.nl_moments_t(psi_t, out=tmp, wcache=True)
        return None

    def nl_moments(self, psi):
        """(phi psi_c / sqrt(1+|psi|^2), zeta_i) stacked -- ``assembly.py:781-791``."""
        out = self.nl_moments_t(self.h2d(psi, "psi"), out=self._dev("out_moments", self.ndof_psi))
        return self.d2h(out, "moments")

    def apply_D(self, psi, x):
        """``assembly.py:817-832``."""
        psi_t, x_t = self.h2d_many([psi, x], ["psi", "x"])
        y = self.apply_D_t(psi_t, x_t, out=self._dev("out_y", self.ndof_psi))
        return self.d2h(y, "y")


class DeviceCellBlockMatrix:
    """``CellBlockMatrix`` (``assembly.py:272-298``) whose state lives on the GPU.

    It holds the point weights of D(psi).  ``@``/``matvec`` run the fused
    matrix-free kernel on those weights -- the same linear operator as the
    dense blocks (``apply_weighted == weighted_block @ c``,
    ``tests/test_assembly.py:126-132``).  The dense per-cell blocks are built
    on the device only when ``blocks`` / ``blocks_t`` / ``tocsc`` are asked for.
    """

    def __init__(self, disc, wcache, clamped):
        self.disc = disc
        self._w = wcache
        self._clamped = clamped
        self._blocks_t = None
        self._blocks_host = None
        self.n = disc.ndof_psi

    @property
    def clamped(self):
        c = self._clamped
        if isinstance(c, torch.Tensor):
            c = bool(c.item())
            self._clamped = c
        return bool(c)

    @property
    def indices(self):
        return self.disc.cell_psi_indices

    @property
    def nb(self):
        return self.disc.n * self.disc.n * self.disc.ncomp

    def blocks_t(self):
        if self._blocks_t is None:
            self._blocks_t = self.disc.blocks_t(wcache=self._w).view(-1, self.nb, self.nb)
        return self._blocks_t

    @property
    def blocks(self):
        if self._blocks_host is None:
            arr = self.blocks_t().cpu().numpy()
            self._blocks_host = [arr[i] for i in range(arr.shape[0])]
        return self._blocks_host

    def matvec_t(self, x_t, out=None):
        return self.disc.apply_cached_t(x_t, out=out, wcache=self._w)

    def matvec_blocks_t(self, x_t, out=None):
        return self.disc.blocks_matvec_t(self.blocks_t(), x_t, out=out)

    def matvec(self, x):
        return self.disc.host_matvec_cached(x, self._w)

    def tocsc(self):
        import scipy.sparse as sp
        rows, cols, vals = [], [], []
        for blk, idx in zip(self.blocks, self.indices):
            jj, kk = np.meshgrid(idx, idx, indexing="ij")
            rows.append(jj.ravel())
            cols.append(kk.ravel())
            vals.append(blk.ravel())
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.n, self.n)).tocsc()

    def __matmul__(self, x):
        return self.matvec(x)


class DeviceCellBlockPreconditioner:
    """``CellBlockPreconditioner`` (``linalg.py:246-260``) with the factors on the GPU.

    The per-cell blocks are LU-factorised with partial pivoting in place on the
    device (``hpgLUFactor`` / the fused ``hpgPrecondFactor``) and ``apply``
    runs the per-cell triangular solves on the global psi vector
    (``hpgLUSolve``).  ``factors`` gives scipy ``lu_factor``-style
    ``(lu, piv)`` host pairs on demand.
    """

    def __init__(self, disc, lu_t, piv_t, info_t=None, check=True, perm_t=None):
        self.disc = disc
        self.lu_t = lu_t
        self.piv_t = piv_t
        self.perm_t = perm_t
        self.info_t = info_t
        self.n = disc.ndof_psi
        self._factors = None
        if check and info_t is not None:
            self.check()

    def check(self):
        """scipy ``lu_factor`` semantics: ValueError on non-finite blocks, a
        warning on an exactly singular block (LAPACK info > 0)."""
        info = int(self.info_t.item())
        if info & 1:
            raise ValueError("array must not contain infs or NaNs")
        if info & 2:
            import warnings
            warnings.warn("a per-cell preconditioner block is exactly singular", RuntimeWarning)

    @classmethod
    def from_operator(cls, disc, D, alpha, beta):
        """Factor ``disc.precond_blocks(D, alpha, beta)`` without materialising them."""
        if beta < 0:
            raise ValueError("beta must be >= 0")
        disc._precond_ready()
        info = torch.zeros(1, dtype=torch.int32, device=disc.device)
        if isinstance(D, DeviceCellBlockMatrix):
            # P_e written by the blocks kernel's epilogue, then factored in place
            lu = disc.precond_blocks_t(D, alpha, beta)
            piv = torch.empty(lu.shape[:2], dtype=torch.int32, device=disc.device)
            perm = torch.empty_like(piv)
            _lib.call("hpgLUFactor", disc.plan.handle, _vp(lu), _vp(piv), _vp(perm), disc.plan.ncells,
                      _vp(info), _stream())
        else:
            lu = disc._blocks_of(D)
            piv = torch.empty(lu.shape[:2], dtype=torch.int32, device=disc.device)
            perm = torch.empty_like(piv)
            _lib.call("hpgPrecondFactor", disc.plan.handle, _vp(lu), _vp(piv), _vp(perm), float(alpha),
                      float(beta), 0, disc.plan.ncells, _vp(info), _stream())
        return cls(disc, lu, piv, info, perm_t=perm)

    @classmethod
    def from_blocks(cls, disc, blocks):
        """Factor given blocks (host list/array or device tensor), as ``CellBlockPreconditioner``."""
        nb = disc.n * disc.n * disc.ncomp
        if isinstance(blocks, torch.Tensor):
            lu = blocks.to(disc.device, torch.float64).reshape(-1, nb, nb).clone()
        else:
            arr = np.ascontiguousarray(np.stack(blocks), dtype=np.float64)
            lu = torch.from_numpy(arr).to(disc.device)
        if lu.shape != (disc.plan.ncells, nb, nb):
            raise ValueError("blocks have the wrong shape")
        piv = torch.empty(lu.shape[:2], dtype=torch.int32, device=disc.device)
        perm = torch.empty_like(piv)
        info = torch.zeros(1, dtype=torch.int32, device=disc.device)
        _lib.call("hpgLUFactor", disc.plan.handle, _vp(lu), _vp(piv), _vp(perm), disc.plan.ncells,
                  _vp(info), _stream())
        return cls(disc, lu, piv, info, perm_t=perm)

    @property
    def indices(self):
        return self.disc.cell_psi_indices

    @property
    def factors(self):
        if self._factors is None:
            lu = self.lu_t.cpu().numpy()
            piv = self.piv_t.cpu().numpy()
            self._factors = [(lu[i], piv[i]) for i in range(lu.shape[0])]
        return self._factors

    def apply_t(self, x_t, out=None):
        d = self.disc
        d._check_len(x_t, self.n, "x")
        out = torch.empty(self.n, dtype=F64, device=d.device) if out is None else out
        _lib.call("hpgLUSolve", d.plan.handle, _vp(self.lu_t), _vp(self.piv_t), _vp(self.perm_t),
                  _vp(x_t), _vp(out), _stream())
        return out

    def apply(self, x):
        d = self.disc
        y = self.apply_t(d.h2d(x, "x"), out=d._dev("out_prec", self.n))
        return d.d2h(y, "prec")

    def __call__(self, x):
        return self.apply(x)
