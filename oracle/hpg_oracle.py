"""CPU oracle for the hpG element-quadrature hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / CPU baseline.  The
product path (``paper_2412_13733_b200``) never calls it.

It is a NumPy restatement of the reference's per-cell algorithm, batched
over cells (the reference loops over cells in Python).  Every function cites
the reference lines it follows (paths relative to
``/root/reference/pkg/src/hpgalerkin/``).  Tables (S, T, Su, Tu) are inputs:
the oracle and the device consume bit-identical arrays.

Parity is PINNED: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the unmodified reference package
(``oracle/make_golden.py``, fixtures in ``tests/golden/``).

Conventions (uniform degree p, tensor mesh ncx x ncy, cell order (cx, cy)
cx-major as ``assembly.py:482``):
* psi tile side n (p-1 obstacle, p gradient), U tile side m = p+1;
* global psi vector = x-major tensor order (``spaces.py:212-214``), i.e. a
  (ncx*n, ncy*n) array; gradient stacks [psi_x; psi_y] (``assembly.py:744``);
* u = interior U coefficients, a (nix, niy) array over the 1D interior dofs
  (hats 1..nc-1 then bubbles cell by cell, ``spaces.py:25-43,188-189``).
"""

import numpy as np

EXP_CLAMP = 700.0   # assembly.py:25


# ---------------------------------------------------------------------------
# layouts

def psi_tiles(vec, ncx, ncy, n):
    """Global x-major psi -> (ncx, ncy, n, n) tiles (``spaces.py:212-219``)."""
    return vec.reshape(ncx, n, ncy, n).transpose(0, 2, 1, 3)


def psi_global(tiles):
    ncx, ncy, n, _ = tiles.shape
    return np.ascontiguousarray(tiles.transpose(0, 2, 1, 3)).reshape(-1)


def cell_psi_indices(ncx, ncy, n):
    """List of index arrays in cell order (``assembly.py:489-490``)."""
    ndof_y = ncy * n
    out = []
    for cx in range(ncx):
        for cy in range(ncy):
            ix = (cx * n + np.arange(n)) * ndof_y
            out.append(np.add.outer(ix, cy * n + np.arange(n)).ravel())
    return out


def u_local_map_1d(nc, p):
    """(nc, p+1) interior index of each cell-local U dof, -1 for boundary hats.

    Local order [hat_L, hat_R, W_0..W_{p-2}] (``spaces.py:40-43``); interior
    numbering drops vertex hats 0 and nc (``spaces.py:36-38``).
    """
    m = p + 1
    out = np.empty((nc, m), dtype=np.int64)
    for c in range(nc):
        out[c, 0] = c - 1 if c >= 1 else -1
        out[c, 1] = c if c + 1 <= nc - 1 else -1
        out[c, 2:] = (nc - 1) + c * (p - 1) + np.arange(p - 1)
    return out


def u_tiles(u, ncx, ncy, p):
    """Interior u -> (ncx, ncy, m, m) cell-local dof tiles (zeros on the boundary)."""
    mx = u_local_map_1d(ncx, p)
    my = u_local_map_1d(ncy, p)
    nix = ncx * (p - 1) + ncx - 1
    niy = ncy * (p - 1) + ncy - 1
    U = np.zeros((nix + 1, niy + 1))
    U[:nix, :niy] = u.reshape(nix, niy)      # row/col -1 -> the zero pad
    return U[mx[:, None, :, None], my[None, :, None, :]]


def u_assemble(local, ncx, ncy, p):
    """Scatter-add (ncx, ncy, m, m) local U contributions into interior u."""
    mx = u_local_map_1d(ncx, p)
    my = u_local_map_1d(ncy, p)
    nix = ncx * (p - 1) + ncx - 1
    niy = ncy * (p - 1) + ncy - 1
    out = np.zeros((nix + 1, niy + 1))
    np.add.at(out, (mx[:, None, :, None], my[None, :, None, :]), local)
    return out[:nix, :niy].reshape(-1)


def legendre_map(p):
    """Per-cell U->Legendre map R ((p+1) x (p+1)), ``spaces.py:45-57``."""
    R = np.zeros((p + 1, p + 1))
    R[0, 0] = 0.5
    R[1, 0] = -0.5
    R[0, 1] = 0.5
    R[1, 1] = 0.5
    for k in range(p - 1):
        R[k, 2 + k] = 1.0 / (2 * k + 3)
        R[k + 2, 2 + k] = -1.0 / (2 * k + 3)
    return R


def deriv_map(p):
    """Reference-derivative coefficients D (p x (p+1)), ``spaces.py:59-68``."""
    D = np.zeros((max(p, 1), p + 1))
    D[0, 0] = -0.5
    D[0, 1] = 0.5
    for k in range(p - 1):
        D[k + 1, 2 + k] = -1.0
    return D


def mass_weights(h, n):
    """w_i = h / (2i+1) per cell (``assembly.py:203``): (ncells, n)."""
    return np.asarray(h, dtype=float)[:, None] / (2.0 * np.arange(n) + 1.0)[None, :]


# ---------------------------------------------------------------------------
# the three stages (assembly.py:187-269)

def synthesize(S, C):
    """V = S C S^T per cell (``assembly.py:243-244``)."""
    return np.einsum("ga,xyab,hb->xygh", S, C, S, optimize=True)


def clamped_exp_neg(V):
    """exp(min(-V, 700)) and the overflow flag (``assembly.py:187-192``).

    The flag is set iff some -V > 700 or V is NaN (NaN != NaN)."""
    t = np.clip(-V, None, EXP_CLAMP)
    return np.exp(t), bool(np.any(t != -V))


def analyse(T, wx, wy, G):
    """M = (wx (x) wy) * (T G T^T) per cell (``assembly.py:249-251``)."""
    M = np.einsum("ag,xygh,bh->xyab", T, G, T, optimize=True)
    return wx[:, None, :, None] * M * wy[None, :, None, :]


def weighted_blocks(S, T, wx, wy, W):
    """Per-cell (n^2, n^2) blocks (``assembly.py:257-263``), cell order."""
    blk = np.einsum("ag,bh,xygh,gj,hk->xyabjk", T, T, W, S, S, optimize=True)
    blk *= (wx[:, None, :, None] * wy[None, :, None, :])[..., None, None]
    ncx, ncy, n = W.shape[0], W.shape[1], S.shape[1]
    return blk.reshape(ncx * ncy, n * n, n * n)


# ---------------------------------------------------------------------------
# obstacle (assembly.py:452-567)

class Problem:
    """Uniform-degree tensor mesh + tables; the oracle's view of a Disc."""

    def __init__(self, kind, xpts, ypts, p, tables):
        self.kind = kind
        self.xpts = np.asarray(xpts, dtype=float)
        self.ypts = np.asarray(ypts, dtype=float)
        self.ncx = self.xpts.size - 1
        self.ncy = self.ypts.size - 1
        self.hx = np.diff(self.xpts)
        self.hy = np.diff(self.ypts)
        self.p = int(p)
        self.m = self.p + 1
        self.n = self.p - 1 if kind == "obstacle" else self.p
        self.t = tables
        self.wx = mass_weights(self.hx, self.n)
        self.wy = mass_weights(self.hy, self.n)
        self.wux = mass_weights(self.hx, self.m)
        self.wuy = mass_weights(self.hy, self.m)
        self.ncomp_dofs = self.ncx * self.n * self.ncy * self.n
        self.ndof_psi = self.ncomp_dofs * (1 if kind == "obstacle" else 2)
        self.nix = self.ncx * self.p - 1
        self.niy = self.ncy * self.p - 1
        self.ndof_u = self.nix * self.niy

    # -- data (assembly.py:301-317, 502-533, 747-748)
    def grids(self):
        gx = 0.5 * (self.xpts[:-1] + self.xpts[1:])[:, None] + \
            0.5 * self.hx[:, None] * self.t.xi[None, :]
        gy = 0.5 * (self.ypts[:-1] + self.ypts[1:])[:, None] + \
            0.5 * self.hy[:, None] * self.t.xi[None, :]
        return gx, gy

    def sample(self, g):
        """Pointwise samples (ncx, ncy, nq, nq) of scalar data g(x, y)."""
        nq = self.t.nq
        if np.isscalar(g):
            return np.full((self.ncx, self.ncy, nq, nq), float(g))
        gx, gy = self.grids()
        X = np.broadcast_to(gx[:, None, :, None], (self.ncx, self.ncy, nq, nq))
        Y = np.broadcast_to(gy[None, :, None, :], (self.ncx, self.ncy, nq, nq))
        return np.asarray(g(X, Y), dtype=float)

    def data_moments(self, vals):
        """(g, zeta_i) from point samples (``assembly.py:514-533``)."""
        return psi_global(analyse(self.t.T, self.wx, self.wy, vals))

    def load_vector(self, vals):
        """(f, v_i) on interior U dofs (``assembly.py:502-512``)."""
        Mu = analyse(self.t.Tu, self.wux, self.wuy, vals)
        R = legendre_map(self.p)
        loc = np.einsum("ia,xyij,jb->xyab", R, Mu, R)
        return u_assemble(loc, self.ncx, self.ncy, self.p)

    # -- psi side
    def _tiles(self, vec, comp=0):
        off = comp * self.ncomp_dofs
        return psi_tiles(vec[off:off + self.ncomp_dofs], self.ncx, self.ncy, self.n)

    def exp_moments(self, psi):
        """(e^{-psi}, zeta) and the clamp flag (``assembly.py:541-548``)."""
        E, flag = clamped_exp_neg(synthesize(self.t.S, self._tiles(psi)))
        return psi_global(analyse(self.t.T, self.wx, self.wy, E)), flag

    def obstacle_weights(self, psi):
        return clamped_exp_neg(synthesize(self.t.S, self._tiles(psi)))

    def obstacle_apply_D(self, psi, x):
        """``assembly.py:559-567`` / ``:265-269``."""
        W, _ = self.obstacle_weights(psi)
        V = synthesize(self.t.S, self._tiles(x)) * W
        return psi_global(analyse(self.t.T, self.wx, self.wy, V))

    def obstacle_blocks(self, psi):
        """``assembly.py:550-557``: blocks (N, n^2, n^2) and the flag."""
        W, flag = self.obstacle_weights(psi)
        return weighted_blocks(self.t.S, self.t.T, self.wx, self.wy, W), flag

    # -- gradient (assembly.py:781-832)
    def grad_fields(self, psi):
        vx = synthesize(self.t.S, self._tiles(psi, 0))
        vy = synthesize(self.t.S, self._tiles(psi, 1))
        return vx, vy

    def nl_moments(self, psi, phi_vals):
        vx, vy = self.grad_fields(psi)
        root = np.sqrt(1.0 + vx * vx + vy * vy)
        mx = analyse(self.t.T, self.wx, self.wy, phi_vals * vx / root)
        my = analyse(self.t.T, self.wx, self.wy, phi_vals * vy / root)
        return np.concatenate([psi_global(mx), psi_global(my)])

    def kernel_fields(self, psi, phi_vals):
        """kxx, kxy, kyy (``assembly.py:793-802``)."""
        vx, vy = self.grad_fields(psi)
        r2 = 1.0 + vx * vx + vy * vy
        inv = r2 ** -0.5
        inv3 = r2 ** -1.5
        return (phi_vals * (inv - vx * vx * inv3), phi_vals * (-vx * vy * inv3),
                phi_vals * (inv - vy * vy * inv3))

    def gradient_apply_D(self, psi, x, phi_vals):
        kxx, kxy, kyy = self.kernel_fields(psi, phi_vals)
        vx = synthesize(self.t.S, self._tiles(x, 0))
        vy = synthesize(self.t.S, self._tiles(x, 1))
        mx = analyse(self.t.T, self.wx, self.wy, kxx * vx + kxy * vy)
        my = analyse(self.t.T, self.wx, self.wy, kxy * vx + kyy * vy)
        return np.concatenate([psi_global(mx), psi_global(my)])

    def gradient_blocks(self, psi, phi_vals):
        """[[Wxx, Wxy], [Wxy, Wyy]] per cell (``assembly.py:804-815``)."""
        kxx, kxy, kyy = self.kernel_fields(psi, phi_vals)
        args = (self.t.S, self.t.T, self.wx, self.wy)
        Wxx = weighted_blocks(*args, kxx)
        Wxy = weighted_blocks(*args, kxy)
        Wyy = weighted_blocks(*args, kyy)
        top = np.concatenate([Wxx, Wxy], axis=2)
        bot = np.concatenate([Wxy, Wyy], axis=2)
        return np.concatenate([top, bot], axis=1)

    # -- exact u-side couplings (assembly.py:81-116,470-477,725-729)
    def BT_u(self, u):
        """B^T u per cell via the Legendre maps."""
        C = u_tiles(u, self.ncx, self.ncy, self.p)
        R = legendre_map(self.p)
        n = self.n
        if self.kind == "obstacle":
            L = np.einsum("ia,xyab,jb->xyij", R, C, R)[:, :, :n, :n]
            return psi_global(self.wx[:, None, :, None] * L * self.wy[None, :, None, :])
        D = deriv_map(self.p)
        w2 = 2.0 / (2.0 * np.arange(n) + 1.0)
        Lx = np.einsum("ia,xyab,jb->xyij", D, C, R)[:, :, :n, :n]
        Ly = np.einsum("ia,xyab,jb->xyij", R, C, D)[:, :, :n, :n]
        bx = w2[None, None, :, None] * Lx * self.wy[None, :, None, :]
        by = self.wx[:, None, :, None] * Ly * w2[None, None, None, :]
        return np.concatenate([psi_global(bx), psi_global(by)])

    def B_psi(self, psi):
        """B psi, assembled into interior U dofs."""
        R = legendre_map(self.p)
        n, m = self.n, self.m
        if self.kind == "obstacle":
            G = np.zeros((self.ncx, self.ncy, m, m))
            G[:, :, :n, :n] = (self.wx[:, None, :, None] * self._tiles(psi)
                               * self.wy[None, :, None, :])
            loc = np.einsum("ia,xyij,jb->xyab", R, G, R)
        else:
            D = np.zeros((m, m))
            D[:self.p] = deriv_map(self.p)
            w2 = 2.0 / (2.0 * np.arange(n) + 1.0)
            Gx = np.zeros((self.ncx, self.ncy, m, m))
            Gy = np.zeros((self.ncx, self.ncy, m, m))
            Gx[:, :, :n, :n] = (w2[None, None, :, None] * self._tiles(psi, 0)
                                * self.wy[None, :, None, :])
            Gy[:, :, :n, :n] = (self.wx[:, None, :, None] * self._tiles(psi, 1)
                                * w2[None, None, None, :])
            loc = (np.einsum("ia,xyij,jb->xyab", D, Gx, R)
                   + np.einsum("ia,xyij,jb->xyab", R, Gy, D))
        return u_assemble(loc, self.ncx, self.ncy, self.p)

    def A_u(self, u):
        """A u with A = kron(Ax, My) + kron(Mx, Ay) (``assembly.py:42-78,470-474``)."""
        C = u_tiles(u, self.ncx, self.ncy, self.p)
        R = legendre_map(self.p)

        def stiff(h):
            K = np.zeros((h.size, self.m, self.m))
            K[:, 0, 0] = K[:, 1, 1] = 1.0 / h
            K[:, 0, 1] = K[:, 1, 0] = -1.0 / h
            for k in range(self.p - 1):
                K[:, 2 + k, 2 + k] = 4.0 / (h * (2 * k + 3))
            return K

        def mass(wu):
            return np.einsum("ia,ci,ib->cab", R, wu, R)

        Kx, Ky = stiff(self.hx), stiff(self.hy)
        Mx, My = mass(self.wux), mass(self.wuy)
        loc = (np.einsum("xab,xybc,ydc->xyad", Kx, C, My)
               + np.einsum("xab,xybc,ydc->xyad", Mx, C, Ky))
        return u_assemble(loc, self.ncx, self.ncy, self.p)

    def residual(self, alpha, psi_prev, u, psi, f_load, phi_moments=None,
                 phi_vals=None):
        """(b_u, b_psi, clamped) of ``proximal.py:112-126``."""
        b_u = alpha * f_load + self.B_psi(psi_prev) - alpha * self.A_u(u) - self.B_psi(psi)
        if self.kind == "obstacle":
            em, clamped = self.exp_moments(psi)
            b_psi = phi_moments - self.BT_u(u) - em
        else:
            clamped = False
            b_psi = self.nl_moments(psi, phi_vals) - self.BT_u(u)
        return b_u, b_psi, clamped


def blocks_matvec(blocks, indices, n, x):
    """CellBlockMatrix.matvec (``assembly.py:281-285``)."""
    out = np.zeros(n)
    for blk, idx in zip(blocks, indices):
        out[idx] = blk @ x[idx]
    return out


# ---------------------------------------------------------------------------
# per-cell Schur preconditioner

def spectral_1d(n, h):
    """Per-cell spectral Gram, stiffness diagonal and mass (``assembly.py:128-170``)."""
    g = np.zeros((n, n))
    m = np.zeros((n, n))
    k = 4.0 * (2.0 * np.arange(n) + 3.0) / h
    for a in range(n):
        g[a, a] = h / (2 * a + 1)
        m[a, a] = h * (1.0 / (2 * a + 1) + 1.0 / (2 * a + 5))
        if a + 2 < n:
            g[a, a + 2] = -h / (2 * a + 5)
            v = -h / (2 * a + 5)
            m[a, a + 2] = v
            m[a + 2, a] = v
    return g, k, m


def schur_hat_triple(n, hx, hy):
    """``ObstacleDisc2D.schur_hat_triple`` (``assembly.py:577-595``), dense as the reference."""
    gx, kx, mx = spectral_1d(n, hx)
    gy, ky, my = spectral_1d(n, hy)
    Ahat = np.kron(np.diag(kx), my) + np.kron(mx, np.diag(ky))
    Bhat = np.kron(gx, gy)
    return Bhat.T @ np.linalg.solve(Ahat, Bhat)


def precond_blocks(prob, blocks, alpha, beta):
    """``precond_blocks`` (obstacle ``assembly.py:597-603``, gradient ``:851-860``)."""
    n = prob.n
    out = []
    cache = {}
    for i, (cx, cy) in enumerate((cx, cy) for cx in range(prob.ncx) for cy in range(prob.ncy)):
        hx, hy = prob.hx[cx], prob.hy[cy]
        if prob.kind == "obstacle":
            key = (round(hx, 15), round(hy, 15))
            if key not in cache:
                cache[key] = schur_hat_triple(n, hx, hy)
            blk = -blocks[i] - cache[key] / alpha
            mass = np.kron(hx / (2.0 * np.arange(n) + 1.0), hy / (2.0 * np.arange(n) + 1.0))
            blk[np.diag_indices_from(blk)] -= beta * mass
        else:
            blk = -blocks[i].copy()
            if beta:
                _, kx, mx = spectral_1d(n, hx)
                _, ky, my = spectral_1d(n, hy)
                E = np.kron(np.diag(kx), my) + np.kron(mx, np.diag(ky))
                m2 = n * n
                blk[:m2, :m2] -= beta * E
                blk[m2:, m2:] -= beta * E
        out.append(blk)
    return out


def lu_precond_apply(blocks, indices, n, x):
    """``CellBlockPreconditioner.apply`` (``linalg.py:246-257``): LAPACK getrf/getrs per cell."""
    import scipy.linalg as sla
    out = np.zeros(n)
    for blk, idx in zip(blocks, indices):
        out[idx] = sla.lu_solve(sla.lu_factor(blk), x[idx])
    return out


def rel_err(a, b):
    """Global max-norm relative error (SURVEY.md §8c parity metric)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = np.max(np.abs(b)) if b.size else 0.0
    num = np.max(np.abs(a - b)) if a.size else 0.0
    return num / den if den > 0 else num
