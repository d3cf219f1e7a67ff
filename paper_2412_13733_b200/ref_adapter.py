"""Drop-in subclasses of the reference's discretisations.

The reference's seam is duck typing on the ``disc`` object plus the
``CellBlockMatrix`` type.  These classes subclass the reference's own
``hpgalerkin.assembly.ObstacleDisc2D`` / ``GradientDisc2D`` /
``CellBlockMatrix`` and override only the hot-path members; every other
member -- ``A``, ``B``, ``E_matrix``, ``mass_psi``, ``cell_psi_indices``,
``schur_hat_triple`` ... -- is the reference's, so the UNMODIFIED
``hpgalerkin.proximal.solve`` / ``newton_solve``, ``linalg.schur_solve`` and
``linalg.monolithic_solve`` run on them:

==========================  ==============================================
reference member            here
==========================  ==============================================
``exp_moments``             ``assembly.py:541-548`` -> hpgObstacleMoments
``nl_moments``              ``assembly.py:781-791`` -> hpgGradientMoments
``apply_D``                 ``assembly.py:559-567 / 817-832`` -> hpg*ApplyD
``assemble_D``              ``assembly.py:550-557 / 804-815`` -> point
                            weights on the device, wrapped as a
                            ``B200CellBlockMatrix`` (``isinstance(D,
                            CellBlockMatrix)`` holds, ``linalg.py:296``)
``precond_blocks``          ``assembly.py:597-603 / 851-860`` -> blocks
                            formed on the device (no ``.blocks`` D2H)
``data_moments``,           ``assembly.py:502-533`` -> device analysis of
``moments_from_values``,    the rule's point samples
``load_vector``
==========================  ==============================================

``rule="reference"`` (default) keeps the reference's 2(p+1)-point projection
quadrature with bit-identical tables; ``rule="gauss", nq=Q`` switches the
quadrature to BASELINE.json's Gauss rule for the whole disc (the reference's
own ``CellKernel1D`` objects get the same tables, so inherited members that
read them -- ``quad_grids``, ``_psi_cell_values`` -- stay consistent).

``hpgalerkin`` is imported here because it is the CLIENT of the drop-in:
whoever uses these classes has the reference installed.  Nothing computes on
the CPU on the overridden paths; a missing GPU or library raises.
"""

import numpy as np

from hpgalerkin import assembly as _ra

from . import disc as _dd

__all__ = ["B200CellBlockMatrix", "B200ObstacleDisc2D", "B200GradientDisc2D"]


class B200CellBlockMatrix(_ra.CellBlockMatrix):
    """``CellBlockMatrix`` (``assembly.py:272-298``) backed by device state.

    ``@`` / ``matvec`` run the matrix-free kernel on the point weights of
    D(psi) kept on the GPU (the same operator as the dense blocks); ``blocks``
    is built on the device and copied to the host only when read (the
    reference's ``precond_blocks`` and ``tocsc`` read it).  ``tocsc`` and
    ``__matmul__`` are the reference's own.
    """

    def __init__(self, device_matrix, indices, n, clamped):
        # no super().__init__: ``blocks`` is a lazy property here
        self.device_matrix = device_matrix
        self.indices = indices
        self.n = n
        self.clamped = bool(clamped)

    @property
    def blocks(self):
        return self.device_matrix.blocks

    def matvec(self, x):
        return self.device_matrix.matvec(np.asarray(x, dtype=float))


def _substitute_tables(disc, tables):
    """Give the reference's per-cell ``CellKernel1D`` objects the rule's tables
    (the Gauss-table substitution of SURVEY.md §8c / Appendix B.2)."""
    for k2 in disc.kernels.values():
        for k1 in (k2.kx, k2.ky):
            k1.nquad = tables.nq
            k1.points = k1.midpoint + 0.5 * k1.h * tables.xi
            k1.S, k1.T, k1.Su, k1.Tu = tables.S, tables.T, tables.Su, tables.Tu


class _B200Mixin:
    """Members shared by both drop-in discs; ``self.device_disc`` is the
    device-resident ``paper_2412_13733_b200.disc`` object of the same mesh."""

    def _make_device(self, cls, mesh2d, f, phi, f_mode, phi_mode, rule, nq):
        # built before the reference constructor, which calls the
        # (overridden) data terms below
        # (nq only selects the Gauss rule's point count; the reference rule fixes 2(p+1))
        self.device_disc = cls(mesh2d, f, phi, f_mode, phi_mode, rule=rule,
                               nq=nq if rule == "gauss" else None)
        self.rule = rule

    def _finish(self):
        if self.rule != "reference":
            _substitute_tables(self, self.device_disc.tables)
        dd = self.device_disc
        if dd.ndof_psi != self.ndof_psi or dd.ndof_u != self.ndof_u:
            raise RuntimeError("device and reference dof layouts disagree")

    # data terms (assembly.py:502-533, 761-771) on the device
    def load_vector(self, f, mode="pointwise"):
        return self.device_disc.load_vector(f, mode)

    def quad_grids(self):
        return self.device_disc.quad_grids()

    def apply_D(self, psi, x):
        return self.device_disc.apply_D(psi, x)

    def _wrap(self, Ddev):
        return B200CellBlockMatrix(Ddev, self.cell_psi_indices, self.ndof_psi, Ddev.clamped)

    def precond_blocks(self, D, alpha, beta):
        Dd = D.device_matrix if isinstance(D, B200CellBlockMatrix) else D
        return self.device_disc.precond_blocks(Dd, alpha, beta)


class B200ObstacleDisc2D(_B200Mixin, _ra.ObstacleDisc2D):
    """``hpgalerkin.assembly.ObstacleDisc2D`` with the quadrature on the B200."""

    def __init__(self, mesh2d, f, phi, f_mode="pointwise", phi_mode="pointwise",
                 rule="reference", nq=None):
        self._make_device(_dd.ObstacleDisc2D, mesh2d, f, phi, f_mode, phi_mode, rule, nq)
        super().__init__(mesh2d, f, phi, f_mode, phi_mode)
        self._finish()

    # ``phi_moments`` stays a plain host array owned by the reference code
    # (proximal.residual reads it, qvi.py:205 overwrites it); the device copy
    # follows every assignment
    @property
    def phi_moments(self):
        return self._phi_moments

    @phi_moments.setter
    def phi_moments(self, value):
        v = np.ascontiguousarray(value, dtype=np.float64)
        self._phi_moments = v
        self.device_disc.phi_moments = v

    def data_moments(self, g, mode="pointwise"):
        return self.device_disc.data_moments(g, mode)

    def moments_from_values(self, values):
        return self.device_disc.moments_from_values(values)

    def exp_moments(self, psi):
        return self.device_disc.exp_moments(psi)

    def assemble_D(self, psi):
        return self._wrap(self.device_disc.assemble_D(psi))


class B200GradientDisc2D(_B200Mixin, _ra.GradientDisc2D):
    """``hpgalerkin.assembly.GradientDisc2D`` with the quadrature on the B200."""

    def __init__(self, mesh2d, f, phi, f_mode="pointwise", phi_mode="pointwise",
                 rule="reference", nq=None):
        self._make_device(_dd.GradientDisc2D, mesh2d, f, phi, f_mode, phi_mode, rule, nq)
        super().__init__(mesh2d, f, phi, f_mode, phi_mode)
        self._finish()
        # point samples of phi on the rule's grid (assembly.py:747-748)
        self.phi_values = self.device_disc.phi_values

    def nl_moments(self, psi):
        return self.device_disc.nl_moments(psi)

    def assemble_D(self, psi):
        return self._wrap(self.device_disc.assemble_D(psi))
