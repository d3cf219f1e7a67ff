"""Tensor-product meshes (the subset of ``hpgalerkin/mesh.py`` the hot path reads).

The discretisation classes only read ``mesh_x.points``, ``mesh_x.degrees``
(and the same for y), so reference ``TensorMesh2D`` objects are accepted
too (duck typing).
"""

import numpy as np


class Mesh1D:
    """Breakpoints plus one polynomial degree per cell (``mesh.py:8-40``)."""

    def __init__(self, points, degrees):
        points = np.ascontiguousarray(points, dtype=float)
        degrees = np.ascontiguousarray(degrees, dtype=int)
        if points.ndim != 1 or points.size < 2:
            raise ValueError("need at least two breakpoints")
        if not np.all(np.isfinite(points)):
            raise ValueError("breakpoints must be finite")
        if np.any(np.diff(points) <= 0):
            raise ValueError("breakpoints must be strictly increasing")
        if degrees.shape != (points.size - 1,):
            raise ValueError("need exactly one degree per cell")
        if np.any(degrees < 1):
            raise ValueError("cell degrees must be >= 1")
        self.points = points
        self.degrees = degrees
        self.points.flags.writeable = False
        self.degrees.flags.writeable = False

    @property
    def ncells(self):
        return self.points.size - 1

    @property
    def widths(self):
        return np.diff(self.points)


class TensorMesh2D:
    def __init__(self, mesh_x, mesh_y):
        self.mesh_x = mesh_x
        self.mesh_y = mesh_y

    @property
    def ncells(self):
        return self.mesh_x.ncells * self.mesh_y.ncells

    @property
    def shape(self):
        return (self.mesh_x.ncells, self.mesh_y.ncells)

    @property
    def degrees_x(self):
        return self.mesh_x.degrees

    @property
    def degrees_y(self):
        return self.mesh_y.degrees


def uniform_mesh_1d(a, b, ncells, degree):
    if ncells < 1:
        raise ValueError("ncells must be >= 1")
    return Mesh1D(np.linspace(a, b, ncells + 1), np.full(ncells, int(degree), dtype=int))


def uniform_mesh_2d(a, b, ncells, degree):
    return TensorMesh2D(uniform_mesh_1d(a, b, ncells, degree),
                        uniform_mesh_1d(a, b, ncells, degree))
