"""B200-native (sm_100a) element-quadrature engine for the hierarchical proximal
Galerkin (hpG) LVPP saddle system of arXiv 2412.13733.

The hot path -- per-Newton-step synthesis, pointwise LVPP map and test-side
analysis of ``hpgalerkin/assembly.py`` -- runs in hand-written FP64 CUDA
kernels (DMMA tensor cores) behind the C ABI of ``include/hpg_b200.h``; the
Python classes here keep the reference's solver-facing API so the reference
Newton loop can call them as a drop-in.
"""

__version__ = "0.1.0"

from .tables import Tables  # noqa: F401
from .mesh import Mesh1D, TensorMesh2D, uniform_mesh_1d, uniform_mesh_2d  # noqa: F401


def __getattr__(name):
    # torch-dependent modules load lazily so the CPU-only pieces import fast
    if name in ("ObstacleDisc2D", "GradientDisc2D", "DeviceCellBlockMatrix", "pinned_array"):
        from . import disc
        return getattr(disc, name)
    if name == "residual":
        from .proximal import residual
        return residual
    raise AttributeError(name)
