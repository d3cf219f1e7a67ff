"""CPU-side checks of the C ABI: the library loads and exports what the header declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hpg_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hpg\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for n in ("hpgPlanCreate", "hpgObstacleMoments", "hpgObstacleApplyD", "hpgGradientMoments",
              "hpgGradientApplyD", "hpgApplyCached", "hpgResidual", "hpgBlocks",
              "hpgBlocksMatvec", "hpgBTu", "hpgBPsi", "hpgAu", "hpgMomentsFromValues",
              "hpgLoadVector", "hpgLastError"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2412_13733_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhpg_b200.so not built (run make)")
    lib = _lib.load()          # loads without a GPU: cudart is linked statically
    for n in declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (hpg\w+)", out))
    assert set(declared()) <= exported
    assert set(_lib.exported_symbols()) == set(declared())
    assert lib.hpgVersion() == 1


def test_library_is_sm100a():
    from paper_2412_13733_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhpg_b200.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass        # FP64 tensor-core path (mma.sync.m8n8k4.f64)


def test_no_gpu_call_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2412_13733_b200 import _lib, disc
    from paper_2412_13733_b200.mesh import uniform_mesh_2d
    with pytest.raises(_lib.HpgError):
        disc.ObstacleDisc2D(uniform_mesh_2d(0.0, 1.0, 2, 3), 1.0, 1.0)
