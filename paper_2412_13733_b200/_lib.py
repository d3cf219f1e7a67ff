"""ctypes binding of the C ABI in ``include/hpg_b200.h`` (libhpg_b200.so).

The library is built in-tree (``make`` / ``__graft_entry__.build()``).  There
is no fallback: if the shared library or a CUDA device is missing, every
entry point raises instead of computing anything on the CPU.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPG_LIB") or os.path.join(_HERE, "libhpg_b200.so")   # HPG_LIB: A/B experiments

HPG_OBSTACLE = 0
HPG_GRADIENT = 1

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int

# name -> argtypes (all return int status)
SIGNATURES = {
    "hpgPlanCreate": [ctypes.POINTER(_P), _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P],
    "hpgPlanDestroy": [_P],
    "hpgPlanInfo": [_P, ctypes.POINTER(ctypes.c_longlong)],
    "hpgObstacleMoments": [_P, _P, _P, _P, _P, _P],
    "hpgObstacleApplyD": [_P, _P, _P, _P, _P],
    "hpgGradientMoments": [_P, _P, _P, _P, _P, _P],
    "hpgGradientApplyD": [_P, _P, _P, _P, _P, _P],
    "hpgApplyCached": [_P, _P, _P, _P, _P],
    "hpgApplyCachedRange": [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P],
    "hpgApplyCachedHostSlab": [_P, _P, _P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P],
    "hpgResidual": [_P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "hpgResidualApply": [_P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "hpgBlocks": [_P, _P, _P, _I, _I, _P],
    "hpgBlocksMatvec": [_P, _P, _P, _P, _P],
    "hpgBTu": [_P, _P, _P, _P],
    "hpgBPsi": [_P, _P, _P, _P],
    "hpgAu": [_P, _P, _P, _P],
    "hpgMomentsFromValues": [_P, _P, _P, _P],
    "hpgLoadVector": [_P, _P, _P, _P],
    "hpgPrecondPrepare": [_P, _P, _P, _P],
    "hpgPrecondBlocks": [_P, _P, _D, _D, _I, _I, _P],
    "hpgPrecondAssemble": [_P, _P, _D, _D, _P, _I, _I, _P],
    "hpgLUFactor": [_P, _P, _P, _P, _I, _P, _P],
    "hpgPrecondFactor": [_P, _P, _P, _P, _D, _D, _I, _I, _P, _P],
    "hpgLUSolve": [_P, _P, _P, _P, _P, _P, _P],
    "hpgLUMaxBlock": [],
    "hpgLUProfile": [_P],
    "hpgStiffnessFactor": [_P, _P, _P, _P, _P, _P],
    "hpgStiffnessSolve": [_P, _P, _P, _P],
    "hpgSchurApply": [_P, _P, _D, _D, _P, _P, _P],
    "hpgUFullSetup": [_P, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "hpgUFullValues": [_P, _P, _P, _P],
    "hpgUFullOperator": [_P, _D, _P, _P, _P, _P, _P],
    "hpgUFullSolve": [_P, _P, _P, _P],
    "hpgGmresCreate": [ctypes.POINTER(_P), ctypes.c_longlong, _I],
    "hpgGmresDestroy": [_P],
    "hpgGmresBind": [_P, _P, _P, _P],
    "hpgGmresCaptureBegin": [_P, _P],
    "hpgGmresCaptureEnd": [_P, _P],
    "hpgGmresSolve": [_P, _D, _D, _P, _P],
    "hpgGmresStatus": [_P, ctypes.POINTER(_I), ctypes.POINTER(_I), _P, _P],
    "hpgAxpby": [ctypes.c_longlong, _D, _P, _D, _P, _P, _P],
    "hpgVersion": [],
}


class HpgError(RuntimeError):
    pass


_lib = None


def load():
    """Load libhpg_b200.so once; raise if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HpgError(f"{LIB_PATH} not built; run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _I
    lib.hpgLastError.argtypes = []
    lib.hpgLastError.restype = ctypes.c_char_p
    _lib = lib
    return lib


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.hpgLastError().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise HpgError(f"{name} failed (code {rc}): {msg}")
    return rc


def exported_symbols():
    return sorted(list(SIGNATURES) + ["hpgLastError"])
