"""ctypes binding of the sm_100a C-ABI library (include/tomobpdn_b200.h).

There is no fallback: if the library is missing or no CUDA device is present, every compute
entry point raises.  Loading the library itself needs no GPU (the CPU test-suite checks that
every symbol of the header is exported).
"""

from __future__ import annotations

import ctypes
import os

from .exceptions import CapacityError, ConfigurationError, NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIB_PATH") or os.path.join(HERE, "lib", "libtomobpdn_b200.so")

TB_OK, TB_ERR_INVALID, TB_ERR_CUDA, TB_ERR_CAPACITY = 0, 1, 2, 3
SOLVER_CODES = {"rbpg": 0, "fista": 1, "ista": 2}

c_void_p, c_int32, c_int64, c_double, c_uint64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64


class SolverConfigC(ctypes.Structure):
    """tb_solver_config (include/tomobpdn_b200.h)."""

    _fields_ = [
        ("num_blocks", c_int32),
        ("max_iters", c_int32),
        ("fixed_iters", c_int32),
        ("backtrack_cap", c_int32),
        ("tol", c_double),
        ("c_alpha", c_double),
        ("alpha_init_scale", c_double),
    ]


# name -> (restype, argtypes); the header is the source of truth (tests check both agree)
SIGNATURES = {
    "tb_version": (ctypes.c_char_p, []),
    "tb_last_error": (ctypes.c_char_p, []),
    "tb_launch_count": (c_int64, []),
    "tb_last_solver_kernel": (ctypes.c_char_p, []),
    "tb_ctx_create": (c_int32, [c_int32, c_void_p, c_int64, c_int64, ctypes.POINTER(c_void_p)]),
    "tb_ctx_destroy": (c_int32, [c_void_p]),
    "tb_spectral_sq_norms": (c_int32, [c_void_p, c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), c_void_p, c_int32, c_double, ctypes.POINTER(c_double), c_void_p]),
    "tb_set_partition": (c_int32, [c_void_p, c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64), ctypes.POINTER(c_double)]),
    "tb_set_lipschitz": (c_int32, [c_void_p, c_double]),
    "tb_default_lambda": (c_int32, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_void_p]),
    "tb_derive_seeds": (c_int32, [c_uint64, c_int64, c_int64, c_void_p, c_void_p]),
    "tb_synthesize_pairs": (c_int32, [c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "tb_solve": (c_int32, [c_void_p, c_int32, ctypes.POINTER(SolverConfigC), c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "tb_tiled_create": (c_int32, [c_void_p, c_int32, ctypes.POINTER(SolverConfigC), c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, ctypes.POINTER(c_void_p)]),
    "tb_tiled_round_a": (c_int32, [c_void_p, c_void_p]),
    "tb_tiled_round_b": (c_int32, [c_void_p, c_void_p]),
    "tb_tiled_remaining": (c_int32, [c_void_p, ctypes.POINTER(c_int64), c_void_p]),
    "tb_tiled_finish": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tb_tiled_destroy": (c_int32, [c_void_p]),
    "tb_apply_filter": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "tb_build_steering": (c_int32, [c_int32, c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_void_p, ctypes.POINTER(c_int32), c_int64, c_int64, c_double, c_void_p, c_void_p]),
    "tb_select": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, ctypes.POINTER(c_int32), c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
}

_LIB = None


def load() -> ctypes.CDLL:
    """Load (once) the in-tree library; raises NumericalError if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise NumericalError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(code: int) -> None:
    """Map a C-ABI return code onto the reference's exception taxonomy."""
    if code == TB_OK:
        return
    msg = (load().tb_last_error() or b"").decode(errors="replace")
    if code == TB_ERR_INVALID:
        raise ConfigurationError(msg)
    if code == TB_ERR_CAPACITY:
        raise CapacityError(msg)
    raise NumericalError(msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def last_solver_kernel() -> str:
    """Kernel family the last solve chose (tb_last_solver_kernel)."""
    return load().tb_last_solver_kernel().decode()


def launch_count() -> int:
    """Kernels launched by the library so far (tb_launch_count)."""
    return int(load().tb_launch_count())
