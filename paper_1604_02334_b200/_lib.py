"""ctypes binding of libmusr_b200.so (C ABI: include/musr_b200.h).

The library is loaded lazily on first use.  There is no fallback: if the
shared object is missing, or no CUDA device is visible, every objective call
raises ``MusrDeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

LIB_PATH = Path(__file__).resolve().parent / "libmusr_b200.so"

MUSR_OK = 0
KIND_CHI2 = 0
KIND_MLH = 1
ROUND_TERMS = 256

_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_VPP = C.POINTER(C.c_void_p)


class MusrDeviceError(RuntimeError):
    """Raised when the GPU library cannot be loaded or a device call fails."""


# (name, restype, argtypes) -- one line per symbol of include/musr_b200.h
SIGNATURES = [
    ("musr_version", C.c_int, []),
    ("musr_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("musr_global_error", C.c_char_p, []),
    ("musr_open", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("musr_nccl_unique_id", C.c_int, [C.c_char_p, C.c_char_p]),
    ("musr_open_sharded", C.c_int,
     [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    ("musr_open_shared", C.c_int,
     [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("musr_collect_results", C.c_int,
     [C.POINTER(C.c_uint64), C.c_int, C.c_uint, _DP, _I64P, _DP]),
    ("musr_close", None, [C.c_void_p]),
    ("musr_last_error", C.c_char_p, [C.c_void_p]),
    ("musr_set_theory", C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]),
    ("musr_set_uniform_program", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    ("musr_set_tile_shape", C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    ("musr_eval_uniform_rows", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    ("musr_compile_theory", C.c_int,
     [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("musr_upload", C.c_int,
     [C.c_void_p, C.c_int, C.c_int, _I32P, _I64P, _I64P, _I64P, _DP, _VPP, _VPP, _VPP,
      _I32P, _I32P, _I32P, C.c_int, _DP, C.c_int, C.c_int]),
    ("musr_eval", C.c_int, [C.c_void_p, C.c_int, _DP, C.c_int, _DP, _I64P, _DP]),
    ("musr_eval_batch", C.c_int, [C.c_void_p, C.c_int, _DP, C.c_int, C.c_int, _DP, _I64P, _DP]),
    ("musr_time_evals", C.c_int,
     [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
      C.POINTER(C.c_double)]),
    ("musr_tiles", C.c_int, [C.c_void_p, _I64P]),
    ("musr_n_datasets", C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    ("musr_minimize", C.c_int,
     [C.c_void_p, C.c_int, _DP, C.c_int, _I32P, C.c_int, _DP, C.c_double, _DP, _DP, _DP,
      C.c_double, C.c_int64, C.c_int, _DP, _DP, _I64P, _I64P, C.POINTER(C.c_int), _DP]),
    ("musr_nm_run", C.c_int,
     [C.c_int, _DP, C.c_double, _DP, _DP, _DP, C.c_double, C.c_int64, C.c_int, C.c_void_p,
      C.c_void_p, _DP, _DP, _I64P, _I64P, C.POINTER(C.c_int), _DP]),
    ("musr_format", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("musr_debug_trace", C.c_int,
     [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]),
    ("musr_fp64_peak", C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    # muSR data files (struct pointers as void*; musrio.py retypes them with its Structures)
    ("musr_file_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p), C.c_void_p]),
    ("musr_file_n_detectors", C.c_int, [C.c_void_p]),
    ("musr_file_detector", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("musr_file_copy", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    ("musr_file_free", None, [C.c_void_p]),
    ("musr_file_store", C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_char_p),
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_int,
                                  C.c_void_p]),
]

_lib: Optional[C.CDLL] = None


def load() -> C.CDLL:
    """Load and type the shared library (raises MusrDeviceError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise MusrDeviceError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1604_02334_b200._build` "
            "(there is no CPU fallback)"
        )
    try:
        lib = C.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise MusrDeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_EVAL_RAW = None


def eval_raw():
    """musr_eval typed with plain integer pointers: the per-evaluation call
    from Python is the hot host path, and raw addresses avoid building
    ctypes pointer objects on every call."""
    global _EVAL_RAW
    if _EVAL_RAW is None:
        lib = load()
        fn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                         C.c_void_p, C.c_void_p)(("musr_eval", lib))
        _EVAL_RAW = fn
    return _EVAL_RAW


_PYFAST = None


def pyfast():
    """The CPython fast path of the drop-in call (csrc/musr_pyfast.c), bound to
    this library's musr_eval.  Built next to the library by _build; missing
    means the package was not built."""
    global _PYFAST
    if _PYFAST is None:
        lib = load()
        try:
            from . import _pyfast as mod
        except ImportError as exc:
            raise MusrDeviceError(
                f"the host extension _pyfast is missing ({exc}): build it with "
                "`python -m paper_1604_02334_b200._build`") from exc
        import numpy as np

        mod.init(C.cast(lib.musr_eval, C.c_void_p).value, np.ndarray, np.dtype(np.float64))
        _PYFAST = mod
    return _PYFAST


def nccl_library_path() -> Optional[str]:
    """Path of the torch-bundled libnccl.so.2, if installed."""
    env = os.environ.get("MUSR_NCCL_LIB")
    if env:
        return env
    try:
        import nvidia.nccl  # type: ignore

        for base in nvidia.nccl.__path__:
            cand = Path(base) / "lib" / "libnccl.so.2"
            if cand.exists():
                return str(cand)
    except ImportError:
        pass
    return None


def check(rc: int, handle=None, what: str = "") -> None:
    if rc == MUSR_OK:
        return
    lib = load()
    msg = lib.musr_last_error(handle) if handle else lib.musr_global_error()
    text = msg.decode(errors="replace") if msg else ""
    raise MusrDeviceError(f"{what} failed (status {rc}): {text}")


def device_count() -> int:
    lib = load()
    n = C.c_int(0)
    lib.musr_device_count(C.byref(n))
    return n.value


def fp64_peak_tflops(device: int = 0) -> float:
    lib = load()
    out = C.c_double(0.0)
    check(lib.musr_fp64_peak(device, C.byref(out)), None, "musr_fp64_peak")
    return out.value
