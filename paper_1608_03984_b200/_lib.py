"""ctypes binding of libb200fd.so (include/b200fd.h).

The library is built in-tree by `make` / `__graft_entry__.build()`.  There is
no CPU fallback: if the shared object is missing, importing anything that
needs it raises `ExtensionMissingError`.
"""

import ctypes
import os
import threading

from .errors import DeviceError, ExtensionMissingError, ValidationError

LIB_NAME = "libb200fd.so"
LIB_PATH = os.environ.get("B200FD_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

ABI_VERSION = 4
MAX_RADIUS = 16

FDR_OK, FDR_EINVAL, FDR_ECUDA = 0, -1, -2
M_NONE, M_SCALAR, M_GRID = 0, 1, 2
(VARIANT_AUTO, VARIANT_DIRECT, VARIANT_TMA, VARIANT_QUEUE, VARIANT_PERSISTENT, VARIANT_CLUSTER,
 VARIANT_TB2, VARIANT_FMA, VARIANT_QUEUE2) = (0, 1, 2, 3, 4, 5, 6, 7, 8)

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32


class AcousticArgs(ctypes.Structure):
    """Mirror of `fdr_acoustic_args` (include/b200fd.h)."""

    _fields_ = [
        ("abi_version", _i32),
        ("order", _i32),
        ("nx", _i32),
        ("ny", _i32),
        ("nz", _i32),
        ("pitch_y", _i32),
        ("pitch_x", ctypes.c_int64),
        ("weights", ctypes.c_float * (MAX_RADIUS + 1)),
        ("coef", ctypes.c_float),
        ("m_mode", _i32),
        ("m_scalar", ctypes.c_float),
        ("m_lo", ctypes.c_float),
        ("m_hi", ctypes.c_float),
        ("m", _vp),
        ("levels", _vp * 3),
        ("sponge_x", _vp),
        ("sponge_y", _vp),
        ("sponge_z", _vp),
        ("series", _vp),
        ("n_series", _i32),
        ("src_x", _i32),
        ("src_y", _i32),
        ("src_z", _i32),
        ("n_rec", _i32),
        ("rec_xyz", _vp),
        ("traces", _vp),
        ("trace_rows", _i32),
        ("it0", _i32),
        ("n_steps", _i32),
        ("variant", _i32),
        ("rec_w", _vp),
        ("src_w", _vp),
    ]


class Acoustic64Args(ctypes.Structure):
    """Mirror of `fdr_acoustic64_args` (include/b200fd.h): the float64 step."""

    _fields_ = [
        ("abi_version", _i32),
        ("order", _i32),
        ("nx", _i32),
        ("ny", _i32),
        ("nz", _i32),
        ("pitch_y", _i32),
        ("pitch_x", ctypes.c_int64),
        ("weights", ctypes.c_double * (MAX_RADIUS + 1)),
        ("coef", ctypes.c_double),
        ("m_mode", _i32),
        ("m_scalar", ctypes.c_double),
        ("m", _vp),
        ("levels", _vp * 3),
        ("sponge_x", _vp),
        ("sponge_y", _vp),
        ("sponge_z", _vp),
        ("series", _vp),
        ("n_series", _i32),
        ("src_x", _i32),
        ("src_y", _i32),
        ("src_z", _i32),
        ("n_rec", _i32),
        ("rec_xyz", _vp),
        ("traces", _vp),
        ("trace_rows", _i32),
        ("it0", _i32),
        ("n_steps", _i32),
        ("variant", _i32),
    ]


# Every symbol include/b200fd.h declares: (name, restype, argtypes).
EXPORTS = (
    ("fdr_abi_version", ctypes.c_int, ()),
    ("fdr_acoustic_args_size", ctypes.c_size_t, ()),
    ("fdr_last_error", ctypes.c_char_p, ()),
    ("fdr_device_count", ctypes.c_int, ()),
    ("fdr_acoustic_run", ctypes.c_int, (ctypes.POINTER(AcousticArgs), _vp)),
    ("fdr_acoustic_slabs_run", ctypes.c_int,
     (ctypes.POINTER(AcousticArgs), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
      ctypes.POINTER(ctypes.c_void_p))),
    ("fdr_acoustic_oracle_step", ctypes.c_int,
     (ctypes.POINTER(AcousticArgs), ctypes.POINTER(ctypes.c_double), ctypes.c_double,
      ctypes.c_double, _vp, _vp)),
    ("fdr_acoustic_workspace_bytes", ctypes.c_size_t, (ctypes.POINTER(AcousticArgs),)),
    (
        "fdr_acoustic_run_host",
        ctypes.c_int,
        (ctypes.POINTER(AcousticArgs), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         ctypes.c_size_t, _vp),
    ),
    (
        "fdr_acoustic_run_host_async",
        ctypes.c_int,
        (ctypes.POINTER(AcousticArgs), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         ctypes.c_size_t, _vp),
    ),
    ("fdr_acoustic_host_upload", ctypes.c_int,
     (ctypes.POINTER(AcousticArgs), _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp)),
    ("fdr_acoustic_host_run_ws", ctypes.c_int,
     (ctypes.POINTER(AcousticArgs), ctypes.c_int, _vp, ctypes.c_size_t, _vp)),
    ("fdr_acoustic_host_download", ctypes.c_int,
     (ctypes.POINTER(AcousticArgs), ctypes.c_int, _vp, _vp, _vp, ctypes.c_size_t, _vp)),
    ("fdr_last_launch_count", ctypes.c_int64, ()),
    ("fdr_pending_error", ctypes.c_int, ()),
    ("fdr_fp32_fma_peak", ctypes.c_int,
     (ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
      ctypes.POINTER(ctypes.c_double))),
    ("fdr_count_nonfinite", ctypes.c_int,
     (_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
      ctypes.POINTER(ctypes.c_int64), _vp)),
    ("fdr_tti_args_size", ctypes.c_size_t, ()),
    ("fdr_tti_run", ctypes.c_int, (ctypes.c_void_p, _vp)),
    ("fdr_elastic_args_size", ctypes.c_size_t, ()),
    ("fdr_elastic_run", ctypes.c_int, (ctypes.c_void_p, _vp)),
    ("fdr_tti64_args_size", ctypes.c_size_t, ()),
    ("fdr_tti64_run", ctypes.c_int, (ctypes.c_void_p, _vp)),
    ("fdr_elastic64_args_size", ctypes.c_size_t, ()),
    ("fdr_elastic64_run", ctypes.c_int, (ctypes.c_void_p, _vp)),
    ("fdr_acoustic64_args_size", ctypes.c_size_t, ()),
    ("fdr_acoustic64_run", ctypes.c_int, (ctypes.POINTER(Acoustic64Args), _vp)),
    ("fdr_selftest_division64", ctypes.c_int64,
     (ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_uint32,
      ctypes.POINTER(ctypes.c_int64))),
    ("fdr_selftest_division", ctypes.c_int64,
     (ctypes.c_int64, ctypes.c_float, ctypes.c_float, ctypes.c_uint32,
      ctypes.POINTER(ctypes.c_int64))),
)

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the library handle with typed entry points."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissingError(
                f"{LIB_PATH} is not built; run `make` or __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in EXPORTS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = list(args)
        if lib.fdr_abi_version() != ABI_VERSION:
            raise ExtensionMissingError(
                f"library ABI {lib.fdr_abi_version()} != binding ABI {ABI_VERSION}"
            )
        if lib.fdr_acoustic_args_size() != ctypes.sizeof(AcousticArgs):
            raise ExtensionMissingError("fdr_acoustic_args layout mismatch between header and binding")
        if lib.fdr_acoustic64_args_size() != ctypes.sizeof(Acoustic64Args):
            raise ExtensionMissingError("fdr_acoustic64_args layout mismatch between header and binding")
        _lib = lib
        return lib


def check(rc: int) -> int:
    """Map a C return code to the reference's exception conventions."""
    if rc >= 0:
        return rc
    msg = (load().fdr_last_error() or b"").decode(errors="replace")
    if rc == FDR_EINVAL:
        raise ValidationError(msg)
    raise DeviceError(msg or f"libb200fd error {rc}")
