"""ctypes binding of libtsm2x.so (declarations: include/tsm2x.h).

The product path has no fallback: if the library is missing or cannot load, every entry point
raises RuntimeError naming the build command. ctypes releases the GIL around each call.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSM2X_LIB_PATH_EXPERIMENT") or os.path.join(_HERE, "libtsm2x.so")

OK, EINVAL, ECUDA, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -4
FLAG_C_IS_ZERO, FLAG_CHECK_ZERO_C, FLAG_DETERMINISTIC = 0x1, 0x2, 0x4
IMPL = {"auto": 0, "ldg": 1, "tma": 2, "tsm2l": 3, "ablation": 4, "tsm2l-splitn": 5}
SINGLE, DOUBLE = 0, 1

EXPORTS = (
    "tsm2x_validate",
    "tsm2x_run",
    "tsm2x_run_ex",
    "tsm2x_run_host",
    "tsm2x_run_host_multi",
    "tsm2x_run_multi",
    "tsm2x_row_range",
    "tsm2x_fill_uniform",
    "tsm2x_release_cached",
    "tsm2x_last_error",
    "tsm2x_version",
    "tsm2x_build_target",
    "tsm2x_launch_count",
    "tsm2x_set_kernel_events",
    "tsm2x_set_tuning",
    "tsm2x_get_tuning",
    "tsm2x_plan_for",
)


class Tuning(ctypes.Structure):
    """struct tsm2x_tuning (B200 parameter selection knobs; 0 = default)."""

    _fields_ = [("consumer", ctypes.c_int32), ("small_kb", ctypes.c_int32), ("big_kb", ctypes.c_int32),
                ("tail_pct", ctypes.c_int32), ("batch_kb", ctypes.c_int32), ("combine", ctypes.c_int32)]


class Plan(ctypes.Structure):
    """struct tsm2x_plan (what a call would launch)."""

    _fields_ = [("impl", ctypes.c_int32), ("consumer", ctypes.c_int32), ("rows_per_block", ctypes.c_int32),
                ("cols_per_pass", ctypes.c_int32), ("cols_per_stage", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("passes", ctypes.c_int32), ("deterministic", ctypes.c_int32), ("grid", ctypes.c_int64),
                ("items", ctypes.c_int64), ("nbig", ctypes.c_int64), ("kbig", ctypes.c_int64),
                ("nsmall", ctypes.c_int64), ("ksmall", ctypes.c_int64), ("batch", ctypes.c_int64)]


class Params(ctypes.Structure):
    """struct tsm2x_params (reference KernelParams, core.py:160-190)."""

    _fields_ = [("t1", ctypes.c_int32), ("t2", ctypes.c_int32), ("t3", ctypes.c_int32),
                ("tcf", ctypes.c_int32), ("variant", ctypes.c_int32)]


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(or `make -C paper_2002_03258_b200/csrc`). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        i64, i32, u32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        pp = ctypes.POINTER(Params)
        lib.tsm2x_validate.argtypes = [i32, i64, i64, i64, pp]
        lib.tsm2x_run.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, pp, u32, vp]
        lib.tsm2x_run_ex.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, pp, u32, i32, vp]
        lib.tsm2x_run_host.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, vp, i64, pp, u32, i32]
        lib.tsm2x_run_host_multi.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, vp, i64, pp, u32, i32,
                                             ctypes.POINTER(ctypes.c_int)]
        lib.tsm2x_run_multi.argtypes = [i32, i32, i64, i64, i64, i32, ctypes.POINTER(ctypes.c_int), vp,
                                        ctypes.POINTER(i64), vp, i64, vp, ctypes.POINTER(i64), pp, u32, vp]
        lib.tsm2x_row_range.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        lib.tsm2x_row_range.restype = None
        lib.tsm2x_fill_uniform.argtypes = [i32, i64, i64, vp, i64, i64, i64, ctypes.c_uint64, vp]
        lib.tsm2x_set_kernel_events.argtypes = [vp, vp]
        lib.tsm2x_set_tuning.argtypes = [ctypes.POINTER(Tuning)]
        lib.tsm2x_get_tuning.argtypes = [ctypes.POINTER(Tuning)]
        lib.tsm2x_plan_for.argtypes = [i32, i64, i64, i64, i64, i32, u32, i32, ctypes.POINTER(Plan)]
        lib.tsm2x_release_cached.argtypes = [i32]
        for name in ("tsm2x_validate", "tsm2x_run", "tsm2x_run_ex", "tsm2x_run_host", "tsm2x_run_host_multi",
                     "tsm2x_run_multi", "tsm2x_fill_uniform",
                     "tsm2x_version", "tsm2x_set_kernel_events", "tsm2x_set_tuning", "tsm2x_get_tuning",
                     "tsm2x_plan_for", "tsm2x_release_cached"):
            getattr(lib, name).restype = ctypes.c_int
        lib.tsm2x_last_error.restype = ctypes.c_char_p
        lib.tsm2x_build_target.restype = ctypes.c_char_p
        lib.tsm2x_launch_count.restype = ctypes.c_int64
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Maps a C return code to the reference's exception types."""
    if rc == OK:
        return
    msg = load().tsm2x_last_error().decode("utf-8", "replace")
    if rc == EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"libtsm2x error {rc}: {msg}")


def launch_count() -> int:
    return int(load().tsm2x_launch_count())
