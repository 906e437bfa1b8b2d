"""ctypes binding of the in-tree C-ABI library ``lib/libabft_b200.so``.

The declarations mirror ``include/abft_b200.h`` one to one.  There is no CPU
fallback: importing the product API on a machine where the library cannot be
loaded raises ``AbftLibraryError`` at the first call that needs the GPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import AbftGuardError, ExactOverflowError, ShapeMismatchError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("ABFT_B200_LIB") or os.path.join(LIB_DIR, "libabft_b200.so")

# enums of abft_b200.h
OK, E_SHAPE, E_VALUE, E_OVERFLOW, E_CUDA, E_UNSUPPORTED = range(6)
F16, BF16 = 0, 1
OUT_F32, OUT_F16, OUT_BF16, OUT_NONE = 0, 1, 2, 3
NUM_EXACT, NUM_BINARY16, NUM_BINARY32, NUM_BF16 = 0, 1, 2, 3
UNPROTECTED, GLOBAL, ONE_SIDED, TWO_SIDED, REPL_FULL, REPL_SINGLE = range(6)

EXPORTED_SYMBOLS = (
    "abft_verify_partials",
    "abft_struct_size",
    "abft_gemm",
    "abft_gemm_plan",
    "abft_ck_rows",
    "abft_aug_weights",
    "abft_colsum",
    "abft_pack",
    "abft_convert_i64",
    "abft_matrix_sum",
    "abft_zero",
    "abft_conv2d",
    "abft_conv_plan",
    "abft_conv_gemm_plan",
    "abft_conv_pack_weight",
    "abft_conv_colck",
    "abft_global_lhs",
    "abft_verify_sums",
    "abft_global_verify",
    "abft_last_error",
    "abft_version",
    "abft_device_sms",
    "abft_window_lhs",
    "abft_gemm_group_prepare",
    "abft_gemm_group_launch",
    "abft_group_problem_bytes",
    "abft_nhwc_border_sums",
    "abft_nhwc_maxpool",
    "abft_nhwc_maxpool_ws",
    "abft_nhwc_avgpool",
    "abft_nhwc_interleave2",
    "abft_sum_partials",
    "abft_fused_lhs_batch_bytes",
    "abft_fused_lhs_batch_prepare",
    "abft_fused_lhs_batch_launch",
)


class AbftLibraryError(AbftGuardError, RuntimeError):
    """The CUDA library is missing, failed to load, or a launch failed."""


class UnsupportedConfigError(AbftGuardError, ValueError):
    """A configuration the sm_100a tensor-core path does not cover."""


class Fault(ctypes.Structure):
    _fields_ = [("row", ctypes.c_int32), ("col", ctypes.c_int32), ("delta", ctypes.c_float)]


class VerdictC(ctypes.Structure):
    _fields_ = [("lhs", ctypes.c_double), ("rhs", ctypes.c_double), ("tol", ctypes.c_double),
                ("detected", ctypes.c_int32), ("k", ctypes.c_int32)]


class ThreadVerdictC(ctypes.Structure):
    _fields_ = [("t_row", ctypes.c_int32), ("t_col", ctypes.c_int32), ("detected", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("max_abs_diff", ctypes.c_double), ("tol", ctypes.c_double)]


class BorderTask(ctypes.Structure):
    """abft_border_task_t: one producer's border buckets (abft_nhwc_border_sums arguments)."""
    _fields_ = [("x", ctypes.c_void_p), ("wsum", ctypes.c_void_p), ("ldx", ctypes.c_int64),
                ("n", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32), ("c", ctypes.c_int32),
                ("ws_ld", ctypes.c_int32)]


class WindowTask(ctypes.Structure):
    """abft_window_task_t: one fused consumer's window lhs (abft_window_lhs arguments)."""
    _fields_ = [("wsum", ctypes.c_void_p), ("rowck", ctypes.c_void_p), ("bias", ctypes.c_void_p),
                ("lhs", ctypes.c_void_p), ("M", ctypes.c_int64), ("ws_ld", ctypes.c_int32), ("C", ctypes.c_int32),
                ("R", ctypes.c_int32), ("S", ctypes.c_int32), ("ck", ctypes.c_int32), ("n_out", ctypes.c_int32)]


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("Bt", ctypes.c_void_p), ("ldbt", ctypes.c_int64),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64),
        ("M", ctypes.c_int32), ("N", ctypes.c_int32), ("K", ctypes.c_int32),
        ("m_ext", ctypes.c_int32), ("n_ext", ctypes.c_int32), ("tol_k", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32), ("numeric", ctypes.c_int32),
        ("scheme", ctypes.c_int32),
        ("thread_m", ctypes.c_int32), ("thread_n", ctypes.c_int32),
        ("relu", ctypes.c_int32), ("ck_split", ctypes.c_int32),
        ("faults", ctypes.c_void_p), ("nfaults", ctypes.c_int32),
        ("out_sum", ctypes.c_void_p),
        ("next_colck", ctypes.c_void_p),
        ("verdicts", ctypes.c_void_p),
        ("fired_count", ctypes.c_void_p),
        ("fired", ctypes.c_void_p),
        ("fired_cap", ctypes.c_int32),
        ("tile_n", ctypes.c_int32),
        ("num_sms", ctypes.c_int32),
        ("ck_rows", ctypes.c_void_p), ("ldck", ctypes.c_int64), ("ck_rows_n", ctypes.c_int32),
        ("a_colck", ctypes.c_void_p),
        ("out_lhs", ctypes.c_void_p),
        ("vsums", ctypes.c_void_p), ("vk", ctypes.c_void_p), ("vn", ctypes.c_int32), ("vdone", ctypes.c_void_p),
        ("vout", ctypes.c_void_p), ("vdetected", ctypes.c_void_p),
        ("pdl", ctypes.c_int32), ("ck_layout", ctypes.c_int32),
        ("lhs_rowck", ctypes.c_void_p),
        ("out_partials", ctypes.c_void_p), ("partials_cap", ctypes.c_int32),
        ("bias", ctypes.c_void_p), ("residual", ctypes.c_void_p), ("ld_res", ctypes.c_int64),
        ("plan_flags", ctypes.c_int32),
        ("wsum", ctypes.c_void_p), ("ws_ld", ctypes.c_int32), ("ws_mode", ctypes.c_int32),
        ("ws_P", ctypes.c_int32), ("ws_Q", ctypes.c_int32),
    ]


class ConvArgs(ctypes.Structure):
    _fields_ = [("gemm", GemmArgs),
                ("n", ctypes.c_int32), ("h", ctypes.c_int32), ("w", ctypes.c_int32), ("c", ctypes.c_int32),
                ("r", ctypes.c_int32), ("s", ctypes.c_int32), ("stride_h", ctypes.c_int32),
                ("stride_w", ctypes.c_int32), ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
                ("c_real", ctypes.c_int32), ("workspace", ctypes.c_void_p), ("ws_bytes", ctypes.c_int64)]


class GlobalTask(ctypes.Structure):
    _fields_ = [("colck", ctypes.c_void_p), ("rowck", ctypes.c_void_p), ("rhs", ctypes.c_void_p),
                ("k", ctypes.c_int32), ("tol_k", ctypes.c_int32)]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.abft_gemm.argtypes = [ctypes.POINTER(GemmArgs), vp]
    lib.abft_gemm_plan.argtypes = [ctypes.POINTER(GemmArgs), vp]
    lib.abft_ck_rows.argtypes = [vp, i32, i32, i64, i32, i32, i32, i32, i32, i32, vp, i64, vp]
    lib.abft_aug_weights.argtypes = [vp, i32, i32, i64, i32, i32, i32, i32, i32, i32, i32, vp, i64, vp]
    lib.abft_colsum.argtypes = [vp, i32, i32, i64, i32, vp, i32, vp]
    lib.abft_pack.argtypes = [vp, i32, i32, i64, vp, i32, i64, i32, vp]
    lib.abft_convert_i64.argtypes = [vp, i64, i32, vp, vp]
    lib.abft_matrix_sum.argtypes = [vp, i32, i32, i64, i32, vp, vp]
    lib.abft_zero.argtypes = [vp, i64, vp]
    lib.abft_global_lhs.argtypes = [vp, i32, vp, vp]
    lib.abft_global_verify.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    lib.abft_verify_sums.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    lib.abft_verify_partials.argtypes = [vp, i32, vp, i32, i32, vp, vp, vp]
    lib.abft_conv2d.argtypes = [ctypes.POINTER(ConvArgs), vp]
    lib.abft_conv_plan.argtypes = [ctypes.POINTER(ConvArgs), vp]
    lib.abft_conv_gemm_plan.argtypes = [ctypes.POINTER(ConvArgs), vp]
    lib.abft_conv_pack_weight.argtypes = [vp, i32, i32, i32, i32, i32, vp, i64, vp]
    lib.abft_conv_colck.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp, i32, vp]
    lib.abft_last_error.restype = ctypes.c_char_p
    for name in EXPORTED_SYMBOLS:
        fn = getattr(lib, name)
        if name != "abft_last_error":
            fn.restype = ctypes.c_int
    lib.abft_fused_lhs_batch_bytes.restype = ctypes.c_int64
    lib.abft_fused_lhs_batch_bytes.argtypes = [i32, i32]
    return lib


def load(path: str = LIB_PATH):
    """Load (once) and return the library handle; raise loudly if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise AbftLibraryError(
                    f"CUDA library not built: {path} is missing (run __graft_entry__.build() "
                    "or `make -C paper_2104_09455_b200/csrc`)")
            try:
                _lib = _declare(ctypes.CDLL(path))
            except OSError as exc:
                raise AbftLibraryError(f"cannot load {path}: {exc}") from None
        return _lib


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference exception hierarchy (errors.py)."""
    if rc == OK:
        return
    msg = load().abft_last_error().decode(errors="replace")
    if rc == E_SHAPE:
        raise ShapeMismatchError(msg)
    if rc == E_VALUE:
        raise ValueError(msg)
    if rc == E_OVERFLOW:
        raise ExactOverflowError(msg)
    if rc == E_UNSUPPORTED:
        raise UnsupportedConfigError(msg)
    raise AbftLibraryError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
