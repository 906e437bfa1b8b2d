"""Host <-> device plumbing: storage conversion, K-major packing, prepared weights.

PyTorch provides device memory and the current stream; all arithmetic runs in
the C-ABI library.  Storage semantics follow the reference's ``storage_array``
(checksum.py:55-62): binary16 -> fp16, exact-int -> integer-valued fp16 (exact
while |v| <= 2048 with fp32 accumulation below 2**24), bfloat16 -> bf16.
binary32 has no tensor-core path with the reference's 2**-23 tolerance and is
rejected.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import ExactOverflowError, ShapeMismatchError
from .shapes import BFLOAT16, BINARY16, BINARY32, EXACT_INT, DType, DTypeTag

FP16_INT_MAX = 2048          # integers |v| <= 2048 are exact in fp16
FP32_INT_MAX = 2 ** 24       # ... and partial sums stay exact in fp32 below 2**24

_torch = None


def torch():
    """Lazy torch import (kept out of module import time for the CPU test suite)."""
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_device():
    t = torch()
    _lib.load()
    if not t.cuda.is_available():
        raise _lib.AbftLibraryError("no CUDA device visible: the B200 path has no CPU fallback")


def sm_count() -> int:
    """SM count of the current device (the persistent grid's upper bound)."""
    return int(torch().cuda.get_device_properties(torch().cuda.current_device()).multi_processor_count)


def stream_handle() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def round8(x: int) -> int:
    return -(-x // 8) * 8


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def dtype_of(x) -> DType:
    """Numeric mode from the element type (checksum.py:46-52, plus torch bf16)."""
    if is_torch(x):
        t = torch()
        if x.dtype in (t.int8, t.int16, t.int32, t.int64, t.uint8):
            return EXACT_INT
        if x.dtype == t.float16:
            return BINARY16
        if x.dtype == t.bfloat16:
            return BFLOAT16
        return BINARY32
    x = np.asarray(x)
    if np.issubdtype(x.dtype, np.integer):
        return EXACT_INT
    return BINARY16 if x.dtype == np.float16 else BINARY32


def numeric_code(dtype: DType) -> int:
    return {DTypeTag.EXACT_INT: _lib.NUM_EXACT, DTypeTag.BINARY16: _lib.NUM_BINARY16,
            DTypeTag.BINARY32: _lib.NUM_BINARY32, DTypeTag.BFLOAT16: _lib.NUM_BF16}[dtype.tag]


def storage_code(dtype: DType) -> int:
    if dtype.tag is DTypeTag.BINARY32:
        raise _lib.UnsupportedConfigError(
            "binary32 GEMMs have no tensor-core path with the reference's 2**-23 tolerance; "
            "use binary16 / bfloat16 storage (or exact-int)")
    return _lib.BF16 if dtype.tag is DTypeTag.BFLOAT16 else _lib.F16


def torch_storage_dtype(dtype: DType):
    t = torch()
    return t.bfloat16 if storage_code(dtype) == _lib.BF16 else t.float16


def shape2d(x, name: str) -> tuple:
    shp = tuple(x.shape)
    if len(shp) != 2 or shp[0] * shp[1] == 0:
        raise ShapeMismatchError(f"{name} must be a non-empty 2-D matrix, got shape {shp}")
    return shp


def max_abs(x) -> float:
    if is_torch(x):
        return float(x.abs().max().item()) if x.numel() else 0.0
    x = np.asarray(x)
    return float(np.abs(x).max()) if x.size else 0.0


def guard_exact(a, b=None, k: Optional[int] = None, what: str = "matmul accumulation") -> None:
    """Exactness guard of the tensor-core exact-int path (cf. checksum.py:72-74)."""
    ma = max_abs(a)
    if ma > FP16_INT_MAX:
        raise ExactOverflowError(f"{what}: |values| up to {ma:.0f} exceed the exact fp16 range {FP16_INT_MAX}")
    if b is not None:
        mb = max_abs(b)
        if mb > FP16_INT_MAX:
            raise ExactOverflowError(f"{what}: |values| up to {mb:.0f} exceed the exact fp16 range {FP16_INT_MAX}")
        if k * max(ma, 1) * max(mb, 1) >= FP32_INT_MAX:
            raise ExactOverflowError(f"{what} may exceed the exact fp32 accumulation range (bound "
                                     f"{k * max(ma, 1) * max(mb, 1):.0f} >= 2**24)")


def _to_storage_tensor(x, dtype: DType):
    """Host or device array -> contiguous CUDA tensor in the storage element type."""
    t = torch()
    sd = torch_storage_dtype(dtype)
    if is_torch(x):
        return x.to(device="cuda", dtype=sd).contiguous()
    x = np.asarray(x)
    if sd == t.float16:
        host = np.ascontiguousarray(x.astype(np.float16))
        return t.from_numpy(host).to("cuda", non_blocking=False)
    return t.from_numpy(np.ascontiguousarray(x.astype(np.float32))).to("cuda").to(t.bfloat16)


def upload(x, dtype: DType, name: str = "A"):
    """[rows x cols] -> CUDA storage tensor [rows x round8(cols)] (zero-padded K)."""
    rows, cols = shape2d(x, name)
    t = torch()
    src = _to_storage_tensor(x, dtype)
    if cols % 8 == 0 and src.data_ptr() % 16 == 0:
        return src
    dst = t.empty((rows, round8(cols)), dtype=src.dtype, device="cuda")
    _lib.call("abft_pack", ptr(src), rows, cols, cols, ptr(dst), round8(cols), round8(cols), 0, stream_handle())
    return dst


def upload_transposed(b, dtype: DType, name: str = "B"):
    """B [K x N] -> B^T [N x round8(K)] K-major (zero-padded K), the weight layout of the kernels."""
    k, n = shape2d(b, name)
    t = torch()
    src = _to_storage_tensor(b, dtype)
    dst = t.empty((n, round8(k)), dtype=src.dtype, device="cuda")
    _lib.call("abft_pack", ptr(src), k, n, n, ptr(dst), round8(k), round8(k), 1, stream_handle())
    return dst


def faults_tensor(cells):
    """[(row, col, delta)] -> device array of abft_fault_t (None when empty)."""
    if not cells:
        return None, 0
    t = torch()
    rec = np.zeros(len(cells), dtype=np.dtype([("row", "<i4"), ("col", "<i4"), ("delta", "<f4")]))
    for i, (r, c, d) in enumerate(cells):
        rec[i] = (int(r), int(c), np.float32(d))
    dev = t.from_numpy(rec.view(np.uint8).copy()).to("cuda")
    return dev, len(cells)


@dataclass
class PreparedWeight:
    """A weight matrix in the kernels' layout plus its offline row checksum.

    bt     [N x K8] K-major storage (B transposed, K zero-padded to a multiple of 8)
    rowck  [K8] fp32 row checksum of B (checksum.py:99-105 / :175-187)
    """

    bt: object
    rowck: object
    k: int
    n: int
    dtype: DType

    @property
    def ldbt(self) -> int:
        return self.bt.shape[1]


def prepare_weight(b, dtype: DType, with_rowck: bool = True) -> PreparedWeight:
    k, n = shape2d(b, "B")
    bt = upload_transposed(b, dtype)
    rowck = None
    if with_rowck:
        # zero-padded to a whole number of 64-column k-blocks (the global lhs_rowck layout)
        rowck = torch().zeros(-(-bt.shape[1] // 64) * 64, dtype=torch().float32, device="cuda")
        _lib.call("abft_colsum", ptr(bt), n, bt.shape[1], bt.shape[1], storage_code(dtype), ptr(rowck), 0,
                  stream_handle())
    return PreparedWeight(bt=bt, rowck=rowck, k=k, n=n, dtype=dtype)


# offline weight-checksum cache keyed by identity (checksum.py:172-191 semantics)
_prepared: dict = {}


def prepared_weight_cached(b, dtype: DType) -> PreparedWeight:
    key = (id(b), dtype.tag)
    hit = _prepared.get(key)
    if hit is not None and hit[0] is b:
        return hit[1]
    pw = prepare_weight(b, dtype)
    _prepared[key] = (b, pw)
    return pw


def clear_prepared_cache() -> None:
    _prepared.clear()


def colck_device(a_dev, rows: int, dtype: DType):
    """Activation column checksum of a device storage matrix -> fp32 [cols]."""
    out = torch().empty(a_dev.shape[1], dtype=torch().float32, device="cuda")
    _lib.call("abft_colsum", ptr(a_dev), rows, a_dev.shape[1], a_dev.stride(0), storage_code(dtype), ptr(out), 0,
              stream_handle())
    return out


def to_host_like(t, like):
    """Return torch results for torch inputs, numpy for everything else."""
    if is_torch(like):
        return t
    return t.detach().cpu().numpy()
