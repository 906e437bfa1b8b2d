"""Typed launchers over the C-ABI (device tensors in, nothing synchronised).

These are the calls the drop-in API (``tiled``, ``checksum``), the network
runner, the profiler and ``bench.py`` share.  Every function enqueues work on
torch's current CUDA stream and returns immediately.
"""

from __future__ import annotations

import ctypes
from typing import Optional

from . import _lib
from .device import ptr, storage_code, stream_handle, torch
from .schemes import SCHEME_CODE, Scheme
from .shapes import DType

OUT_CODES = {"f32": _lib.OUT_F32, "f16": _lib.OUT_F16, "bf16": _lib.OUT_BF16, None: _lib.OUT_NONE}


def gemm(a, lda: int, bt, ldbt: int, m: int, n: int, k: int, dtype: DType, numeric: int,
         scheme: Scheme = Scheme.UNPROTECTED, out=None, ldc: int = 0, out_kind: Optional[str] = "f32",
         relu: bool = False, thread_m: int = 16, thread_n: int = 8, m_ext: int = 0, n_ext: int = 0,
         tol_k: int = 0, faults=None, nfaults: int = 0, out_sum=None, next_colck=None, verdicts=None,
         fired_count=None, fired=None, fired_cap: int = 0, ck_split: bool = False, tile_n: int = 0,
         num_sms: int = 0, ck_rows=None, plan_only: bool = False):
    """Enqueue one protected GEMM (or, with plan_only, return the kernel plan dict)."""
    args = _lib.GemmArgs()
    args.A, args.lda = a.data_ptr(), lda
    args.Bt, args.ldbt = bt.data_ptr(), ldbt
    args.C, args.ldc = (out.data_ptr() if out is not None else None), (ldc or n)
    args.M, args.N, args.K = m, n, k
    args.m_ext, args.n_ext, args.tol_k = m_ext or m, n_ext or n, tol_k or k
    args.dtype, args.out_dtype, args.numeric = storage_code(dtype), OUT_CODES[out_kind], numeric
    args.scheme = SCHEME_CODE[scheme]
    args.thread_m, args.thread_n = thread_m, thread_n
    args.relu, args.ck_split = int(relu), int(ck_split)
    args.faults, args.nfaults = (faults.data_ptr() if faults is not None else None), nfaults
    args.out_sum = out_sum.data_ptr() if out_sum is not None else None
    args.next_colck = next_colck.data_ptr() if next_colck is not None else None
    args.verdicts = verdicts.data_ptr() if verdicts is not None else None
    args.fired_count = fired_count.data_ptr() if fired_count is not None else None
    args.fired = fired.data_ptr() if fired is not None else None
    args.fired_cap = fired_cap
    args.tile_n, args.num_sms = tile_n, num_sms
    if ck_rows is not None:
        args.ck_rows, args.ldck, args.ck_rows_n = ck_rows.data_ptr(), ck_rows.stride(0), ck_rows.shape[0]
    if plan_only:
        out = (ctypes.c_int32 * 8)()
        _lib.check(_lib.load().abft_gemm_plan(ctypes.byref(args), out))
        return dict(tile_n=out[0], bn_eff=out[1], groups=out[2], nck_pad=out[3], stages=out[4],
                    ck_offline_recommended=bool(out[5]), n_blocks=out[6], grid=out[7])
    _lib.check(_lib.load().abft_gemm(ctypes.byref(args), stream_handle()))
    return None


def ck_rows(bt, n: int, k: int, dtype: DType, plan: dict, thread_n: int, split: bool):
    """Offline checksum rows of a K-major weight for one kernel plan (abft_ck_rows)."""
    t = torch()
    rows = plan["n_blocks"] * plan["nck_pad"]
    out = t.empty((rows, bt.shape[1]), dtype=bt.dtype, device="cuda")
    _lib.call("abft_ck_rows", ptr(bt), n, k, bt.stride(0), storage_code(dtype), plan["bn_eff"], thread_n,
              int(split), plan["nck_pad"], plan["n_blocks"], ptr(out), out.stride(0), stream_handle())
    return out


def colsum(x, rows: int, cols: int, ldx: int, dtype: DType, out, accumulate: bool = False) -> None:
    _lib.call("abft_colsum", ptr(x), rows, cols, ldx, storage_code(dtype), ptr(out), int(accumulate),
              stream_handle())


def matrix_sum(x, out) -> None:
    t = torch()
    elem = {t.float16: 0, t.bfloat16: 1, t.float32: 2}[x.dtype]
    _lib.call("abft_matrix_sum", ptr(x), x.shape[0], x.shape[1], x.stride(0), elem, ptr(out), stream_handle())


def global_tasks(tasks):
    """[(colck, rowck, rhs_tensor_or_None, k)] -> device array of abft_global_task_t."""
    t = torch()
    arr = (_lib.GlobalTask * len(tasks))()
    for i, (ca, rb, rhs, k) in enumerate(tasks):
        arr[i].colck, arr[i].rowck = ca.data_ptr(), rb.data_ptr()
        arr[i].rhs = rhs.data_ptr() if rhs is not None else None
        arr[i].k, arr[i].pad = k, 0
    host = t.frombuffer(bytearray(bytes(arr)), dtype=t.uint8)
    return host.to("cuda")


def global_lhs(tasks_dev, ntasks: int, sums) -> None:
    _lib.call("abft_global_lhs", ptr(tasks_dev), ntasks, ptr(sums), stream_handle())


def global_verify(tasks_dev, ntasks: int, numeric: int, sums, out=None, detected_count=None) -> None:
    _lib.call("abft_global_verify", ptr(tasks_dev), ntasks, numeric, ptr(sums), ptr(out), ptr(detected_count),
              stream_handle())


def verify_sums(sums, ks_dev, ntasks: int, numeric: int, out=None, detected_count=None) -> None:
    _lib.call("abft_verify_sums", ptr(sums), ptr(ks_dev), ntasks, numeric, ptr(out), ptr(detected_count),
              stream_handle())


def zero(t) -> None:
    """cudaMemsetAsync of a whole (contiguous) tensor on the current stream."""
    _lib.call("abft_zero", ptr(t), t.numel() * t.element_size(), stream_handle())
