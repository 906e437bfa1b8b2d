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


def _gemm_args(a, lda: int, bt, ldbt: int, m: int, n: int, k: int, dtype: DType, numeric: int,
               scheme: Scheme = Scheme.UNPROTECTED, out=None, ldc: int = 0, out_kind: Optional[str] = "f32",
               relu: bool = False, thread_m: int = 16, thread_n: int = 8, m_ext: int = 0, n_ext: int = 0,
               tol_k: int = 0, faults=None, nfaults: int = 0, out_sum=None, next_colck=None, verdicts=None,
               fired_count=None, fired=None, fired_cap: int = 0, ck_split: bool = False, tile_n: int = 0,
               num_sms: int = 0, ck_rows=None, a_colck=None, out_lhs=None, verify=None, pdl: bool = False,
               ck_layout: int = None, lhs_rowck=None, out_partials=None, bias=None, residual=None,
               ld_res: int = 0, plan_flags: int = 0, wsum=None, ws_ld: int = 0, ws_mode: int = 0, ws_P: int = 0,
               ws_Q: int = 0):
    args = _lib.GemmArgs()
    args.A, args.lda = a.data_ptr(), lda
    args.Bt, args.ldbt = (bt.data_ptr() if bt is not None else 16), ldbt
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
    if ck_layout is not None:
        args.ck_layout = int(ck_layout)
    elif ck_rows is not None:
        args.ck_layout = int(getattr(ck_rows, "_abft_aug", 0))
    args.a_colck = a_colck.data_ptr() if a_colck is not None else None
    args.out_lhs = out_lhs.data_ptr() if out_lhs is not None else None
    args.lhs_rowck = lhs_rowck.data_ptr() if lhs_rowck is not None else None
    if out_partials is not None:     # [cap, 2] fp64 per-CTA (lhs, rhs) slots
        t = torch()
        if out_partials.dtype != t.float64 or not out_partials.is_contiguous() or out_partials.dim() != 2 \
                or out_partials.shape[1] != 2:
            raise ValueError("out_partials must be a contiguous float64 [cap, 2] tensor")
        if out_sum is not None or out_lhs is not None:
            raise ValueError("out_partials replaces out_sum / out_lhs; pass one or the other")
        args.out_partials, args.partials_cap = out_partials.data_ptr(), out_partials.shape[0]
    if bias is not None:             # [>= N] fp32 per-column bias (BN folded)
        if bias.dtype != torch().float32 or not bias.is_contiguous():
            raise ValueError("bias must be a contiguous float32 tensor")
        args.bias = bias.data_ptr()
    if residual is not None:         # [M x N] storage-dtype shortcut, added before the ReLU
        args.residual, args.ld_res = residual.data_ptr(), (ld_res or residual.stride(0))
    args.plan_flags = int(plan_flags)
    if wsum is not None:             # fp32 [buckets][ws_ld] window sums of this layer's stored output
        if wsum.dtype != torch().float32 or not wsum.is_contiguous():
            raise ValueError("wsum must be a contiguous float32 tensor")
        args.wsum, args.ws_ld, args.ws_mode, args.ws_P, args.ws_Q = wsum.data_ptr(), ws_ld, ws_mode, ws_P, ws_Q
    args.pdl = int(pdl)
    vt = ()
    if verify is not None:
        # fused deferred verification in the launch's last CTA: (sums [n][2], ks [n], done, out, count)
        vsums, vks, vdone, vout, vdet = verify
        args.vsums, args.vk, args.vn = vsums.data_ptr(), vks.data_ptr(), vks.numel()
        args.vdone, args.vout = vdone.data_ptr(), vout.data_ptr()
        args.vdetected = vdet.data_ptr() if vdet is not None else None
        vt = (vsums, vks, vdone, vout, vdet)
    # the struct holds raw device pointers: keep every tensor it points to alive with it
    args._keep = [x for x in (a, bt, out, faults, out_sum, next_colck, verdicts, fired_count, fired, ck_rows,
                              a_colck, out_lhs, lhs_rowck, out_partials, bias, residual, wsum) + vt
                  if x is not None]
    return args


def gemm(a, lda: int, bt, ldbt: int, m: int, n: int, k: int, dtype: DType, numeric: int,
         scheme: Scheme = Scheme.UNPROTECTED, plan_only: bool = False, **kw):
    """Enqueue one protected GEMM (or, with plan_only, return the kernel plan dict).

    Keyword arguments are the fields of abft_gemm_args_t (see _gemm_args)."""
    args = _gemm_args(a, lda, bt, ldbt, m, n, k, dtype, numeric, scheme, **kw)
    if plan_only:
        out = (ctypes.c_int32 * 10)()
        _lib.check(_lib.load().abft_gemm_plan(ctypes.byref(args), out))
        return dict(tile_n=out[0], bn_eff=out[1], groups=out[2], nck_pad=out[3], stages=out[4],
                    ck_offline_recommended=bool(out[5]), n_blocks=out[6], grid=out[7], aug_rows=out[8])
    _lib.check(_lib.load().abft_gemm(ctypes.byref(args), stream_handle()))
    return None


def conv_args(x, geom: dict, bt, oc: int, dtype: DType, numeric: int, scheme: Scheme = Scheme.UNPROTECTED,
              workspace=None, **kw):
    """abft_conv_args_t for an NHWC input x [n, h, w, c] and packed weights bt [OC x K].

    geom: n, h, w, c, r, s, stride_h, stride_w, pad_h, pad_w (+ c_real, the model's channels)."""
    g = _gemm_args(x, geom["c"], bt, bt.stride(0) if bt is not None else 8, 0, oc, 0, dtype, numeric, scheme, **kw)
    args = _lib.ConvArgs()
    args.gemm = g
    for f in ("n", "h", "w", "c", "r", "s", "stride_h", "stride_w", "pad_h", "pad_w"):
        setattr(args, f, int(geom[f]))
    args.c_real = int(geom.get("c_real", 0))
    if workspace is not None:
        args.workspace, args.ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    args._keep = g._keep + [x] + ([workspace] if workspace is not None else [])
    return args


def conv_plan(args) -> dict:
    """abft_conv_plan: A-load mode, packed-weight channel stride ck and K, P, Q, M, workspace bytes."""
    out = (ctypes.c_int32 * 8)()
    _lib.check(_lib.load().abft_conv_plan(ctypes.byref(args), out))
    return dict(a_mode=out[0], ck=out[1], p=out[2], q=out[3], k=out[4], m=out[5], ws=out[6])


def conv_gemm_plan(args) -> dict:
    """abft_conv_gemm_plan: the conv kernel's tile plan (abft_gemm_plan's fields + a_mode) — the
    plan augmented weights / checksum rows of a conv call are built for."""
    out = (ctypes.c_int32 * 10)()
    _lib.check(_lib.load().abft_conv_gemm_plan(ctypes.byref(args), out))
    return dict(tile_n=out[0], bn_eff=out[1], groups=out[2], nck_pad=out[3], stages=out[4],
                ck_offline_recommended=bool(out[5]), n_blocks=out[6], grid=out[7], aug_rows=out[8], a_mode=out[9])


def conv2d(args) -> None:
    """Enqueue one protected implicit-GEMM convolution (abft_conv2d)."""
    _lib.check(_lib.load().abft_conv2d(ctypes.byref(args), stream_handle()))


def conv_pack_weight(w, ck: int, k_pitch: int = 0):
    """torch-layout weight [OC, cin, r, s] (CUDA fp16/bf16) -> packed K-major [OC, k_pitch]."""
    t = torch()
    oc, cin, r, s = (int(v) for v in w.shape)
    w = w.contiguous()
    k_pitch = k_pitch or -(-(r * s * ck) // 8) * 8
    out = t.empty((oc, k_pitch), dtype=w.dtype, device="cuda")
    _lib.call("abft_conv_pack_weight", ptr(w), oc, cin, r, s, ck, ptr(out), k_pitch, stream_handle())
    return out


def conv_colck(x, geom: dict, dtype: DType, out, accumulate: bool = False) -> None:
    """Windowed activation checksum of the conv's im2col matrix -> out [r*s*c] fp32."""
    _lib.call("abft_conv_colck", ptr(x), geom["n"], geom["h"], geom["w"], geom["c"], geom["r"], geom["s"],
              geom["stride_h"], geom["stride_w"], geom["pad_h"], geom["pad_w"], storage_code(dtype), ptr(out),
              int(accumulate), stream_handle())


def ck_rows(bt, n: int, k: int, dtype: DType, plan: dict, thread_n: int, split: bool):
    """Offline checksum rows of a K-major weight for one kernel plan (abft_ck_rows)."""
    t = torch()
    rows = plan["n_blocks"] * plan["nck_pad"]
    out = t.empty((rows, bt.shape[1]), dtype=bt.dtype, device="cuda")
    _lib.call("abft_ck_rows", ptr(bt), n, k, bt.stride(0), storage_code(dtype), plan["bn_eff"], thread_n,
              int(split), plan["nck_pad"], plan["n_blocks"], ptr(out), out.stride(0), stream_handle())
    return out


def aug_weights(bt, n: int, k: int, dtype: DType, plan: dict, thread_n: int, split: bool):
    """Augmented weights of a plan (ck_layout 1): each CTA N-tile's weight rows followed by its
    checksum rows, so the tile's outputs and checksums come from one MMA instruction."""
    t = torch()
    groups = plan["bn_eff"] // thread_n
    blk = plan["tile_n"] + groups * (2 if split else 1)
    out = t.empty((plan["n_blocks"] * blk, bt.shape[1]), dtype=bt.dtype, device="cuda")
    _lib.call("abft_aug_weights", ptr(bt), n, k, bt.stride(0), storage_code(dtype), plan["tile_n"], plan["bn_eff"],
              thread_n, int(split), plan["nck_pad"], plan["n_blocks"], ptr(out), out.stride(0), stream_handle())
    out._abft_aug = 1
    return out


def global_ck_rows(bt, n: int, k: int, dtype: DType, plan: dict, augmented: bool = True):
    """Checksum rows of the global scheme's lhs slice: per CTA N-tile, the hi/lo split of the
    tile's weight row sums (nt = bn_eff), for the plan of an out_lhs call — appended to the
    weight tiles (default) or as separate rows (abft_ck_rows)."""
    if augmented:
        return aug_weights(bt, n, k, dtype, plan, plan["bn_eff"], True)
    return ck_rows(bt, n, k, dtype, plan, plan["bn_eff"], True)


def colsum(x, rows: int, cols: int, ldx: int, dtype: DType, out, accumulate: bool = False) -> None:
    _lib.call("abft_colsum", ptr(x), rows, cols, ldx, storage_code(dtype), ptr(out), int(accumulate),
              stream_handle())


def weight_rowck(bt, n: int, k: int, dtype: DType):
    """rowck(B) fp32: column sums of B^T [n x k] (checksum.py:99-105), zero-padded to whole
    64-column k-blocks — the global scheme's lhs_rowck."""
    out = torch().zeros(-(-bt.stride(0) // 64) * 64, dtype=torch().float32, device="cuda")
    colsum(bt, n, bt.stride(0), bt.stride(0), dtype, out)
    return out


def matrix_sum(x, out) -> None:
    t = torch()
    elem = {t.float16: 0, t.bfloat16: 1, t.float32: 2}[x.dtype]
    _lib.call("abft_matrix_sum", ptr(x), x.shape[0], x.shape[1], x.stride(0), elem, ptr(out), stream_handle())


def global_tasks(tasks):
    """[(colck, rowck, rhs_tensor_or_None, k[, tol_k])] -> device array of abft_global_task_t."""
    t = torch()
    arr = (_lib.GlobalTask * len(tasks))()
    for i, task in enumerate(tasks):
        ca, rb, rhs, k = task[:4]
        arr[i].colck, arr[i].rowck = ca.data_ptr(), rb.data_ptr()
        arr[i].rhs = rhs.data_ptr() if rhs is not None else None
        arr[i].k, arr[i].tol_k = k, (task[4] if len(task) > 4 else 0)
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


def verify_partials(partials, ks_dev, ntasks: int, numeric: int, out=None, detected_count=None) -> None:
    """abft_verify_partials: partials [n, cap, 2] fp64 per-CTA (lhs, rhs) slots -> verdicts."""
    _lib.call("abft_verify_partials", ptr(partials), partials.shape[1], ptr(ks_dev), ntasks, numeric, ptr(out),
              ptr(detected_count), stream_handle())


def zero(t) -> None:
    """cudaMemsetAsync of a whole (contiguous) tensor on the current stream."""
    _lib.call("abft_zero", ptr(t), t.numel() * t.element_size(), stream_handle())


# ---------------------------------------------------------------- CNN glue (abft_glue.cu)
def maxpool_nhwc(x, n: int, h: int, w: int, c: int, ldx: int, k: int, stride: int, pad: int, ceil_mode: bool,
                 dtype: DType, out, ldo: int) -> None:
    _lib.call("abft_nhwc_maxpool", ptr(x), n, h, w, c, ctypes.c_int64(ldx), k, stride, pad, int(ceil_mode),
              storage_code(dtype), ptr(out), ctypes.c_int64(ldo), stream_handle())


def maxpool_nhwc_ws(x, n: int, h: int, w: int, c: int, ldx: int, k: int, stride: int, pad: int, ceil_mode: bool,
                    dtype: DType, out, ldo: int, wsum, ws_ld: int, ws_mode: int) -> None:
    """Max pooling that also accumulates the window column sums of its output (the next layer's
    fused global lhs)."""
    _lib.call("abft_nhwc_maxpool_ws", ptr(x), n, h, w, c, ctypes.c_int64(ldx), k, stride, pad, int(ceil_mode),
              storage_code(dtype), ptr(out), ctypes.c_int64(ldo), ptr(wsum), int(ws_ld), int(ws_mode),
              stream_handle())


def avgpool_nhwc(x, n: int, hw: int, c: int, ldx: int, dtype: DType, out, ldo: int) -> None:
    _lib.call("abft_nhwc_avgpool", ptr(x), n, hw, c, ctypes.c_int64(ldx), storage_code(dtype), ptr(out),
              ctypes.c_int64(ldo), stream_handle())


def interleave2(x1, ld1: int, b, ld2: int, pixels: int, half: int, out, ldo: int, half_pad: int,
                dtype: DType) -> None:
    _lib.call("abft_nhwc_interleave2", ptr(x1), ctypes.c_int64(ld1), ptr(b), ctypes.c_int64(ld2),
              ctypes.c_int64(pixels), half, ptr(out), ctypes.c_int64(ldo), half_pad, storage_code(dtype),
              stream_handle())


def sum_partials(partials, ntasks: int, sums) -> None:
    """[n, cap, 2] per-CTA (lhs, rhs) slots -> sums [n, 2] fp64 (one launch)."""
    _lib.call("abft_sum_partials", ptr(partials), partials.shape[1], ntasks, ptr(sums), stream_handle())


def border_sums(x, n: int, h: int, w: int, c: int, ldx: int, dtype: DType, wsum, ws_ld: int) -> None:
    """abft_nhwc_border_sums: buckets 1..8 of a 3x3 consumer's window sums from the border pixels."""
    _lib.call("abft_nhwc_border_sums", ptr(x), n, h, w, c, ctypes.c_int64(ldx), storage_code(dtype), ptr(wsum),
              int(ws_ld), stream_handle())


def window_lhs(wsum, ws_ld: int, c: int, r: int, s: int, ck: int, rowck, bias, n_out: int, m: int, lhs) -> None:
    """abft_window_lhs: lhs[0] += colck_im2col(A) . rowck(B) (+ m * sum(bias)) from a producer's
    window sums (fp32 [buckets][ws_ld]); rowck fp32 in the packed (r, s, ck) K order."""
    _lib.call("abft_window_lhs", ptr(wsum), int(ws_ld), int(c), int(r), int(s), int(ck), ptr(rowck),
              ptr(bias) if bias is not None else None, int(n_out), ctypes.c_int64(int(m)), ptr(lhs), stream_handle())


class FusedLhsBatch:
    """Every producer's border buckets and every fused consumer's window lhs of a forward as two
    launches (abft_fused_lhs_batch_*): the table is written once, launch() is graph-capturable."""

    def __init__(self, border, window, dtype: DType):
        import torch
        nb, nw = len(border), len(window)
        bt = (_lib.BorderTask * max(nb, 1))()
        for i, (x, n, h, w, c, ldx, wsum, ws_ld) in enumerate(border):
            bt[i] = _lib.BorderTask(ptr(x), ptr(wsum), int(ldx), int(n), int(h), int(w), int(c), int(ws_ld))
        wt = (_lib.WindowTask * max(nw, 1))()
        for i, (wsum, ws_ld, c, r, s, ck, rowck, bias, n_out, m, lhs) in enumerate(window):
            wt[i] = _lib.WindowTask(ptr(wsum), ptr(rowck), ptr(bias) if bias is not None else None, ptr(lhs),
                                    int(m), int(ws_ld), int(c), int(r), int(s), int(ck), int(n_out))
        nbytes = int(_lib.load().abft_fused_lhs_batch_bytes(nb, nw))
        self.table = torch.empty(-(-nbytes // 16) * 16, dtype=torch.uint8, device="cuda")
        self.grids = (ctypes.c_int32 * 2)()
        _lib.check(_lib.load().abft_fused_lhs_batch_prepare(bt, nb, wt, nw, ctypes.c_void_p(self.table.data_ptr()),
                                                            ctypes.c_int64(self.table.numel()), self.grids))
        self.dtype = storage_code(dtype)
        self._keep = (border, window)
        self.empty = nb == 0 and nw == 0

    def launch(self) -> None:
        if not self.empty:
            _lib.check(_lib.load().abft_fused_lhs_batch_launch(ctypes.c_void_p(self.table.data_ptr()), self.grids,
                                                               self.dtype, stream_handle()))


def group_problem_bytes() -> int:
    return int(_lib.load().abft_group_problem_bytes())


def gemm_group_prepare(args_list, table) -> None:
    """abft_gemm_group_prepare: write the problem table of a grouped launch (synchronous)."""
    arr = (_lib.GemmArgs * len(args_list))(*args_list)
    _lib.check(_lib.load().abft_gemm_group_prepare(arr, len(args_list), ctypes.c_void_p(table.data_ptr()),
                                                   ctypes.c_int64(table.numel() * table.element_size())))


def gemm_group_launch(args_arr, count: int, table) -> None:
    """abft_gemm_group_launch over a prepared table (stream-ordered, graph-capturable); args_arr is the
    ctypes array built once by the caller."""
    _lib.check(_lib.load().abft_gemm_group_launch(args_arr, count, ctypes.c_void_p(table.data_ptr()),
                                                  stream_handle()))

