"""Protected convolution layer on B200 — the conv half of "the protected linear/conv layer call".

The reference models convolutions only through their GEMM lowering (shapes.py:156-180,
``layer_to_gemm``: M = n*P*Q output pixels, N = OC, K = C*R*S) and checks them with the
same ``execute`` / ``global_abft_check`` as any GEMM.  ``conv2d`` keeps exactly that
contract — same schemes, tiling meaning, fault coordinates (row = output pixel index
(n*P + p)*Q + q, col = output channel), verdict ordering and report type as ``execute``
on the im2col matrix — but never builds the im2col matrix: the sm_100a kernel reads the
NHWC activation through a TMA im2col map (implicit GEMM).  The global scheme's lhs
colck(A) . rowck(B) is regrouped as 1^T (A (B 1)): one extra MMA N-slice against the
weight tile's row sums, summed over rows in the same kernel, so the im2col matrix's
column checksum is never needed (the standalone windowed pass ``abft_conv_colck`` is kept
as the alternative and cross-check).

K ordering is (r, s, c); input channels are zero-padded to a multiple of 8
(the reference's x8 padding rule, shapes.py:187-195, also the TMA 16-byte pitch rule).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import device as D
from . import kernels
from .errors import ShapeMismatchError
from .schemes import THREAD_LEVEL_SCHEMES, FaultSpec, Scheme, TilingConfig, fault_cell, validate_faults
from .shapes import DType, GemmShape


def _up(x: int, q: int) -> int:
    return -(-x // q) * q


@dataclass
class PreparedConv:
    """A conv weight in the kernel layout plus its offline row checksum (checksum.py:175-187)."""

    bt: object          # [OC x K] K-major, element (r, s, c) at (r*S + s)*ck + c
    rowck: object       # [K] fp32
    oc: int
    cin: int            # the model's input channels (K = cin*r*s in the reference lowering)
    ck: int             # channel stride of the packed weight (plan out[1])
    r: int
    s: int
    dtype: DType


def geometry(x_dev, r: int, s: int, stride, padding, cin: int) -> dict:
    sh, sw = (stride, stride) if np.isscalar(stride) else stride
    ph, pw = (padding, padding) if np.isscalar(padding) else padding
    n, h, w, c = (int(v) for v in x_dev.shape)
    if cin > c:
        raise ShapeMismatchError(f"weights have {cin} input channels, the activation only {c}")
    return dict(n=n, h=h, w=w, c=c, r=int(r), s=int(s), stride_h=int(sh), stride_w=int(sw), pad_h=int(ph),
                pad_w=int(pw), c_real=int(cin))


def plan(x_dev, geom: dict, oc: int, dtype: DType) -> dict:
    """abft_conv_plan for this input / geometry: A-load mode, packed-weight layout, workspace."""
    return kernels.conv_plan(kernels.conv_args(x_dev, geom, None, oc, dtype, D.numeric_code(dtype)))


def prepare_conv_weight(weight, dtype: DType, ck: int, k_pitch: int) -> PreparedConv:
    """torch-layout weight [OC, C, R, S] (numpy or torch) -> PreparedConv with the plan's layout."""
    t = D.torch()
    if len(tuple(weight.shape)) != 4:
        raise ShapeMismatchError(f"conv weight must be [OC, C, R, S], got {tuple(weight.shape)}")
    oc, cin, r, s = (int(v) for v in weight.shape)
    sd = D.torch_storage_dtype(dtype)
    if D.is_torch(weight):
        w = weight.to(device="cuda", dtype=sd).contiguous()
    else:
        w = t.from_numpy(np.ascontiguousarray(np.asarray(weight).astype(np.float32))).to("cuda").to(sd)
    bt = kernels.conv_pack_weight(w, ck, k_pitch)
    rowck = t.zeros(-(-bt.shape[1] // 64) * 64, dtype=t.float32, device="cuda")     # k-block padded
    kernels.colsum(bt, oc, bt.shape[1], bt.stride(0), dtype, rowck)
    return PreparedConv(bt=bt, rowck=rowck, oc=oc, cin=cin, ck=ck, r=r, s=s, dtype=dtype)


def upload_nhwc(x, dtype: DType):
    """NHWC activation (numpy or torch) -> CUDA storage tensor with channels padded to x8."""
    t = D.torch()
    if len(tuple(x.shape)) != 4:
        raise ShapeMismatchError(f"conv input must be NHWC [n, h, w, c], got {tuple(x.shape)}")
    n, h, w, c = (int(v) for v in x.shape)
    sd = D.torch_storage_dtype(dtype)
    src = x.to(device="cuda", dtype=sd) if D.is_torch(x) else \
        t.from_numpy(np.ascontiguousarray(np.asarray(x).astype(np.float32))).to("cuda").to(sd)
    c8 = D.round8(c)
    if c8 == c and src.is_contiguous():
        return src
    out = t.zeros((n, h, w, c8), dtype=sd, device="cuda")
    out[..., :c] = src
    return out


def standalone_colck(x_dev, geom: dict, pl: dict, dtype: DType, out) -> None:
    """The layer's activation checksum by a separate pass over the input (abft_colsum for a
    pointwise conv, abft_conv_colck otherwise); layout = the packed weight's K (plan)."""
    t = D.torch()
    n, h, w, c = geom["n"], geom["h"], geom["w"], geom["c"]
    if pl["a_mode"] == 0:
        kernels.colsum(x_dev, n * h * w, c, c, dtype, out)
        return
    r, s = geom["r"], geom["s"]
    if pl["ck"] == c:
        kernels.conv_colck(x_dev, geom, dtype, out)
        return
    # repack the [(r, s, c)] windowed sums into the plan's (r, s, ck) layout
    tmp = t.empty(r * s * c, dtype=t.float32, device="cuda")
    kernels.conv_colck(x_dev, geom, dtype, tmp)
    out.zero_()
    cc = min(c, pl["ck"])
    out[: r * s * pl["ck"]].view(r * s, pl["ck"])[:, :cc] = tmp.view(r * s, c)[:, :cc]


def conv2d(x, weight, stride=1, padding=0, tiling: TilingConfig = TilingConfig(),
           scheme: Scheme = Scheme.UNPROTECTED, faults: Sequence[FaultSpec] = (), dtype: DType | None = None,
           colck_source: str = "fused", tile_n: int = 0, plan_flags: int = 0):
    """Protected NHWC convolution; returns the reference's ExecutionReport for the lowered GEMM.

    ``report.output`` is [n, P, Q, OC] fp32 (int64 in exact-int mode); ``report.shape`` is
    the reference lowering GemmShape(n*P*Q, OC, C*R*S).  Global scheme: lhs comes from the
    conv kernel's checksum N-slice, sum over rows of A . rowck(B tile) ("slice"), from the
    checksum warps' dot of the staged A tiles with rowck(B) ("dot"; the default "fused" is
    "slice"), or from colck(A) . rowck(B) with the windowed checksum of a standalone pass
    ("standalone").  ``plan_flags``: abft_gemm_args_t.plan_flags (kernel plan hints)."""
    from .checksum import Verdict
    from .tiled import _TV_DTYPE, ExecutionReport, _counts, _thread_verdicts

    D.require_device()
    t = D.torch()
    if dtype is None:
        dtype = D.dtype_of(x)
    if len(tuple(x.shape)) != 4 or len(tuple(weight.shape)) != 4 or int(x.shape[3]) != int(weight.shape[1]):
        raise ShapeMismatchError(f"conv operands do not conform: x {tuple(x.shape)}, weight {tuple(weight.shape)}")
    if dtype.is_exact:
        D.guard_exact(x, weight, int(weight.shape[1]) * int(weight.shape[2]) * int(weight.shape[3]))
    x_dev = upload_nhwc(x, dtype)
    oc, cin, kr, ks = (int(v) for v in weight.shape)
    geom = geometry(x_dev, kr, ks, stride, padding, cin)
    numeric = D.numeric_code(dtype)
    pl = plan(x_dev, geom, oc, dtype)
    pc = prepare_conv_weight(weight, dtype, pl["ck"], pl["k"])
    m, P, Q = pl["m"], pl["p"], pl["q"]
    k_ref = pc.cin * pc.r * pc.s
    shape = GemmShape(m=m, n=pc.oc, k=k_ref)
    validate_faults(faults, shape, tiling)
    padded = GemmShape(m=_up(m, tiling.tb_m), n=_up(pc.oc, tiling.tb_n), k=_up(k_ref, tiling.k_step))
    cells = [fault_cell(f, tiling) for f in faults]
    f_dev, nf = D.faults_tensor(cells)
    out = t.empty((m, pc.oc), dtype=t.float32, device="cuda")
    ws = t.empty(max(pl["ws"], 16), dtype=t.uint8, device="cuda") if pl["ws"] else None
    thread_level = scheme in THREAD_LEVEL_SCHEMES
    verdicts = None
    if thread_level:
        ntr, ntc = padded.m // tiling.thread_m, padded.n // tiling.thread_n
        verdicts = t.empty(ntr * ntc * _TV_DTYPE.itemsize, dtype=t.uint8, device="cuda")
    if colck_source not in ("fused", "slice", "dot", "standalone"):
        raise ValueError(f"colck_source must be 'fused', 'slice', 'dot' or 'standalone', got {colck_source!r}")
    glob = scheme is Scheme.GLOBAL_ABFT
    sums = t.zeros(2, dtype=t.float64, device="cuda") if glob else None       # [lhs, rhs]
    kw = dict(out=out, ldc=pc.oc, out_kind="f32", thread_m=tiling.thread_m, thread_n=tiling.thread_n,
              m_ext=padded.m, n_ext=padded.n, tol_k=padded.k, faults=f_dev, nfaults=nf,
              out_sum=sums[1:2] if glob else None, verdicts=verdicts, ck_split=not dtype.is_exact, tile_n=tile_n,
              plan_flags=plan_flags)
    colck = None
    if glob and colck_source == "fused":
        colck_source = "slice"
    if glob and colck_source == "dot":
        # lhs = sum over rows of A . rowck(B) by the checksum warps from the staged A tiles
        kw["out_lhs"], kw["lhs_rowck"] = sums[0:1], pc.rowck
    if glob and colck_source == "slice":
        # lhs from the kernel's checksum slice: sum over rows of A . rowck(B tile)
        kw["out_lhs"] = sums[0:1]
        gplan = kernels.conv_gemm_plan(kernels.conv_args(x_dev, geom, pc.bt, pc.oc, dtype, numeric, scheme,
                                                         workspace=ws, ck_layout=1, **kw))
        kw["ck_rows"] = kernels.global_ck_rows(pc.bt, pc.oc, pl["k"], dtype, gplan)
    if scheme in (Scheme.THREAD_ONE_SIDED, Scheme.THREAD_TWO_SIDED):
        # weights with each tile's checksum rows appended (one MMA per k-step)
        oplan = kernels.conv_gemm_plan(kernels.conv_args(x_dev, geom, pc.bt, pc.oc, dtype, numeric, scheme,
                                                         workspace=ws, ck_layout=1, **kw))
        kw["ck_rows"] = kernels.aug_weights(pc.bt, pc.oc, pl["k"], dtype, oplan, tiling.thread_n,
                                            not dtype.is_exact)
    kernels.conv2d(kernels.conv_args(x_dev, geom, pc.bt, pc.oc, dtype, numeric, scheme, workspace=ws, **kw))
    if glob:
        vbuf = t.empty(32, dtype=t.uint8, device="cuda")
        if colck_source == "standalone":
            # lhs = colck(A) . rowck(B) from a separate windowed pass over the input
            colck = t.zeros(pc.bt.shape[1], dtype=t.float32, device="cuda")
            standalone_colck(x_dev, geom, pl, dtype, colck)
            kernels.global_verify(kernels.global_tasks([(colck, pc.rowck, sums[1:2], pc.bt.shape[1], k_ref)]), 1,
                                  numeric, t.empty(2, dtype=t.float64, device="cuda"), out=vbuf)
        else:
            kernels.verify_sums(sums, t.tensor([k_ref], dtype=t.int32, device="cuda"), 1, numeric, out=vbuf)
        raw = vbuf.cpu().numpy().view(np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"),
                                                ("det", "<i4"), ("k", "<i4")]))[0]
        lhs, rhs = float(raw["lhs"]), float(raw["rhs"])
        if dtype.is_exact:
            lhs, rhs = int(round(lhs)), int(round(rhs))
        vtuple = (Verdict(detected=bool(raw["det"]), lhs=lhs, rhs=rhs, tolerance_used=float(raw["tol"])),)
    elif thread_level:
        vtuple = _thread_verdicts(verdicts.cpu().numpy(), dtype.is_exact)
    else:
        vtuple = ()
    output = out.view(geom["n"], P, Q, pc.oc)
    if dtype.is_exact:
        output = output.round().to(t.int64)
    return ExecutionReport(output=D.to_host_like(output, x), verdicts=vtuple,
                           detected=any(v.detected for v in vtuple),
                           op_counts=_counts(scheme, tiling, padded, shape), scheme=scheme, shape=shape,
                           padded_shape=padded)
