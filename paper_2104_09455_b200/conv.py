"""Protected convolution layer on B200 — the conv half of "the protected linear/conv layer call".

The reference models convolutions only through their GEMM lowering (shapes.py:156-180,
``layer_to_gemm``: M = n*P*Q output pixels, N = OC, K = C*R*S) and checks them with the
same ``execute`` / ``global_abft_check`` as any GEMM.  ``conv2d`` keeps exactly that
contract — same schemes, tiling meaning, fault coordinates (row = output pixel index
(n*P + p)*Q + q, col = output channel), verdict ordering and report type as ``execute``
on the im2col matrix — but never builds the im2col matrix: the sm_100a kernel reads the
NHWC activation through a TMA im2col map (implicit GEMM), and the global scheme's
activation checksum — the column sum of the im2col matrix — is accumulated by the same
kernel from the A tiles it stages (or by the standalone windowed pass ``abft_conv_colck``).

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

    bt: object          # [OC x r*s*ck] K-major
    rowck: object       # [r*s*ck] fp32
    oc: int
    cin: int            # the model's input channels (K = cin*r*s in the reference lowering)
    ck: int             # physical channels of the NHWC input (multiple of 8)
    r: int
    s: int
    dtype: DType


def prepare_conv_weight(weight, dtype: DType, ck: int | None = None) -> PreparedConv:
    """torch-layout weight [OC, C, R, S] (numpy or torch) -> PreparedConv on the device."""
    t = D.torch()
    if len(tuple(weight.shape)) != 4:
        raise ShapeMismatchError(f"conv weight must be [OC, C, R, S], got {tuple(weight.shape)}")
    oc, cin, r, s = (int(v) for v in weight.shape)
    ck = ck or D.round8(cin)
    if ck < cin or ck % 8:
        raise ShapeMismatchError(f"physical channels {ck} must cover {cin} and be a multiple of 8")
    sd = D.torch_storage_dtype(dtype)
    if D.is_torch(weight):
        w = weight.to(device="cuda", dtype=sd).contiguous()
    else:
        w = t.from_numpy(np.ascontiguousarray(np.asarray(weight).astype(np.float32))).to("cuda").to(sd)
    bt = kernels.conv_pack_weight(w, ck)
    rowck = t.empty(bt.shape[1], dtype=t.float32, device="cuda")
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


def geometry(x_dev, pc: PreparedConv, stride, padding) -> dict:
    sh, sw = (stride, stride) if np.isscalar(stride) else stride
    ph, pw = (padding, padding) if np.isscalar(padding) else padding
    n, h, w, c = (int(v) for v in x_dev.shape)
    if c != pc.ck:
        raise ShapeMismatchError(f"input has {c} physical channels, weights were packed for {pc.ck}")
    return dict(n=n, h=h, w=w, c=c, r=pc.r, s=pc.s, stride_h=int(sh), stride_w=int(sw), pad_h=int(ph),
                pad_w=int(pw))


def conv2d(x, weight, stride=1, padding=0, tiling: TilingConfig = TilingConfig(),
           scheme: Scheme = Scheme.UNPROTECTED, faults: Sequence[FaultSpec] = (), dtype: DType | None = None,
           colck_source: str = "fused"):
    """Protected NHWC convolution; returns the reference's ExecutionReport for the lowered GEMM.

    ``report.output`` is [n, P, Q, OC] fp32 (int64 in exact-int mode); ``report.shape`` is
    the reference lowering GemmShape(n*P*Q, OC, C*R*S).  Global scheme: the windowed
    activation checksum comes from the A tiles inside the conv kernel ("fused") or from the
    standalone pass over the input ("standalone", abft_conv_colck)."""
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
    pc = prepare_conv_weight(weight, dtype, ck=int(x_dev.shape[3]))
    geom = geometry(x_dev, pc, stride, padding)
    numeric = D.numeric_code(dtype)
    probe = kernels.conv_args(x_dev, geom, pc.bt, pc.oc, dtype, numeric)
    plan = kernels.conv_plan(probe)
    m, P, Q = plan["m"], plan["p"], plan["q"]
    k_ref = pc.cin * pc.r * pc.s
    shape = GemmShape(m=m, n=pc.oc, k=k_ref)
    validate_faults(faults, shape, tiling)
    padded = GemmShape(m=_up(m, tiling.tb_m), n=_up(pc.oc, tiling.tb_n), k=_up(k_ref, tiling.k_step))
    cells = [fault_cell(f, tiling) for f in faults]
    f_dev, nf = D.faults_tensor(cells)
    out = t.empty((m, pc.oc), dtype=t.float32, device="cuda")
    thread_level = scheme in THREAD_LEVEL_SCHEMES
    verdicts = None
    if thread_level:
        ntr, ntc = padded.m // tiling.thread_m, padded.n // tiling.thread_n
        verdicts = t.empty(ntr * ntc * _TV_DTYPE.itemsize, dtype=t.uint8, device="cuda")
    if colck_source not in ("fused", "standalone"):
        raise ValueError(f"colck_source must be 'fused' or 'standalone', got {colck_source!r}")
    out_sum = t.zeros(1, dtype=t.float64, device="cuda") if scheme is Scheme.GLOBAL_ABFT else None
    colck = t.zeros(pc.bt.shape[1], dtype=t.float32, device="cuda") if scheme is Scheme.GLOBAL_ABFT else None
    fused = colck if colck_source == "fused" else None
    args = kernels.conv_args(x_dev, geom, pc.bt, pc.oc, dtype, numeric, scheme, out=out, ldc=pc.oc, out_kind="f32",
                             thread_m=tiling.thread_m, thread_n=tiling.thread_n, m_ext=padded.m, n_ext=padded.n,
                             tol_k=padded.k, faults=f_dev, nfaults=nf, out_sum=out_sum, verdicts=verdicts,
                             ck_split=not dtype.is_exact, a_colck=fused)
    kernels.conv2d(args)
    if scheme is Scheme.GLOBAL_ABFT:
        if colck_source == "standalone":
            kernels.conv_colck(x_dev, geom, dtype, colck)
        sums = t.empty(2, dtype=t.float64, device="cuda")
        vbuf = t.empty(32, dtype=t.uint8, device="cuda")
        kernels.global_verify(kernels.global_tasks([(colck, pc.rowck, out_sum, pc.bt.shape[1], k_ref)]), 1,
                              numeric, sums, out=vbuf)
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
