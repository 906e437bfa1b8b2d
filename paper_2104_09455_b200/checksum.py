"""Global-ABFT checksum math on B200 — drop-in for the reference's checksum.py.

Every reduction runs in the C-ABI library: column / row checksums (abft_colsum,
vectorised and coalesced), the checksum dot product and the deferred verdict
(abft_global_lhs / abft_verify_sums, fp64), the output summation (fused in the
GEMM epilogue, or abft_matrix_sum standalone).  ``run_protected_pipeline``
(reference :198-237) runs the layer chain as one fused GEMM per layer — output
summation and the next layer's activation checksum in the epilogue — and one
batched verification at the end; the host synchronises once.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Mapping, Sequence

import numpy as np

from . import device as D
from . import kernels
from .errors import ShapeMismatchError
from .schemes import Scheme
from .shapes import BFLOAT16, BINARY16, BINARY32, DType, DTypeTag, EXACT_INT

R_BINARY16 = 2.0 ** -10
R_BINARY32 = 2.0 ** -23
R_BFLOAT16 = 2.0 ** -7


@dataclass(frozen=True)
class Verdict:
    detected: bool
    lhs: float
    rhs: float
    tolerance_used: float


def dtype_of(a) -> DType:
    return D.dtype_of(a)


def storage_array(values, dtype: DType) -> np.ndarray:
    """Host-side cast onto the mode's storage grid (checksum.py:55-62)."""
    a = np.asarray(values)
    if dtype.tag is DTypeTag.EXACT_INT:
        return a.astype(np.int64)
    if dtype.tag is DTypeTag.BINARY16:
        return a.astype(np.float16)
    return a.astype(np.float32)


def comparison_tolerance(dtype: DType, k: int, lhs: float, rhs: float) -> float:
    """tau = r * K * max(|lhs|, |rhs|, 1) (checksum.py:143-148)."""
    if dtype.tag is DTypeTag.EXACT_INT:
        return 0.0
    r = {DTypeTag.BINARY16: R_BINARY16, DTypeTag.BINARY32: R_BINARY32, DTypeTag.BFLOAT16: R_BFLOAT16}[dtype.tag]
    return r * k * max(abs(lhs), abs(rhs), 1.0)


def make_verdict(dtype: DType, k: int, lhs, rhs) -> Verdict:
    tol = comparison_tolerance(dtype, k, lhs, rhs)
    return Verdict(detected=bool(abs(lhs - rhs) > tol), lhs=lhs, rhs=rhs, tolerance_used=tol)


def _mode_for(x, dtype):
    mode = dtype or D.dtype_of(x)
    if mode.tag is DTypeTag.BINARY32:
        mode = BINARY16 if not D.is_torch(x) else mode
    return mode


def _finish_vector(vec, like, exact: bool):
    if exact:
        vec = vec.round().to(D.torch().int64)
    return D.to_host_like(vec, like)


def column_checksum(a, dtype: DType | None = None):
    """Per-column sums of A [M x K] -> [K] (checksum.py:90-96), on the GPU."""
    m, k = D.shape2d(a, "A")
    D.require_device()
    mode = dtype or D.dtype_of(a)
    if mode.is_exact:
        D.guard_exact(a)
        if m * max(D.max_abs(a), 1) >= D.FP32_INT_MAX:
            raise D.ExactOverflowError("column checksum may exceed the exact fp32 range")
    dev = D.upload(a, mode if not mode.tag is DTypeTag.BINARY32 else BINARY16, "A")
    out = D.colck_device(dev, m, mode if not mode.tag is DTypeTag.BINARY32 else BINARY16)[:k]
    return _finish_vector(out, a, mode.is_exact)


def row_checksum(b, dtype: DType | None = None):
    """Per-row sums of B [K x N] -> [K] (checksum.py:99-105), on the GPU."""
    k, n = D.shape2d(b, "B")
    D.require_device()
    mode = dtype or D.dtype_of(b)
    if mode.is_exact:
        D.guard_exact(b)
        if n * max(D.max_abs(b), 1) >= D.FP32_INT_MAX:
            raise D.ExactOverflowError("row checksum may exceed the exact fp32 range")
    smode = mode if mode.tag is not DTypeTag.BINARY32 else BINARY16
    pw = D.prepare_weight(b, smode)
    return _finish_vector(pw.rowck[:k], b, mode.is_exact)


def checksum_dot(ca, rb):
    """colck . rowck (checksum.py:108-117): fp64 on the GPU; int for integer inputs."""
    t = D.torch()
    ca_t = ca if D.is_torch(ca) else t.from_numpy(np.ascontiguousarray(np.ravel(np.asarray(ca))))
    rb_t = rb if D.is_torch(rb) else t.from_numpy(np.ascontiguousarray(np.ravel(np.asarray(rb))))
    ca_t, rb_t = ca_t.reshape(-1), rb_t.reshape(-1)
    if ca_t.shape != rb_t.shape:
        raise ShapeMismatchError(f"checksum lengths differ: {ca_t.shape[0]} vs {rb_t.shape[0]}")
    exact = not ca_t.is_floating_point() and not rb_t.is_floating_point()
    D.require_device()
    x = ca_t.to("cuda", t.float32).contiguous()
    y = rb_t.to("cuda", t.float32).contiguous()
    if exact and max(D.max_abs(ca_t), D.max_abs(rb_t)) >= D.FP32_INT_MAX:
        raise D.ExactOverflowError("checksum dot operands exceed the exact fp32 range")
    sums = t.zeros(2, dtype=t.float64, device="cuda")
    kernels.global_lhs(kernels.global_tasks([(x, y, None, x.shape[0])]), 1, sums)
    val = float(sums[0].item())
    return int(round(val)) if exact else val


def output_summation(c):
    """Sum of all entries of C (checksum.py:120-127), fp64 on the GPU."""
    D.shape2d(c, "C")
    D.require_device()
    t = D.torch()
    ct = c if D.is_torch(c) else t.from_numpy(np.ascontiguousarray(np.asarray(c)))
    exact = not ct.is_floating_point()
    if ct.dtype not in (t.float16, t.bfloat16, t.float32):
        ct = ct.to(t.float32)
    ct = ct.to("cuda").contiguous()
    out = t.zeros(1, dtype=t.float64, device="cuda")
    kernels.matrix_sum(ct, out)
    val = float(out.item())
    return int(round(val)) if exact else val


def accumulate_matmul(a, b):
    """A @ B with fp32 accumulation on the tensor cores (checksum.py:130-140)."""
    from .tiled import execute
    if len(np.shape(a)) != 2 or len(np.shape(b)) != 2 or np.shape(a)[1] != np.shape(b)[0]:
        raise ShapeMismatchError(f"A is {tuple(np.shape(a))} but B is {tuple(np.shape(b))}")
    return execute(a, b).output


def global_abft_check(a, b, c, dtype: DType | None = None) -> Verdict:
    """colck(A) . rowck(B) vs sum(C) (checksum.py:156-169), K = A's column count."""
    sa, sb, sc = D.shape2d(a, "A"), D.shape2d(b, "B"), D.shape2d(c, "C")
    if sa[1] != sb[0] or sc != (sa[0], sb[1]):
        raise ShapeMismatchError(f"non-conformable check: A {sa}, B {sb}, C {sc}")
    mode = dtype or D.dtype_of(a)
    lhs = checksum_dot(column_checksum(a, mode), row_checksum(b, mode))
    rhs = output_summation(c)
    return make_verdict(mode, sa[1], lhs, rhs)


# ---------------------------------------------- offline weight checksum cache
_weight_cache: dict = {}


def offline_weight_checksum(b):
    """Row checksum built once per weight and reused (identity-keyed, checksum.py:172-187)."""
    key = id(b)
    hit = _weight_cache.get(key)
    if hit is not None and hit[0] is b:
        return hit[1]
    ck = row_checksum(b)
    _weight_cache[key] = (b, ck)
    return ck


def clear_weight_checksum_cache() -> None:
    _weight_cache.clear()
    D.clear_prepared_cache()


def relu(x):
    return np.maximum(x, 0)


def run_protected_pipeline(a0, weights: Sequence, activation: Callable = relu, dtype: DType | None = None,
                           faults: Mapping[int, Sequence[tuple]] | None = None) -> list:
    """Global-ABFT layer chain with ReLU, deferred verdicts (checksum.py:198-237).

    Per layer one fused kernel: fp32 GEMM, faults into the raw accumulator,
    output summation (rhs), ReLU + rounding to storage, and lhs = colck(a) .
    rowck(w) regrouped as the row sum of the checksum column a . rowck(w tile)
    from one extra MMA N-slice.  Verification of all layers is one batched
    launch after the chain; the host reads the verdicts once.
    ReLU is fused into the store.  Any other activation (the reference accepts any callable on
    the accumulate-precision array, checksum.py:201, :235) is applied between the layers: the
    kernel stores the layer's fp32 result (checks unchanged), the callable maps it, and the
    result is rounded to storage for the next layer — one host round trip per layer.
    """
    fused = activation is relu
    m, k0 = D.shape2d(a0, "A0")
    D.require_device()
    mode = dtype or D.dtype_of(a0)
    faults = faults or {}
    t = D.torch()
    dims = [k0]
    for idx, w in enumerate(weights):
        kw, nw = D.shape2d(w, f"weights[{idx}]")
        if kw != dims[-1]:
            raise ShapeMismatchError(f"layer {idx}: activations are ({m}, {dims[-1]}) but weights are ({kw}, {nw})")
        dims.append(nw)
    if mode.is_exact:
        D.guard_exact(a0)
    act = D.upload(a0, mode, "A0")
    numeric = D.numeric_code(mode)
    nl = len(weights)
    if nl == 0:
        return []
    sums = t.zeros((nl, 2), dtype=t.float64, device="cuda")     # per layer (lhs, rhs)
    for idx, w in enumerate(weights):
        if mode.is_exact:
            D.guard_exact(w, act, dims[idx], f"layer {idx} accumulation")
        pw = D.prepared_weight_cached(w, mode)
        n = dims[idx + 1]
        nxt = t.empty((m, D.round8(n)), dtype=D.torch_storage_dtype(mode), device="cuda")
        if n % 8:
            nxt.zero_()
        raw = nxt if fused else t.zeros((m, D.round8(n)), dtype=t.float32, device="cuda")
        f_dev, nf = D.faults_tensor(list(faults.get(idx, ())))
        kind = ("bf16" if mode.tag is DTypeTag.BFLOAT16 else "f16") if fused else "f32"
        kw = dict(out=raw, ldc=raw.stride(0), out_kind=kind, relu=fused, faults=f_dev, nfaults=nf,
                  out_sum=sums[idx, 1:2], out_lhs=sums[idx, 0:1])
        plan = kernels.gemm(act, act.stride(0), pw.bt, pw.ldbt, m, n, dims[idx], mode, numeric, Scheme.GLOBAL_ABFT,
                            plan_only=True, ck_layout=1, **kw)
        ckr = kernels.global_ck_rows(pw.bt, n, dims[idx], mode, plan)
        kernels.gemm(act, act.stride(0), pw.bt, pw.ldbt, m, n, dims[idx], mode, numeric, Scheme.GLOBAL_ABFT,
                     ck_rows=ckr, **kw)
        if not fused:
            c = raw[:, :n].cpu().numpy()
            if mode.is_exact:
                c = np.rint(c).astype(np.int64)
            y = np.asarray(activation(c))
            if y.shape != c.shape:
                raise ShapeMismatchError(f"activation changed the layer {idx} output shape {c.shape} -> {y.shape}")
            nxt[:, :n].copy_(D.torch().from_numpy(np.ascontiguousarray(y.astype(np.float32))).to("cuda"))
        if mode.is_exact:
            # the next layer consumes these values exactly only inside the fp16 integer range
            if D.max_abs(nxt) > D.FP16_INT_MAX:
                raise D.ExactOverflowError(f"layer {idx} activations leave the exact fp16 range")
        act = nxt
    ks_dev = t.tensor(dims[:-1], dtype=t.int32, device="cuda")
    vbuf = t.empty(nl * 32, dtype=t.uint8, device="cuda")
    kernels.verify_sums(sums, ks_dev, nl, numeric, out=vbuf)
    raw = vbuf.cpu().numpy().view(np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"),
                                            ("det", "<i4"), ("k", "<i4")]))
    verdicts = []
    for r in raw:
        lhs, rhs = float(r["lhs"]), float(r["rhs"])
        if mode.is_exact:
            lhs, rhs = int(round(lhs)), int(round(rhs))
        verdicts.append(Verdict(detected=bool(r["det"]), lhs=lhs, rhs=rhs, tolerance_used=float(r["tol"])))
    return verdicts
