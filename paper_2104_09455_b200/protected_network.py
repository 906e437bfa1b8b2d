"""Whole-network protected inference (config C5): a torchvision CNN run end to end on B200
with every linear layer (conv / FC) protected by its own ABFT scheme.

The reference models a network only as its linear-layer list (shapes.py:198-212
``model_to_gemm_sequence``) and protects a chain of linear layers with deferred
verification (checksum.py:198-237 ``run_protected_pipeline``: per-layer colck / rowck /
output summation, one verdict pass at the end).  The paper measures a network's overhead
over its linear layers with per-layer scheme selection.
``ProtectedNetwork`` is that pipeline on a real CNN:

- BatchNorm folded into each conv's weight and a per-channel **bias**; the bias epilogue of
  the protected kernel keeps the checks exact (global lhs += M * sum(bias), one-sided group
  column += the group's bias sum — SURVEY H3), so the checked identity is the reference's.
- Residual shortcuts are added in the producing conv's epilogue (after the checks, before the
  ReLU); concatenation (SqueezeNet Fire, ShuffleNet units) writes channel slices of one
  buffer; pooling and ShuffleNet's channel shuffle are native NHWC glue kernels.
- Depthwise / grouped convolutions are treated as dense (block-diagonal weights), as the
  paper does (documents.py:111-112).
- Every global-ABFT layer writes per-CTA (lhs, rhs) partials; thread-level layers count fired
  tiles; ONE verification launch at the end forms every layer's verdict with the tau rule of
  checksum.py:143-153 (K = the model's unpadded C*R*S) — the deferred verification of
  checksum.py:207-211, :237.  All buffers are planned once; a forward is one stream of
  launches with no allocation and no host synchronisation, captured in one CUDA graph.
- Batch sharding: each rank runs batch/world; its per-layer partial sums and
  flag counters go out in ONE all-reduce at the end of the forward, then the verdicts are
  formed from the full-batch sums — exactly the single-GPU verdicts (lhs and rhs are linear
  in the rows; thread-level checks are row-local).

Activations are NHWC fp16/bf16 with channels padded to a multiple of 8 (the reference's
x8 padding rule, shapes.py:187-195); padding channels hold zeros.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import device as D
from . import kernels
from .checksum import Verdict
from .schemes import Scheme, TilingConfig
from .shapes import BINARY16, DType, GemmShape

SELECTABLE = (Scheme.UNPROTECTED, Scheme.GLOBAL_ABFT, Scheme.THREAD_ONE_SIDED)
GLOBAL_DOT = "global-dot"      # argument-set key of the global scheme with the checksum-warp lhs
# ... and with the lhs from the producer's fused window sums (abft_window_lhs): the kernel runs the
# output summation only (plan_flags bit 10)
GLOBAL_FUSED = "global-fused"
ARG_KEYS = SELECTABLE + (GLOBAL_DOT, GLOBAL_FUSED)
EXT_LHS = 1024
PAIR_FLAG = 4096   # plan_flags bit 12: CTA pairs (2-CTA clusters, M = 256 cta_group::2 MMAs)
_VERDICT_DTYPE = np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"), ("det", "<i4"), ("k", "<i4")])


def _r8(x: int) -> int:
    return -(-x // 8) * 8


# ------------------------------------------------------------------------------- tensors
@dataclass
class Act:
    """An NHWC activation: ``buf`` [n, h, w, cp] (a view; its pixel stride may exceed cp when it
    is a channel slice of a wider buffer), ``c`` logical channels living at physical channels
    ``phys`` (None = 0..c-1); every other physical channel holds zeros."""

    buf: object
    c: int
    phys: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return int(self.buf.shape[0])

    @property
    def h(self) -> int:
        return int(self.buf.shape[1])

    @property
    def w(self) -> int:
        return int(self.buf.shape[2])

    @property
    def cp(self) -> int:
        return int(self.buf.shape[3])

    @property
    def ld(self) -> int:
        return int(self.buf.stride(2))

    def phys_map(self) -> np.ndarray:
        return np.arange(self.c) if self.phys is None else self.phys

    def matrix(self):
        """[n*h*w, cp] view with row stride ld (the GEMM A operand of a pointwise conv / FC)."""
        return self.buf.as_strided((self.n * self.h * self.w, self.cp), (self.ld, 1))


# ------------------------------------------------------------------------------- linear layers
@dataclass
class LinearLayer:
    """One protected conv / FC layer: NHWC x -> out (+bias, +residual, ReLU)."""

    index: int
    name: str
    x: Act
    out: Act
    weight: object            # fp32 [oc, c_logical, r, s] (BN folded)
    bias: Optional[object]    # fp32 [oc] or None
    stride: int
    pad: int
    relu: bool
    residual: Optional[Act] = None
    kind: str = "conv"
    c_real: int = 0           # physical channels past which x is known zero (stem: 3 of 8)
    scheme: Scheme = Scheme.UNPROTECTED
    # built state
    gemm_path: bool = False
    k_ref: int = 0
    m: int = 0
    args: Dict = field(default_factory=dict)
    fault_args: Dict = field(default_factory=dict)
    tile_n: Dict = field(default_factory=dict)     # per-scheme CTA tile override (0 / absent: planner's)
    flags: Dict = field(default_factory=dict)      # per-scheme plan hints (abft_gemm_args_t.plan_flags)
    gvar: str = "slice"       # global-ABFT lhs: "slice" (checksum MMA N-slice), "dot" (checksum warps) or
                              # "fused" (the producer's window sums, when `producer` is set)
    producer: Optional["LinearLayer"] = None   # the layer whose stored output is exactly this layer's input
    ws_mode: int = 0          # as a producer: 0 none, 1 column sums, 2 3x3 window buckets (for fused consumers)
    ws_active: bool = False   # as a producer: a consumer currently takes its global lhs from our window sums

    @property
    def oc(self) -> int:
        return int(self.weight.shape[0])

    @property
    def r(self) -> int:
        return int(self.weight.shape[2])

    @property
    def s(self) -> int:
        return int(self.weight.shape[3])

    def gemm_shape(self) -> GemmShape:
        """The reference lowering (shapes.py:169-177): M = n*P*Q, N = OC, K = C*R*S."""
        return GemmShape(self.m, self.oc, self.k_ref)

    def flops(self) -> int:
        return 2 * self.m * self.oc * self.k_ref

    def bytes(self) -> int:
        """Algorithmic bytes of the implicit GEMM: input tensor + weights + output."""
        x = self.x
        return 2 * (x.n * x.h * x.w * x.c + self.k_ref * self.oc + self.m * self.oc)


@dataclass
class PoolProducer:
    """A max-pooling glue op as the producer of a fused consumer's window sums (the pooled output
    feeds a 1x1 or 3x3 / stride 1 / pad 1 conv directly)."""

    name: str
    out: Act
    ws_mode: int = 0
    ws_active: bool = False
    index: int = -1
    _wsum: object = None


@dataclass
class GlueOp:
    name: str
    fn: Callable[[], None]


# ------------------------------------------------------------------------------- the network
class ProtectedNetwork:
    """A torchvision CNN (eval mode) as a protected NHWC pipeline on the current CUDA device.

    model: torchvision ResNet / VGG / AlexNet / SqueezeNet / ShuffleNetV2 instance (weights on
    any device; BatchNorm statistics are folded).  batch, h, w: the input extent.  schemes:
    one Scheme for every layer, a per-layer list, or "ig" (set later by ``select_ig``)."""

    def __init__(self, model, batch: int, h: int = 224, w: int = 224, dtype: DType = BINARY16,
                 schemes=Scheme.UNPROTECTED, tiling: TilingConfig = TilingConfig(), ck_split: bool = True):
        D.require_device()
        t = D.torch()
        self.t = t
        self.dtype = dtype
        self.sd = D.torch_storage_dtype(dtype)
        self.numeric = D.numeric_code(dtype)
        self.tiling = tiling
        self.ck_split = ck_split
        self.batch, self.h, self.w = batch, h, w
        self.ops: List[object] = []          # LinearLayer | GlueOp in execution order
        self.layers: List[LinearLayer] = []
        self.pools: List[PoolProducer] = []   # max-pooling glue ops (window-sum producers)
        self.input = Act(t.zeros((batch, h, w, 8), dtype=self.sd, device="cuda"), 3)
        self.name = type(model).__name__.lower()
        model = model.eval()
        with t.no_grad():
            self.output = _build(self, model)
        nl = len(self.layers)
        self._find_fused_edges()
        # per-forward accumulators, ONE block cleared by one memset: per-CTA (lhs, rhs) slots of every
        # layer [nl][cap][2] fp64, the counters [fired thread tiles, flagged layers] int32, then the
        # producers' window-sum buckets [9][cp] fp32
        self.cap = max(1, D.sm_count())
        prods = list(self.layers) + self.pools
        ws_floats = [9 * P.out.cp if P.ws_mode else 0 for P in prods]
        base = 16 * self.cap * nl + 16
        self._block = t.zeros(base + 4 * sum(ws_floats), dtype=t.uint8, device="cuda")
        self.partials = self._block[:16 * self.cap * nl].view(t.float64).view(nl, self.cap, 2)
        self.counters = self._block[16 * self.cap * nl:16 * self.cap * nl + 8].view(t.int32)
        off = base
        for P, nf in zip(prods, ws_floats):
            P._wsum = self._block[off:off + 4 * nf].view(t.float32) if nf else None
            off += 4 * nf
        self.sums = t.zeros((nl, 2), dtype=t.float64, device="cuda")
        self.verdict_buf = t.zeros(nl * _VERDICT_DTYPE.itemsize, dtype=t.uint8, device="cuda")
        # the reduction vector of the sharded verification: [sums (2 nl) | fired | flagged]
        self.reduce_buf = t.zeros(2 * nl + 2, dtype=t.float64, device="cuda")
        for L in self.layers:
            self._build_layer(L)
        self.ks = t.tensor([L.k_ref for L in self.layers], dtype=t.int32, device="cuda")
        self.set_schemes(schemes)

    def _find_fused_edges(self) -> None:
        """Consumers whose input is exactly a producer layer's stored output (no glue in between, a
        dense NHWC buffer) and whose im2col column sums the producer's epilogue can accumulate:
        pointwise stride-1 layers (column sums) and 3x3 / stride 1 / pad 1 convs (window buckets)."""
        by_out = {id(L.out): L for L in self.layers}
        by_out.update({id(P.out): P for P in self.pools})
        for L in self.layers:
            P = by_out.get(id(L.x))
            if P is None or P.out.phys is not None or P.out.cp != int(P.out.buf.shape[3]) or L.kind != "conv":
                continue
            pointwise = (L.r, L.s, L.stride, L.pad) == (1, 1, 1, 0)
            window = (L.r, L.s, L.stride, L.pad) == (3, 3, 1, 1)
            # (smem buckets: the producer kernel's [9][N] / [N] fp32, the pool kernel's [9][C])
            if not (pointwise or window) or P.out.cp > (512 if window else 2048):
                continue
            L.producer = P
            P.ws_mode = max(P.ws_mode, 2 if window else 1)

    def producers(self):
        return [P for P in list(self.layers) + self.pools if P.ws_mode]

    def fused_consumers(self, P: LinearLayer):
        return [L for L in self.layers if L.producer is P]

    def _refresh_window_sums(self) -> None:
        """Producers accumulate window sums exactly while a consumer runs the fused global lhs."""
        for P in self.producers():
            active = any(C.scheme is Scheme.GLOBAL_ABFT and C.gvar == "fused" for C in self.fused_consumers(P))
            if active != P.ws_active:
                P.ws_active = active
                if isinstance(P, PoolProducer):
                    continue          # the pool's launch reads ws_active itself
                for key in ARG_KEYS:
                    if key in P.args:
                        P.args[key] = self._make_args(P, key)
                for key in list(P.fault_args):
                    P.fault_args[key] = self._make_args(P, key, faults=P._fault_keep)

    # ---------------------------------------------------------------- building blocks
    def new_act(self, n: int, h: int, w: int, c: int, cp: Optional[int] = None) -> Act:
        cp = cp or _r8(c)
        return Act(self.t.zeros((n, h, w, cp), dtype=self.sd, device="cuda"), c)

    def add_linear(self, name: str, x: Act, weight, bias, stride: int = 1, pad: int = 0, relu: bool = True,
                   residual: Optional[Act] = None, out: Optional[Act] = None, kind: str = "conv",
                   c_real: int = 0) -> Act:
        t = self.t
        weight = weight.detach().to(device="cuda", dtype=t.float32)
        if bias is not None:
            bias = bias.detach().to(device="cuda", dtype=t.float32)
        oc, cin, r, s = (int(v) for v in weight.shape)
        if cin != x.c:
            raise ValueError(f"{name}: weight has {cin} input channels, the activation {x.c}")
        P = (x.h + 2 * pad - r) // stride + 1
        Q = (x.w + 2 * pad - s) // stride + 1
        if out is None:
            out = self.new_act(x.n, P, Q, oc)
        if (out.n, out.h, out.w) != (x.n, P, Q) or out.cp < _r8(oc):
            raise ValueError(f"{name}: output buffer {tuple(out.buf.shape)} does not fit [{x.n},{P},{Q},{oc}]")
        L = LinearLayer(index=len(self.layers), name=name, x=x, out=out, weight=weight, bias=bias, stride=stride,
                        pad=pad, relu=relu, residual=residual, kind=kind, c_real=c_real)
        self.layers.append(L)
        self.ops.append(L)
        return out

    def add_glue(self, name: str, fn: Callable[[], None]) -> None:
        self.ops.append(GlueOp(name, fn))

    def maxpool(self, x: Act, k: int, stride: int, pad: int = 0, ceil_mode: bool = False) -> Act:
        def osz(n):
            num = n + 2 * pad - k
            o = (-(-num // stride) if ceil_mode else num // stride) + 1
            if ceil_mode and (o - 1) * stride >= n + pad:
                o -= 1
            return o
        out = Act(self.t.zeros((x.n, osz(x.h), osz(x.w), x.cp), dtype=self.sd, device="cuda"), x.c, x.phys)
        prod = PoolProducer("maxpool", out)
        self.pools.append(prod)

        def run():
            kernels.maxpool_nhwc(x.buf, x.n, x.h, x.w, x.cp, x.ld, k, stride, pad, ceil_mode, self.dtype, out.buf,
                                 out.ld)
            if prod.ws_active:
                # the consumer's column sums by one streaming pass over the pooled output (measured
                # cheaper than accumulating them inside the pooling kernel, abft_nhwc_maxpool_ws)
                kernels.colsum(out.buf, out.n * out.h * out.w, out.cp, out.ld, self.dtype, prod._wsum, accumulate=True)
        self.add_glue("maxpool", run)
        prod.run = run
        return out

    def avgpool(self, x: Act) -> Act:
        """Global average pooling -> [n, 1, 1, cp]."""
        out = Act(self.t.zeros((x.n, 1, 1, x.cp), dtype=self.sd, device="cuda"), x.c, x.phys)
        self.add_glue("avgpool", lambda: kernels.avgpool_nhwc(x.buf, x.n, x.h * x.w, x.cp, x.ld, self.dtype,
                                                              out.buf, out.ld))
        return out

    def shuffle_cat(self, x1: Act, b: Act) -> Act:
        """channel_shuffle(cat(x1, b), 2) in the halves layout (see abft_nhwc_interleave2)."""
        half = x1.c
        if b.c != half or x1.phys is not None or b.phys is not None:
            raise ValueError("shuffle_cat: two dense halves of equal width")
        hp = _r8(half)
        out = Act(self.t.zeros((x1.n, x1.h, x1.w, 2 * hp), dtype=self.sd, device="cuda"), 2 * half,
                  np.concatenate([np.arange(half), hp + np.arange(half)]))
        pixels = x1.n * x1.h * x1.w
        self.add_glue("shuffle", lambda: kernels.interleave2(x1.buf, x1.ld, b.buf, b.ld, pixels, half, out.buf,
                                                             out.ld, hp, self.dtype))
        return out

    # ---------------------------------------------------------------- per-layer kernel arguments
    def _build_layer(self, L: LinearLayer) -> None:
        t = self.t
        x = L.x
        oc8 = _r8(L.oc)
        # weights scattered onto the physical input channels (zeros elsewhere), output channels to oc8
        wp = t.zeros((oc8, x.cp, L.r, L.s), dtype=t.float32, device="cuda")
        idx = t.as_tensor(x.phys_map(), device="cuda", dtype=t.long)
        wp[:L.oc].index_copy_(1, idx, L.weight)
        bias = None
        if L.bias is not None:
            bias = t.zeros(oc8, dtype=t.float32, device="cuda")
            bias[:L.oc] = L.bias
        L.k_ref = x.c * L.r * L.s
        P, Q = L.out.h, L.out.w
        L.m = x.n * P * Q
        L.gemm_path = L.r == 1 and L.s == 1 and L.stride == 1 and L.pad == 0
        wq = wp.to(self.sd)
        L._bias_dev = bias
        rows_pad = -(-oc8 // 256) * 256     # packed weights carry zero rows to whole tiles (plan_flags bit 1)
        if L.gemm_path:
            L._a = x.matrix()
            L._bt_pad = t.zeros((rows_pad, x.cp), dtype=self.sd, device="cuda")
            L._bt_pad[:oc8] = wq.view(oc8, x.cp)
            L._bt = L._bt_pad[:oc8]
            L._k = x.cp
        else:
            if x.ld != x.cp:
                raise ValueError(f"{L.name}: a non-pointwise conv needs a dense NHWC input")
            from .conv import geometry
            L._geom = geometry(x.buf, L.r, L.s, (L.stride, L.stride), (L.pad, L.pad), x.cp)
            if L.c_real:
                L._geom["c_real"] = L.c_real
            pl = kernels.conv_plan(kernels.conv_args(x.buf, L._geom, None, oc8, self.dtype, self.numeric))
            L._ws = t.empty(max(pl["ws"], 16), dtype=t.uint8, device="cuda") if pl["ws"] else None
            if pl["ck"] < x.cp:
                # dense-K modes pack only the first ck physical channels (the rest of x is zero)
                if L.c_real > pl["ck"] or bool((wq[:, pl["ck"]:] != 0).any()):
                    raise ValueError(f"{L.name}: weights on channels past the packed {pl['ck']}")
                wq = wq[:, :pl["ck"]].contiguous()
            packed = kernels.conv_pack_weight(wq, pl["ck"], pl["k"])
            L._bt_pad = t.zeros((rows_pad, packed.shape[1]), dtype=self.sd, device="cuda")
            L._bt_pad[:oc8] = packed
            L._bt = L._bt_pad[:oc8]
            L._k = pl["k"]
        L._c = L.out.matrix()
        L._res = L.residual.matrix() if L.residual is not None else None
        # rowck(B) in the packed K layout, zero-padded to whole 64-column k-blocks: the "dot" lhs
        L._rowck = kernels.weight_rowck(L._bt, oc8, L._k, self.dtype)
        for key in self.keys_of(L):
            L.args[key] = self._make_args(L, key)

    @staticmethod
    def keys_of(L: LinearLayer):
        """The argument sets a layer has: every selectable scheme, the dot lhs, and the fused lhs when
        a producer's epilogue can supply its activation checksum."""
        return ARG_KEYS if L.producer is not None else tuple(k for k in ARG_KEYS if k != GLOBAL_FUSED)

    def _kw(self, L: LinearLayer, key, faults=None) -> dict:
        scheme = Scheme.GLOBAL_ABFT if key in (GLOBAL_DOT, GLOBAL_FUSED) else key
        tl = self.tiling
        kw = dict(out=L._c, ldc=L.out.ld, out_kind="bf16" if self.sd == self.t.bfloat16 else "f16", relu=L.relu,
                  bias=L._bias_dev, residual=L._res, ld_res=L.residual.ld if L.residual is not None else 0,
                  tile_n=L.tile_n.get(key, 0), plan_flags=L.flags.get(key, 0) | (EXT_LHS if key == GLOBAL_FUSED else 0))
        if L.ws_active:
            # the epilogue sums all rows only (bucket 0); a 3x3 consumer's border buckets come from
            # abft_nhwc_border_sums over the border pixels (cheaper than per-chunk border reductions)
            kw.update(wsum=L._wsum, ws_ld=L.out.cp, ws_mode=1, ws_P=L.out.h, ws_Q=L.out.w)
        if faults is not None:
            kw["faults"], kw["nfaults"] = faults
        if scheme is Scheme.GLOBAL_ABFT:
            kw["out_partials"] = self.partials[L.index]
            if key == GLOBAL_DOT:
                kw["lhs_rowck"] = L._rowck
        elif scheme is Scheme.THREAD_ONE_SIDED:
            oc8 = _r8(L.oc)
            kw.update(thread_m=tl.thread_m, thread_n=tl.thread_n, m_ext=-(-L.m // tl.thread_m) * tl.thread_m,
                      n_ext=-(-oc8 // tl.thread_n) * tl.thread_n, tol_k=-(-L.k_ref // tl.k_step) * tl.k_step,
                      fired_count=self.counters[0:1], ck_split=self.ck_split)
        return kw

    def _launch_args(self, L: LinearLayer, scheme: Scheme, kw: dict, ck_layout=None):
        oc8 = _r8(L.oc)
        if L.gemm_path:
            return ("gemm", (L._a, L.x.ld, L._bt, L._k, L.m, oc8, L._k, self.dtype, self.numeric, scheme),
                    dict(kw, ck_layout=ck_layout) if ck_layout is not None else kw)
        return ("conv", kernels.conv_args(L.x.buf, L._geom, L._bt, oc8, self.dtype, self.numeric, scheme,
                                          workspace=L._ws, **(dict(kw, ck_layout=ck_layout)
                                                              if ck_layout is not None else kw)), None)

    def _plan(self, L: LinearLayer, scheme: Scheme, kw: dict) -> dict:
        kind, a, k2 = self._launch_args(L, scheme, kw, ck_layout=1)
        if kind == "gemm":
            return kernels.gemm(*a, plan_only=True, **k2)
        return kernels.conv_gemm_plan(a)

    def _make_args(self, L: LinearLayer, key, faults=None):
        kw = self._kw(L, key, faults)
        scheme = Scheme.GLOBAL_ABFT if key in (GLOBAL_DOT, GLOBAL_FUSED) else key
        oc8 = _r8(L.oc)
        if key is Scheme.GLOBAL_ABFT:
            # augmented weights per plan (tile / N blocks): plan hints such as CTA pairs may pick
            # another tile than the default plan
            pl = self._plan(L, scheme, kw)
            cache = L.__dict__.setdefault("_gck_by_plan", {})
            ck_key = (pl["tile_n"], pl["aug_rows"], pl["n_blocks"], pl["nck_pad"])
            if ck_key not in cache:
                cache[ck_key] = kernels.global_ck_rows(L._bt, oc8, L._k, self.dtype, pl)
            kw["ck_rows"] = cache[ck_key]
        elif scheme is Scheme.THREAD_ONE_SIDED:
            if not hasattr(L, "_ock"):
                L._ock = kernels.aug_weights(L._bt, oc8, L._k, self.dtype, self._plan(L, scheme, kw),
                                             self.tiling.thread_n, self.ck_split)
            kw["ck_rows"] = L._ock
        kind, a, k2 = self._launch_args(L, scheme, kw)
        if kind == "gemm":
            return ("gemm", kernels._gemm_args(*a, **k2))
        return ("conv", a)

    def plan_of(self, L: LinearLayer, scheme: Scheme) -> dict:
        """The kernel plan (tile_n, stages, grid, ...) a layer launches with under `scheme`."""
        return self._plan(L, scheme, self._kw(L, scheme))

    def set_tile(self, L: LinearLayer, key, tile_n: int, flags: int = 0) -> None:
        """Force the CTA tile (0: the planner's choice) and plan hints of one layer's launch under
        `key` (a Scheme or GLOBAL_DOT)."""
        old = (L.tile_n.get(key, 0), L.flags.get(key, 0))
        L.tile_n[key], L.flags[key] = int(tile_n), int(flags)
        try:
            kind, a = self._make_args(L, key)
            # the plan must exist for these hints (a hint the layer's A-load mode cannot take, e.g.
            # CTA pairs on a gathered stem, fails here rather than at launch)
            if kind == "conv":
                kernels.conv_gemm_plan(a)
            else:
                kernels._lib.check(kernels._lib.load().abft_gemm_plan(kernels.ctypes.byref(a),
                                                                       (kernels.ctypes.c_int32 * 10)()))
            L.args[key] = (kind, a)
        except Exception:
            L.tile_n[key], L.flags[key] = old
            raise

    def config_of(self, L: LinearLayer, key) -> tuple:
        return L.tile_n.get(key, 0), L.flags.get(key, 0)

    def set_global_variant(self, L: LinearLayer, variant: str) -> None:
        """The global-ABFT lhs source of one layer: "slice" (an extra MMA N-slice against the weight
        tile's row sums), "dot" (the checksum warps dot each staged A tile with rowck(B) on CUDA
        cores; the CTA tile stays as wide as the unprotected one) or "fused" (the producer layer's
        epilogue accumulates this layer's activation checksum — window sums of its stored output —
        and abft_window_lhs dots it with rowck(B) after the layer: no checksum work in this kernel)."""
        if variant not in ("slice", "dot", "fused"):
            raise ValueError("global variant is 'slice', 'dot' or 'fused'")
        if variant == "fused" and L.producer is None:
            raise ValueError(f"{L.name}: no producer layer supplies its window sums")
        L.gvar = variant
        self._refresh_window_sums()

    @staticmethod
    def _key(L: LinearLayer, scheme: Scheme):
        if scheme is Scheme.GLOBAL_ABFT and L.gvar == "dot":
            return GLOBAL_DOT
        if scheme is Scheme.GLOBAL_ABFT and L.gvar == "fused":
            return GLOBAL_FUSED
        return scheme

    def fused_batch(self):
        """The forward's deferred fused-checksum work: the border buckets of every producer with a
        fused 3x3 consumer and the window lhs of every fused consumer, as two launches after the
        layers (every activation keeps its own buffer, so the producers' outputs are still there)."""
        fused = [L for L in self.layers
                 if L.producer is not None and L.scheme is Scheme.GLOBAL_ABFT and L.gvar == "fused"]
        sig = tuple(L.index for L in fused)
        # one table per set of fused layers, kept for the network's lifetime: captured graphs of
        # earlier configurations still point at theirs
        cache = self.__dict__.setdefault("_fused_batches", {})
        if sig not in cache:
            border, window, seen = [], [], set()
            for L in fused:
                P, x = L.producer, L.x
                if L.r == 3 and id(P) not in seen:
                    seen.add(id(P))
                    border.append((x.buf, x.n, x.h, x.w, x.cp, x.ld, P._wsum, P.out.cp))
                window.append((P._wsum, P.out.cp, L.x.cp, L.r, L.s, L._k // (L.r * L.s), L._rowck, L._bias_dev,
                               _r8(L.oc), L.m, self.partials[L.index, 0, 0:1]))
            cache[sig] = kernels.FusedLhsBatch(border, window, self.dtype)
        return cache[sig]

    def launch(self, L: LinearLayer, scheme=None, deferred: bool = False) -> None:
        """One layer's kernel under `scheme` (default: the layer's; GLOBAL_DOT / GLOBAL_FUSED pick a
        global variant explicitly).  The fused variant is the kernel (output summation only) plus
        the window-lhs launch adding colck(A) . rowck(B) + M * sum(bias) to the layer's lhs slot
        (deferred=True: left to the forward's batched launches, fused_batch)."""
        if scheme in (GLOBAL_DOT, GLOBAL_FUSED):
            key = scheme
        else:
            key = self._key(L, L.scheme if scheme is None else scheme)
        kind, args = L.fault_args.get(key) or L.args[key]
        if kind == "gemm":
            kernels._lib.check(kernels._lib.load().abft_gemm(kernels.ctypes.byref(args), D.stream_handle()))
        else:
            kernels.conv2d(args)
        if key == GLOBAL_FUSED and not deferred:
            P = L.producer
            # (once per forward and producer: by its first 3x3 consumer running the fused lhs)
            fc = [C for C in self.fused_consumers(P)
                  if C.r == 3 and C.scheme is Scheme.GLOBAL_ABFT and C.gvar == "fused"]
            if L.r == 3 and (not fc or fc[0] is L):
                x = L.x
                kernels.border_sums(x.buf, x.n, x.h, x.w, x.cp, x.ld, self.dtype, P._wsum, P.out.cp)
            kernels.window_lhs(P._wsum, P.out.cp, L.x.cp, L.r, L.s, L._k // (L.r * L.s), L._rowck, L._bias_dev,
                               _r8(L.oc), L.m, self.partials[L.index, 0, 0:1])

    # ---------------------------------------------------------------- schemes / faults
    def set_schemes(self, schemes) -> None:
        if isinstance(schemes, Scheme):
            schemes = [schemes] * len(self.layers)
        if isinstance(schemes, str):
            schemes = [Scheme(schemes)] * len(self.layers)
        if len(schemes) != len(self.layers):
            raise ValueError("one scheme per linear layer")
        for L, s in zip(self.layers, schemes):
            if s not in SELECTABLE:
                raise ValueError(f"network layers take {[x.value for x in SELECTABLE]}, got {s}")
            L.scheme = s
        self._refresh_window_sums()

    def schemes(self) -> List[Scheme]:
        return [L.scheme for L in self.layers]

    def inject(self, faults: Dict[int, Sequence]) -> None:
        """Deterministic faults {layer index: [(row, col, delta)]} (row = output pixel index
        (n*P + p)*Q + q, col = output channel): delta is added to the fp32 accumulator before any
        checksum, bias, ReLU or store (tiled.py:197-200).  {} clears them."""
        for L in self.layers:
            L.fault_args = {}
        for i, cells in faults.items():
            L = self.layers[int(i)]
            if not cells:
                continue
            ft = D.faults_tensor(list(cells))
            L._fault_keep = ft
            for key in self.keys_of(L):
                L.fault_args[key] = self._make_args(L, key, faults=ft)

    # ---------------------------------------------------------------- forward
    def load_input(self, x) -> None:
        """x: [n, 3, h, w] (NCHW, any float dtype / device) -> the NHWC input buffer (stream-ordered)."""
        self.input.buf[..., :3].copy_(x.permute(0, 2, 3, 1), non_blocking=True)

    def forward(self, x=None, verify: bool = True):
        """Enqueue one protected forward (no host sync): clear the accumulators, run every op, then
        (verify=True) ONE verification launch over all layers.  Returns the logits tensor [n, classes]."""
        if x is not None:
            self.load_input(x)
        kernels.zero(self._block)
        for op in self.ops:
            if isinstance(op, LinearLayer):
                self.launch(op, deferred=True)
            else:
                op.fn()
        self.fused_batch().launch()
        if verify:
            self.verify()
        return self.logits()

    def forward_glue(self) -> None:
        """Only the glue ops of a forward (pooling / shuffle): subtracted from whole-forward times to
        get the overhead over the linear layers alone."""
        for op in self.ops:
            if not isinstance(op, LinearLayer):
                op.fn()

    def n_launches(self) -> int:
        """Kernel launches of one forward (layers, glue, the verification launch)."""
        fb = self.fused_batch()
        return len(self.ops) + int(any(L.scheme is Scheme.GLOBAL_ABFT for L in self.layers)) + \
            int(fb.grids[0] > 0) + int(fb.grids[1] > 0)

    def verify(self) -> None:
        if any(L.scheme is Scheme.GLOBAL_ABFT for L in self.layers):
            kernels.verify_partials(self.partials, self.ks, len(self.layers), self.numeric, out=self.verdict_buf,
                                    detected_count=self.counters[1:2])

    def verify_sharded(self, group=None) -> None:
        """Batch sharding: this rank's per-layer (lhs, rhs) sums and flag counters go out in ONE
        all-reduce, then the verdicts are formed from the full-batch sums (checksum.py:237)."""
        import torch.distributed as dist
        nl = len(self.layers)
        kernels.sum_partials(self.partials, nl, self.sums)
        self.reduce_buf[:2 * nl].copy_(self.sums.view(-1))
        self.reduce_buf[2 * nl] = self.counters[0]
        self.reduce_buf[2 * nl + 1] = 0.0
        dist.all_reduce(self.reduce_buf, group=group)
        self.sums.view(-1).copy_(self.reduce_buf[:2 * nl])
        self.counters[0] = self.reduce_buf[2 * nl].to(self.t.int32)
        self.counters[1] = 0
        if any(L.scheme is Scheme.GLOBAL_ABFT for L in self.layers):
            kernels.verify_sums(self.sums, self.ks, nl, self.numeric, out=self.verdict_buf,
                                detected_count=self.counters[1:2])

    def logits(self):
        o = self.output
        return o.buf.reshape(o.n, -1)[:, :o.c] if o.phys is None else o.buf.reshape(o.n, -1)[:, o.phys]

    def flags(self) -> tuple:
        """(fired thread tiles, flagged global layers) — one small D2H read."""
        c = self.counters.cpu().tolist()
        return int(c[0]), int(c[1])

    def verdicts(self) -> List[Optional[Verdict]]:
        """Per layer: the global verdict (Verdict) of a global-ABFT layer, else None."""
        raw = self.verdict_buf.cpu().numpy().view(_VERDICT_DTYPE)
        out = []
        for L, v in zip(self.layers, raw):
            out.append(Verdict(detected=bool(v["det"]), lhs=float(v["lhs"]), rhs=float(v["rhs"]),
                               tolerance_used=float(v["tol"])) if L.scheme is Scheme.GLOBAL_ABFT else None)
        return out

    def flops(self) -> int:
        return sum(L.flops() for L in self.layers)

    def gemm_layers(self):
        return [(L.index, L.gemm_shape()) for L in self.layers]


def verify_sharded_many(nets: Sequence[ProtectedNetwork], group=None, _cache={}) -> None:
    """Batch-sharded verification of several networks with ONE all-reduce: every network's
    per-layer (lhs, rhs) sums and fired-tile count, then each network's verdicts from the
    full-batch sums (exactly the single-GPU verdicts; checksum.py:237)."""
    import torch.distributed as dist
    t = D.torch()
    key = tuple(id(n) for n in nets)
    buf = _cache.get(key)
    sizes = [2 * len(n.layers) + 1 for n in nets]
    if buf is None:
        buf = _cache[key] = t.zeros(sum(sizes), dtype=t.float64, device="cuda")
    o = 0
    for n, sz in zip(nets, sizes):
        nl = len(n.layers)
        kernels.sum_partials(n.partials, nl, n.sums)
        buf[o:o + 2 * nl].copy_(n.sums.view(-1))
        buf[o + 2 * nl:o + sz].copy_(n.counters[0:1])
        o += sz
    dist.all_reduce(buf, group=group)
    o = 0
    for n, sz in zip(nets, sizes):
        nl = len(n.layers)
        n.sums.view(-1).copy_(buf[o:o + 2 * nl])
        n.counters[0:1].copy_(buf[o + 2 * nl:o + sz])
        n.counters[1:2].zero_()
        if any(L.scheme is Scheme.GLOBAL_ABFT for L in n.layers):
            kernels.verify_sums(n.sums, n.ks, nl, n.numeric, out=n.verdict_buf, detected_count=n.counters[1:2])
        o += sz


class GraphedNetwork:
    """One protected forward (accumulator memset, every layer and glue op, the verification
    launch) captured once in a CUDA graph and replayed; the input is the network's static input
    buffer (``load_input`` before ``replay``)."""

    def __init__(self, net: ProtectedNetwork, warmup: int = 2, verify: bool = True):
        t = D.torch()
        self.net = net
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            for _ in range(warmup):
                net.forward(verify=verify)
        t.cuda.current_stream().wait_stream(s)
        net.fused_batch()          # (its device table is written synchronously: never during capture)
        t.cuda.synchronize()
        self.graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.graph, stream=s):
            net.forward(verify=verify)
        t.cuda.synchronize()

    def replay(self) -> None:
        self.graph.replay()


# ------------------------------------------------------------------------------- model builders
def fold_bn(conv, bn):
    """Conv2d (+ BatchNorm2d in eval mode) -> (weight fp32 [oc, cin, r, s], bias fp32 [oc] or None)."""
    t = D.torch()
    w = conv.weight.detach().to(t.float64)
    b = conv.bias.detach().to(t.float64) if conv.bias is not None else None
    if bn is None:
        return w.float(), (b.float() if b is not None else None)
    scale = bn.weight.detach().to(t.float64) / t.sqrt(bn.running_var.detach().to(t.float64) + bn.eps)
    shift = bn.bias.detach().to(t.float64) - bn.running_mean.detach().to(t.float64) * scale
    if b is not None:
        shift = shift + b * scale
    return (w * scale.view(-1, 1, 1, 1)).float(), shift.float()


def dense_weight(conv):
    """A grouped / depthwise conv weight expanded to its dense block-diagonal equivalent
    (the paper treats grouped convs as dense)."""
    t = D.torch()
    w = conv.weight.detach()
    g = conv.groups
    if g == 1:
        return w
    oc, cpg, r, s = (int(v) for v in w.shape)
    cin = cpg * g
    opg = oc // g
    dense = t.zeros((oc, cin, r, s), dtype=w.dtype, device=w.device)
    for gi in range(g):
        dense[gi * opg:(gi + 1) * opg, gi * cpg:(gi + 1) * cpg] = w[gi * opg:(gi + 1) * opg]
    return dense


def _conv(net: ProtectedNetwork, name: str, x: Act, conv, bn=None, relu: bool = True, residual=None, out=None,
          c_real: int = 0) -> Act:
    class _C:   # the dense view of a grouped conv, for fold_bn
        pass
    c = _C()
    c.weight, c.bias = dense_weight(conv), conv.bias
    w, b = fold_bn(c, bn)
    return net.add_linear(name, x, w, b, stride=conv.stride[0], pad=conv.padding[0], relu=relu, residual=residual,
                          out=out, c_real=c_real)


def _fc(net: ProtectedNetwork, name: str, x: Act, lin, relu: bool, chw=None) -> Act:
    """Linear on a flattened NHWC activation; chw = (c, h, w) of the torchvision flatten order
    (NCHW) when the input is a spatial map, permuted here to the NHWC order."""
    t = D.torch()
    w = lin.weight.detach().to(t.float32)
    if chw is not None:
        c, h, ww = chw
        w = w.view(-1, c, h, ww).permute(0, 2, 3, 1).reshape(w.shape[0], -1)
    feats = x.h * x.w * x.cp
    if x.phys is not None or x.cp != x.c:
        if x.h * x.w != 1:
            raise ValueError(f"{name}: padded channels in a spatial FC input are not supported")
    flat = Act(x.buf.reshape(x.n, 1, 1, feats), x.h * x.w * x.c,
               None if (x.phys is None and x.cp == x.c) else x.phys_map())
    return net.add_linear(name, flat, w.view(w.shape[0], -1, 1, 1), lin.bias, relu=relu, kind="fc")


def _build(net: ProtectedNetwork, model) -> Act:
    import torchvision.models as tvm
    if isinstance(model, tvm.ResNet):
        return _build_resnet(net, model)
    if isinstance(model, (tvm.VGG, tvm.AlexNet)) or type(model).__name__ == "NoScopeCNN":
        return _build_vgg(net, model)
    if isinstance(model, tvm.SqueezeNet):
        return _build_squeezenet(net, model)
    if isinstance(model, tvm.ShuffleNetV2):
        return _build_shufflenet(net, model)
    raise ValueError(f"unsupported network {type(model).__name__}: ResNet, VGG, AlexNet, SqueezeNet, ShuffleNetV2, "
                     f"NoScopeCNN")


def _build_resnet(net, m) -> Act:
    """torchvision ResNet (Bottleneck or BasicBlock): stem, maxpool, residual stages, avgpool, fc."""
    import torchvision.models.resnet as R
    a = _conv(net, "conv1", net.input, m.conv1, m.bn1, c_real=3)
    a = net.maxpool(a, m.maxpool.kernel_size, m.maxpool.stride, m.maxpool.padding)
    for li, layer in enumerate((m.layer1, m.layer2, m.layer3, m.layer4), start=1):
        for bi, blk in enumerate(layer):
            p = f"layer{li}.{bi}"
            idt = a
            if blk.downsample is not None:
                idt = _conv(net, p + ".downsample", a, blk.downsample[0], blk.downsample[1], relu=False)
            if isinstance(blk, R.Bottleneck):
                t1 = _conv(net, p + ".conv1", a, blk.conv1, blk.bn1)
                t2 = _conv(net, p + ".conv2", t1, blk.conv2, blk.bn2)
                a = _conv(net, p + ".conv3", t2, blk.conv3, blk.bn3, relu=True, residual=idt)
            else:
                t1 = _conv(net, p + ".conv1", a, blk.conv1, blk.bn1)
                a = _conv(net, p + ".conv2", t1, blk.conv2, blk.bn2, relu=True, residual=idt)
    a = net.avgpool(a)
    return _fc(net, "fc", a, m.fc, relu=False)


def _build_vgg(net, m) -> Act:
    """torchvision VGG / AlexNet (and the NoScope CNNs, which have no adaptive pool): conv(+ReLU) /
    maxpool features, identity adaptive pool at 224, then the classifier's Linear(+ReLU) layers
    (Dropout is the identity in eval)."""
    import torch.nn as nn
    a = net.input
    mods = list(m.features)
    first = True
    for i, mod in enumerate(mods):
        if isinstance(mod, nn.Conv2d):
            relu = i + 1 < len(mods) and isinstance(mods[i + 1], nn.ReLU)
            a = _conv(net, f"features.{i}", a, mod, None, relu=relu, c_real=3 if first else 0)
            first = False
        elif isinstance(mod, nn.MaxPool2d):
            a = net.maxpool(a, mod.kernel_size, mod.stride, mod.padding, mod.ceil_mode)
    osz = m.avgpool.output_size if hasattr(m, "avgpool") else (a.h, a.w)
    osz = (osz, osz) if isinstance(osz, int) else tuple(osz)
    if (a.h, a.w) != osz:
        raise ValueError(f"adaptive pool {osz} on a {a.h}x{a.w} map: only the identity case (224 input) is supported")
    chw = (a.c, a.h, a.w)
    lins = [(i, mod) for i, mod in enumerate(m.classifier) if isinstance(mod, nn.Linear)]
    cls = list(m.classifier)
    for j, (i, lin) in enumerate(lins):
        relu = i + 1 < len(cls) and isinstance(cls[i + 1], nn.ReLU)
        a = _fc(net, f"classifier.{i}", a, lin, relu=relu, chw=chw if j == 0 else None)
    return a


def _build_squeezenet(net, m) -> Act:
    """torchvision SqueezeNet: Fire modules write both expand convs into one buffer (the concat)."""
    import torch.nn as nn
    import torchvision.models.squeezenet as S
    a = net.input
    mods = list(m.features)
    for i, mod in enumerate(mods):
        if isinstance(mod, nn.Conv2d):
            a = _conv(net, f"features.{i}", a, mod, None, relu=True, c_real=3)
        elif isinstance(mod, nn.MaxPool2d):
            a = net.maxpool(a, mod.kernel_size, mod.stride, mod.padding, mod.ceil_mode)
        elif isinstance(mod, S.Fire):
            sq = _conv(net, f"features.{i}.squeeze", a, mod.squeeze, None, relu=True)
            e1, e3 = mod.expand1x1.out_channels, mod.expand3x3.out_channels
            cat = net.new_act(sq.n, sq.h, sq.w, e1 + e3)
            o1 = Act(cat.buf[..., :_r8(e1)], e1)
            o3 = Act(cat.buf[..., _r8(e1):_r8(e1) + _r8(e3)], e3)
            _conv(net, f"features.{i}.expand1x1", sq, mod.expand1x1, None, relu=True, out=o1)
            _conv(net, f"features.{i}.expand3x3", sq, mod.expand3x3, None, relu=True, out=o3)
            a = cat if _r8(e1) == e1 else Act(cat.buf, e1 + e3, np.concatenate([np.arange(e1), _r8(e1) + np.arange(e3)]))
    conv = m.classifier[1]
    a = _conv(net, "classifier.1", a, conv, None, relu=True)
    return net.avgpool(a)


def _build_shufflenet(net, m) -> Act:
    """torchvision ShuffleNetV2: depthwise convs as dense, units' cat + channel_shuffle by the
    interleave glue into the halves layout, chunk(2) as channel-slice views."""
    a = _conv(net, "conv1", net.input, m.conv1[0], m.conv1[1], c_real=3)
    a = net.maxpool(a, m.maxpool.kernel_size, m.maxpool.stride, m.maxpool.padding)
    for si, stage in enumerate((m.stage2, m.stage3, m.stage4), start=2):
        for ui, unit in enumerate(stage):
            p = f"stage{si}.{ui}"
            b2 = unit.branch2
            if unit.stride == 1:
                hp = _r8(a.c // 2)
                half = a.c // 2
                x1 = Act(a.buf[..., :hp], half)
                x2 = Act(a.buf[..., hp:2 * hp], half)
                t1 = _conv(net, p + ".branch2.0", x2, b2[0], b2[1])
                t2 = _conv(net, p + ".branch2.3", t1, b2[3], b2[4], relu=False)
                bo = _conv(net, p + ".branch2.5", t2, b2[5], b2[6])
                a = net.shuffle_cat(x1, bo)
            else:
                b1 = unit.branch1
                u1 = _conv(net, p + ".branch1.0", a, b1[0], b1[1], relu=False)
                o1 = _conv(net, p + ".branch1.2", u1, b1[2], b1[3])
                t1 = _conv(net, p + ".branch2.0", a, b2[0], b2[1])
                t2 = _conv(net, p + ".branch2.3", t1, b2[3], b2[4], relu=False)
                bo = _conv(net, p + ".branch2.5", t2, b2[5], b2[6])
                a = net.shuffle_cat(o1, bo)
    a = _conv(net, "conv5", a, m.conv5[0], m.conv5[1])
    a = net.avgpool(a)
    return _fc(net, "fc", a, m.fc, relu=False)


# ------------------------------------------------------------------------------- helpers
def calibrate_bn(model, batch: int = 8, h: int = 224, w: int = 224, seed: int = 0):
    """Give a randomly initialised model realistic BatchNorm statistics (one training-mode pass
    over seeded inputs with momentum 1) and non-trivial affine parameters, so the folded
    weights / biases of the protected network are those of a normalised network — activations
    stay O(1) through every layer as in a trained model.  Returns the model in eval mode."""
    import torch
    import torch.nn as nn
    g = torch.Generator().manual_seed(seed)
    if not any(isinstance(mod, nn.BatchNorm2d) for mod in model.modules()):
        return model.eval()
    for mod in model.modules():
        if isinstance(mod, nn.BatchNorm2d):
            mod.momentum = 1.0
            with torch.no_grad():
                mod.weight.copy_(0.5 + torch.rand(mod.weight.shape, generator=g))
                mod.bias.copy_(0.2 * (torch.rand(mod.bias.shape, generator=g) - 0.5))
    model.train()
    with torch.no_grad():
        model(torch.rand((batch, 3, h, w), generator=g) * 2 - 1)
    return model.eval()


def build_model(name: str, seed: int = 0, calibrate: bool = True):
    """A torchvision model with seeded random weights (no checkpoints offline) and calibrated BN."""
    import torch
    import torchvision
    if name.startswith("noscope_"):
        from . import noscope
        return noscope.build(name, seed)
    torch.manual_seed(seed)
    model = getattr(torchvision.models, name)(weights=None)
    if calibrate:
        calibrate_bn(model, seed=seed)
    return model.eval()
