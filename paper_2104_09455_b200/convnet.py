"""Per-layer protected execution of CNN layers for the network-level measurements (C3-C5).

The paper measures a network's ABFT overhead as the sum of its linear layers' times
(cost.py:186-187 sums T_r / T_o the same way), each layer timed under
each scheme on its real input extent.  ``LayerRunner`` holds one layer's device
buffers (NHWC input, packed weight, checksums, output) and enqueues it under
unprotected / global / one-sided ABFT:

  unprotected       implicit-GEMM conv (or GEMM), fp16 store
  global-abft       the same kernel with the output summation (rhs) in its epilogue and the
                    lhs colck(A) . rowck(B) regrouped as sum_rows A . rowck(B tile): one
                    extra MMA N-slice against the weight tile's row sums, summed in the
                    epilogue (the input comes out of pooling / residual / BN glue, so a
                    producer-fused activation checksum is not available); or the
                    lhs as the checksum warps' dot of the staged A tiles with rowck(B)
                    (the tile stays as wide as the unprotected one); or the windowed
                    activation checksum by a standalone pass
                    + its share of the network's single batched verification
  thread-one-sided  checksum N-slice in the same MMA, per-row compares in the epilogue

Activations are seeded U(-1, 1) synthetic tensors of each layer's input shape, weights
U(-a, a) with a = 1/sqrt(fan_in) (keeps outputs O(1) so fp16 stores are finite).
"""

from __future__ import annotations

from typing import Dict

from . import device as D
from . import kernels
from .conv import PreparedConv, geometry, prepare_conv_weight, standalone_colck
from .conv import plan as conv_plan
from .networks import LayerSpec
from .schemes import Scheme, TilingConfig
from .shapes import BINARY16, DType


class LayerRunner:
    def __init__(self, spec: LayerSpec, dtype: DType = BINARY16, tiling: TilingConfig = TilingConfig(),
                 seed: int = 0, offline_ck: bool = True):
        t = D.torch()
        self.spec, self.dtype, self.tiling = spec, dtype, tiling
        self.numeric = D.numeric_code(dtype)
        sd = D.torch_storage_dtype(dtype)
        g = t.Generator(device="cuda")
        g.manual_seed(seed)
        c8 = D.round8(spec.cin)
        self.x = t.zeros((spec.n, spec.h, spec.w, c8), dtype=sd, device="cuda")
        self.x[..., :spec.cin] = (t.rand((spec.n, spec.h, spec.w, spec.cin), generator=g, device="cuda") * 2 - 1).to(sd)
        bound = 1.0 / (spec.cin * spec.r * spec.s) ** 0.5
        w = ((t.rand((spec.oc, spec.cin, spec.r, spec.s), generator=g, device="cuda") * 2 - 1) * bound).to(sd)
        self.geom = geometry(self.x, spec.r, spec.s, (spec.stride_h, spec.stride_w), (spec.pad_h, spec.pad_w),
                             spec.cin)
        self.plan = conv_plan(self.x, self.geom, spec.oc, dtype)
        self.pc: PreparedConv = prepare_conv_weight(w, dtype, self.plan["ck"], self.plan["k"])
        self.ws = t.empty(self.plan["ws"], dtype=t.uint8, device="cuda") if self.plan["ws"] else None
        self.m = spec.n * spec.p * spec.q
        self.n8 = D.round8(spec.oc)
        self.out = t.empty((self.m, self.n8), dtype=sd, device="cuda")
        self.scratch = t.zeros(64, dtype=t.float64, device="cuda")     # [0] lhs, [1] rhs, [2] counters
        self.lhs_rhs = self.scratch[0:2]
        self.rhs = self.scratch[1:2]
        self.counters = self.scratch[2:3].view(t.int32)
        self.colck = t.zeros(self.pc.bt.shape[1], dtype=t.float32, device="cuda")
        self.k_ref = spec.cin * spec.r * spec.s
        self.ks = t.tensor([self.k_ref], dtype=t.int32, device="cuda")
        self.task = kernels.global_tasks([(self.colck, self.pc.rowck, self.rhs, self.pc.bt.shape[1], self.k_ref)])
        self.sums = t.zeros(2, dtype=t.float64, device="cuda")
        self.verdict = t.zeros(32, dtype=t.uint8, device="cuda")
        self._args: Dict[Scheme, object] = {}
        self.ck_rows = None
        self.offline_ck = offline_ck
        for s in (Scheme.UNPROTECTED, Scheme.GLOBAL_ABFT, Scheme.THREAD_ONE_SIDED):
            self._args[s] = self._make_args(s)
        # global scheme with the activation checksum from a separate pass instead of in-kernel,
        # and with the lhs as the checksum warps' dot of the staged A tiles with rowck(B)
        self._args["global-standalone"] = self._make_args(Scheme.GLOBAL_ABFT, fused_colck=False)
        self._args["global-dot"] = self._make_args(Scheme.GLOBAL_ABFT, dot=True)
        self.global_variant = "fused"

    def _make_args(self, scheme: Scheme, fused_colck: bool = True, dot: bool = False):
        t = self.tiling
        kw = dict(out=self.out, ldc=self.n8, out_kind="bf16" if self.out.dtype == D.torch().bfloat16 else "f16",
                  relu=True)
        if scheme is Scheme.GLOBAL_ABFT:
            kw["out_sum"] = self.rhs
            if dot:
                kw["out_lhs"], kw["lhs_rowck"] = self.scratch[0:1], self.pc.rowck
            elif fused_colck:
                # lhs from the kernel's checksum N-slice against the weight tile's row sums
                kw["out_lhs"] = self.scratch[0:1]
                gplan = kernels.conv_gemm_plan(kernels.conv_args(self.x, self.geom, self.pc.bt, self.spec.oc,
                                                                 self.dtype, self.numeric, scheme, workspace=self.ws,
                                                                 ck_layout=1, **kw))
                kw["ck_rows"] = kernels.global_ck_rows(self.pc.bt, self.spec.oc, self.pc.bt.shape[1], self.dtype,
                                                       gplan)
        elif scheme is Scheme.THREAD_ONE_SIDED:
            kw.update(thread_m=t.thread_m, thread_n=t.thread_n, m_ext=-(-self.m // t.thread_m) * t.thread_m,
                      n_ext=-(-self.spec.oc // t.thread_n) * t.thread_n,
                      tol_k=-(-self.k_ref // t.k_step) * t.k_step, fired_count=self.counters)
        args = kernels.conv_args(self.x, self.geom, self.pc.bt, self.spec.oc, self.dtype, self.numeric, scheme,
                                 workspace=self.ws, **kw)
        if scheme is Scheme.THREAD_ONE_SIDED and self.offline_ck:
            # weights with each tile's checksum rows appended (one MMA per k-step)
            plan = kernels.conv_gemm_plan(kernels.conv_args(self.x, self.geom, self.pc.bt, self.spec.oc, self.dtype,
                                                            self.numeric, scheme, workspace=self.ws, ck_layout=1,
                                                            **kw))
            self.ck_rows = kernels.aug_weights(self.pc.bt, self.spec.oc, self.pc.bt.shape[1], self.dtype, plan,
                                               t.thread_n, False)
            args = kernels.conv_args(self.x, self.geom, self.pc.bt, self.spec.oc, self.dtype, self.numeric,
                                     scheme, ck_rows=self.ck_rows, workspace=self.ws, **kw)
        return args

    def flops(self) -> int:
        return 2 * self.m * self.spec.oc * self.k_ref

    def conv(self, scheme) -> None:
        kernels.conv2d(self._args["global-dot"] if scheme is Scheme.GLOBAL_ABFT and self.global_variant == "dot"
                       else self._args[scheme])

    def conv_variant(self, key) -> None:
        kernels.conv2d(self._args[key])

    def global_standalone(self) -> None:
        """Global ABFT with the standalone checksum pass (the other measured variant)."""
        self.colck_pass()
        kernels.conv2d(self._args["global-standalone"])

    def colck_pass(self) -> None:
        """Standalone activation checksum (one extra read of the input): the plain column
        sum for a pointwise conv (its A is the NHWC matrix itself), the windowed one otherwise."""
        standalone_colck(self.x, self.geom, self.plan, self.dtype, self.colck)

    def verify(self) -> None:
        if self.global_variant in ("fused", "dot"):
            kernels.verify_sums(self.lhs_rhs, self.ks, 1, self.numeric, out=self.verdict,
                                detected_count=self.counters)
        else:
            kernels.global_verify(self.task, 1, self.numeric, self.sums, out=self.verdict,
                                  detected_count=self.counters)

    def run(self, scheme: Scheme) -> None:
        """One protected execution of the layer (verification included for global)."""
        if scheme is Scheme.GLOBAL_ABFT:
            kernels.zero(self.scratch)
            if self.global_variant in ("fused", "dot"):
                self.conv(scheme)
            else:
                self.global_standalone()
            self.verify()
        else:
            self.conv(scheme)

    def flags(self) -> int:
        return int(self.counters.item())
