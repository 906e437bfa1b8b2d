"""Protected multi-layer inference with a per-layer ABFT plan (the paper's deployment mode).

A ``ProtectedChain`` is a sequence of linear layers (FC, or conv already lowered to a
GEMM) with ReLU between them — the chain of ``run_protected_pipeline``
(checksum.py:198-237) — where every layer carries its own scheme:

  unprotected   plain tcgen05 GEMM
  global-abft   output summation (rhs) in the epilogue; lhs colck(A) . rowck(B) regrouped
                as sum_rows A . rowck(B tile) — one extra MMA N-slice against the weight
                tile's row sums, summed in the same epilogue, so no activation checksum
                pass is needed; the verdicts of all layers run in one launch at the end
  thread-one-sided  checksum N-slice in the same MMA, per-row compare in the
                epilogue; fired thread tiles counted on device

Everything for one forward is enqueued on the current stream with no host sync and
can be captured in a CUDA graph; ``flags()`` reads back two counters (fired thread
tiles, flagged global layers) — the deferred verification of the reference.

Multi-GPU: batch sharding needs no collective on the hot path; ``global_partials``
exposes the per-layer [lhs, rhs] sums so callers can all-reduce them (NCCL) and call
``verify_reduced`` to obtain exactly the full-batch global verdicts.
"""

from __future__ import annotations

import os

_NO_PDL = bool(os.environ.get("ABFT_NO_PDL"))     # measurement toggle

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import device as D
from . import kernels
from .schemes import Scheme, TilingConfig
from .shapes import BINARY16, DType


@dataclass
class _Layer:
    k: int            # padded K (multiple of 8): the GEMM launch's K
    n: int            # padded N (multiple of 8)
    pw: D.PreparedWeight
    scheme: Scheme
    ck_rows: object = None
    relu: bool = True
    k_ref: int = 0    # the model's unpadded K: the global scheme's tau K (checksum.py:147-153)


@dataclass
class ProtectedChain:
    """Layers given as K x N weights (torch fp16/bf16 CUDA tensors or numpy)."""

    weights: Sequence
    batch: int
    schemes: Sequence[Scheme]
    dtype: DType = BINARY16
    tiling: TilingConfig = TilingConfig()
    relu_last: bool = True
    ck_split: bool = False
    faults: Optional[dict] = None        # {layer: [(row, col, delta)]}: deltas added to the fp32 accumulator
    pdl: bool = True                     # programmatic dependent launch between consecutive layers
    tile_ns: Optional[Sequence[int]] = None   # per-layer CTA tile (0: the planner's), e.g. a grouped launch's
    plan_flags: int = 0                  # abft_gemm_args_t.plan_flags for every layer
    # (sums [nl, 2] fp64, counters int32 [2], vdone int32 [1][, partials [nl, cap, 2] fp64]) views of
    # a ChainGroup's block: the group clears them and verifies every member's global layers in one
    # launch; with partials, each CTA of a global layer writes its (lhs, rhs) to its own slot
    shared: Optional[tuple] = None
    layers: List[_Layer] = field(default_factory=list, init=False)

    def __post_init__(self):
        D.require_device()
        t = D.torch()
        self._fault_dev = {int(i): D.faults_tensor(list(f)) for i, f in (self.faults or {}).items() if f}
        if len(self.schemes) != len(self.weights):
            raise ValueError("one scheme per layer")
        self.numeric = D.numeric_code(self.dtype)
        sd = D.torch_storage_dtype(self.dtype)
        prev_n = None
        for i, (w, sch) in enumerate(zip(self.weights, self.schemes)):
            k, n = D.shape2d(w, f"weights[{i}]")
            kp = D.round8(k)
            if prev_n is not None and kp != prev_n:
                raise ValueError(f"layer {i}: K={k} does not chain with the previous N={prev_n}")
            pw = D.prepare_weight(w, self.dtype)
            self.layers.append(_Layer(k=kp, n=D.round8(n), pw=pw, scheme=sch,
                                      relu=(i < len(self.weights) - 1) or self.relu_last, k_ref=k))
            prev_n = D.round8(n)
        m = self.batch
        self.x = t.zeros((m, self.layers[0].k), dtype=sd, device="cuda")
        self.acts = [t.zeros((m, L.n), dtype=sd, device="cuda") for L in self.layers]
        nl = len(self.layers)
        if self.shared is None:
            # every per-forward accumulator lives in ONE block so a single memset node clears it:
            # [(lhs, rhs) fp64 per layer][counters int32 x 2][verification done-count int32, pad]
            off_cnt = 16 * nl
            self.scratch = t.zeros(off_cnt + 16, dtype=t.uint8, device="cuda")
            self.sums = self.scratch[:off_cnt].view(t.float64).view(nl, 2)
            self.counters = self.scratch[off_cnt:off_cnt + 8].view(t.int32)   # [fired thread tiles, flagged layers]
            self.vdone = self.scratch[off_cnt + 8:off_cnt + 12].view(t.int32)
        else:
            self.scratch = None
            self.sums, self.counters, self.vdone = self.shared[:3]
        self.partials = self.shared[3] if self.shared is not None and len(self.shared) > 3 else None
        self.verdict_buf = t.zeros(max(nl, 1) * 32, dtype=t.uint8, device="cuda")
        self.global_ids = [i for i, L in enumerate(self.layers) if L.scheme is Scheme.GLOBAL_ABFT]
        self._ks_all = t.tensor([L.k_ref for L in self.layers], dtype=t.int32, device="cuda")
        self._ks = t.tensor([self.layers[i].k_ref for i in self.global_ids] or [0], dtype=t.int32, device="cuda")
        # offline checksum rows: the global scheme's lhs slice (always), and the one-sided
        # check's rows where the plan says B tiles are re-read by several M-blocks
        for i, L in enumerate(self.layers):
            if L.scheme in (Scheme.THREAD_ONE_SIDED, Scheme.GLOBAL_ABFT):
                # weights with each tile's checksum rows appended: outputs and checksums from one MMA
                kw = self._gemm_kwargs(i, L)
                plan = kernels.gemm(self.x, self.x.stride(0), L.pw.bt, L.pw.ldbt, self.batch, L.n, L.k, self.dtype,
                                    self.numeric, L.scheme, plan_only=True, ck_layout=1, **kw)
                if L.scheme is Scheme.GLOBAL_ABFT:
                    L.ck_rows = kernels.global_ck_rows(L.pw.bt, L.n, L.k, self.dtype, plan)
                else:
                    L.ck_rows = kernels.aug_weights(L.pw.bt, L.n, L.k, self.dtype, plan, self.tiling.thread_n,
                                                    self.ck_split)

    def _gemm_kwargs(self, i: int, L: _Layer) -> dict:
        t = self.tiling
        m = self.batch
        kw = dict(out=self.acts[i], ldc=self.acts[i].stride(0),
                  out_kind="bf16" if self.acts[i].dtype == D.torch().bfloat16 else "f16", relu=L.relu,
                  tile_n=self.tile_ns[i] if self.tile_ns else 0, plan_flags=self.plan_flags)
        if i in self._fault_dev:
            kw["faults"], kw["nfaults"] = self._fault_dev[i]
        if L.scheme is Scheme.GLOBAL_ABFT:
            if getattr(self, "partials", None) is not None:
                kw["out_partials"] = self.partials[i]
            else:
                kw["out_lhs"] = self.sums[i, 0:1]
                kw["out_sum"] = self.sums[i, 1:2]
        elif L.scheme is not Scheme.UNPROTECTED:
            kw.update(thread_m=t.thread_m, thread_n=t.thread_n, m_ext=-(-m // t.thread_m) * t.thread_m,
                      n_ext=-(-L.n // t.thread_n) * t.thread_n, tol_k=-(-L.k // t.k_step) * t.k_step,
                      fired_count=self.counters[0:1], ck_split=self.ck_split)
        return kw

    def forward(self, x=None) -> object:
        """Enqueue one protected forward (no host sync); returns the last activation tensor."""
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        if self.scratch is not None:
            kernels.zero(self.scratch)
        a = self.x
        last = len(self.layers) - 1
        for i, L in enumerate(self.layers):
            kw = self._gemm_kwargs(i, L)
            kw["pdl"] = i > 0 and self.pdl and not _NO_PDL      # layer i's prologue overlaps layer i-1
            if i == last and self.global_ids and self.shared is None:
                # deferred verification of every layer's (lhs, rhs), fused into the last layer's
                # launch (its last CTA); layers without the global scheme hold (0, 0), never flag
                kw["verify"] = (self.sums, self._ks_all, self.vdone, self.verdict_buf, self.counters[1:2])
            kernels.gemm(a, a.stride(0), L.pw.bt, L.pw.ldbt, self.batch, L.n, L.k, self.dtype, self.numeric,
                         L.scheme, ck_rows=L.ck_rows, **kw)
            a = self.acts[i]
        return a

    # ---- multi-GPU helpers (batch sharding): per-layer partial sums, all-reduced by the caller
    def global_partials(self):
        """[n_global, 2] fp64 (lhs, rhs) of this shard, valid after forward() on the stream.
        A ChainGroup member's global layers write per-CTA slots (``partials``), summed here."""
        if self.partials is not None:
            return self.partials[self.global_ids].sum(dim=1)
        return self.sums[self.global_ids]

    def verify_reduced(self, sums):
        """Verdicts from all-reduced (lhs, rhs) sums; returns the device counter of flagged layers."""
        t = D.torch()
        cnt = t.zeros(1, dtype=t.int32, device="cuda")
        kernels.verify_sums(sums.contiguous(), self._ks, len(self.global_ids), self.numeric, out=self.verdict_buf,
                            detected_count=cnt)
        return cnt

    def flags(self) -> tuple:
        """(fired thread tiles, flagged global layers) — one small D2H read."""
        c = self.counters.cpu().tolist()
        return int(c[0]), int(c[1])

    def flops(self) -> int:
        return sum(2 * self.batch * L.n * L.k for L in self.layers)


class GraphedForward:
    """A ProtectedChain forward captured once in a CUDA graph and replayed."""

    def __init__(self, chain: ProtectedChain, warmup: int = 2):
        t = D.torch()
        self.chain = chain
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            for _ in range(warmup):
                chain.forward()
        t.cuda.current_stream().wait_stream(s)
        t.cuda.synchronize()
        self.graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.graph, stream=s):
            chain.forward()
        t.cuda.synchronize()

    def replay(self):
        self.graph.replay()


class ChainGroup:
    """Independent chains (e.g. the requests of one serving step) sharing one accumulator block:
    ONE memset clears every member's (lhs, rhs) sums and counters, the members run their
    layers (on any streams), and ONE launch then forms the verdicts of every global layer of
    every member — the reference's deferred verification (checksum.py:207-211) batched across
    the group, instead of a done-count round trip at the end of each member's last kernel."""

    def __init__(self, specs, grouped: bool = False, **chain_kw):
        """specs: [(weights, batch, schemes)]; chain_kw: ProtectedChain fields shared by all.
        grouped: run each layer depth of all members as grouped launches (abft_gemm_group_*: one
        persistent launch per (depth, scheme) over every member's tiles) instead of one launch per
        layer and member; members must have equally many layers and no injected faults."""
        t = D.torch()
        nls = [len(w) for w, _, _ in specs]
        self.grouped = bool(grouped)
        if self.grouped:
            if len(set(nls)) != 1 or chain_kw.get("faults"):
                raise ValueError("grouped ChainGroup: members with equally many layers and no faults")
            # one CTA tile per depth (the group's common kernel configuration); k-block pairs off and
            # double output staging, which would otherwise depend on each member's K
            tiles = []
            for d in range(nls[0]):
                nmax = max(D.round8(D.shape2d(w[d], "w")[1]) for w, _, _ in specs)
                tiles.append(64 if nmax <= 64 else 128)
            chain_kw = dict(chain_kw, tile_ns=tiles, plan_flags=1 | 4)
        total = sum(nls)
        off_cnt = 16 * total
        off_flag = off_cnt + 16 * len(specs)
        # per-CTA (lhs, rhs) slots of every layer: plain stores instead of contended atomics
        self.cap = max(1, D.sm_count())
        off_part = off_flag + 16
        self.block = t.zeros(off_part + 16 * self.cap * total, dtype=t.uint8, device="cuda")
        self.sums = self.block[:off_cnt].view(t.float64).view(total, 2)
        cnt = self.block[off_cnt:off_flag].view(t.int32).view(len(specs), 4)
        self.partials = self.block[off_part:].view(t.float64).view(total, self.cap, 2)
        self.chains = []
        o = 0
        for (w, b, sch), nl in zip(specs, nls):
            self.chains.append(ProtectedChain(w, b, sch, shared=(self.sums[o:o + nl], cnt[len(self.chains), 0:2],
                                                                 cnt[len(self.chains), 2:3],
                                                                 self.partials[o:o + nl]), **chain_kw))
            o += nl
        self.counters = cnt
        ks = [L.k_ref for ch in self.chains for L in ch.layers]
        self.has_global = any(ch.global_ids for ch in self.chains)
        self.ks = t.tensor(ks, dtype=t.int32, device="cuda")
        self.verdicts = t.zeros(total * 32, dtype=t.uint8, device="cuda")
        self.flagged = self.block[off_flag:off_flag + 4].view(t.int32)
        self.tail = self.block[off_cnt:off_part]    # counters + flag count: one D2H read
        self.numeric = self.chains[0].numeric
        self._groups = []
        if self.grouped:
            self._build_groups()

    def _build_groups(self) -> None:
        """Per layer depth and scheme: the members' launch arguments and a prepared problem table."""
        t = D.torch()
        pb = kernels.group_problem_bytes()
        for d in range(len(self.chains[0].layers)):
            by_scheme = {}
            for ch in self.chains:
                L = ch.layers[d]
                a = ch.x if d == 0 else ch.acts[d - 1]
                kw = ch._gemm_kwargs(d, L)
                kw["pdl"] = d > 0 and ch.pdl and not _NO_PDL
                args = kernels._gemm_args(a, a.stride(0), L.pw.bt, L.pw.ldbt, ch.batch, L.n, L.k, ch.dtype, ch.numeric,
                                          L.scheme, ck_rows=L.ck_rows, **kw)
                by_scheme.setdefault(L.scheme, []).append(args)
            for sch, lst in by_scheme.items():
                raw = t.empty(pb * len(lst) + 64, dtype=t.uint8, device="cuda")
                off = (-raw.data_ptr()) % 64
                table = raw[off:off + pb * len(lst)]
                kernels.gemm_group_prepare(lst, table)
                arr = (kernels._lib.GemmArgs * len(lst))(*lst)
                self._groups.append((arr, len(lst), table, raw, lst))

    def begin(self) -> None:
        """Clear every member's per-forward accumulators and the flag count (one memset)."""
        kernels.zero(self.block)

    def end(self) -> None:
        """One verification launch over all members' layers (non-global layers hold (0, 0))."""
        if self.has_global:
            kernels.verify_partials(self.partials, self.ks, self.ks.numel(), self.numeric, out=self.verdicts,
                                    detected_count=self.flagged)

    def forward(self) -> None:
        self.begin()
        if self.grouped:
            for arr, n, table, _raw, _keep in self._groups:
                kernels.gemm_group_launch(arr, n, table)
        else:
            for ch in self.chains:
                ch.forward()
        self.end()

    def flags(self) -> tuple:
        """(fired thread tiles over all members, flagged global layers over all members)."""
        c = self.counters.cpu()
        return int(c[:, 0].sum()), int(self.flagged.item())
