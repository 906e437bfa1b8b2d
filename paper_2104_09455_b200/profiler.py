"""Per-layer B200 timings for the intensity-guided selector ("measure each
layer under both schemes").

``profile_layers`` times every layer of a chain on the GPU under unprotected, global
and one-sided ABFT and returns the reference's ``MeasuredTimings`` (cost.py:131-171),
so the unchanged ``select`` (cost.py:174-238) picks per layer from measurements
rather than from a T4-calibrated model:

  T_o     the layer's GEMM alone (CUDA-graph replayed, CUDA events)
  T_one   GEMM with the checksum N-slice and the per-row compare (flags mode)
  T_glob  GEMM with the output summation (rhs) and the checksum N-slice whose row sum
          is lhs = sum_rows A . rowck(B tile) (both inside the one kernel)
          (the chain's verification is fused into the last CTA of its last launch)
"""

from __future__ import annotations

from typing import Sequence

from . import device as D
from . import kernels
from .cost import MeasuredTimings
from .network import ProtectedChain
from .schemes import Scheme, TilingConfig
from .shapes import BINARY16, DType


def capture_graph(fn, iters: int):
    """`iters` back-to-back calls of fn() captured in one CUDA graph (after one eager call); the
    launches' arguments are fixed at capture."""
    t = D.torch()
    s = t.cuda.Stream()
    s.wait_stream(t.cuda.current_stream())
    with t.cuda.stream(s):
        fn()
        t.cuda.synchronize()
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    t.cuda.synchronize()
    g.replay()
    t.cuda.synchronize()
    return g


def interleaved_min_us(graphs, iters: int, reps: int = 5) -> list:
    """Per-launch time (us) of each captured graph, best over `reps` rounds that replay every graph in
    turn: candidates compared under the same clock / power state (a power-capped B200 drifts by
    several % between back-to-back measurements of the same kernel)."""
    t = D.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    best = [float("inf")] * len(graphs)
    for _ in range(reps):
        for i, g in enumerate(graphs):
            e0.record()
            g.replay()
            e1.record()
            t.cuda.synchronize()
            best[i] = min(best[i], e0.elapsed_time(e1) * 1e3 / iters)
    return best


def graph_time_us(fn, iters: int = 40, reps: int = 5) -> float:
    """Best-of-reps mean time of `iters` back-to-back calls replayed from one CUDA graph."""
    t = D.torch()
    s = t.cuda.Stream()
    s.wait_stream(t.cuda.current_stream())
    with t.cuda.stream(s):
        fn()
        t.cuda.synchronize()
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    t.cuda.synchronize()
    g.replay()
    t.cuda.synchronize()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(reps):
        e0.record()
        g.replay()
        e1.record()
        t.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / iters)
    return best


def profile_layers(weights: Sequence, batch: int, dtype: DType = BINARY16,
                   tiling: TilingConfig = TilingConfig(), iters: int = 40, in_chain: bool = False) -> MeasuredTimings:
    """Measured per-layer times (seconds) for unprotected / global-abft / thread-one-sided.

    in_chain=False: each layer's kernel timed alone (back-to-back launches of that layer).
    in_chain=True: each layer timed where it runs — inside the chain (programmatic dependent
    launch from the previous layer, accumulators and verification owned by a ChainGroup as in
    a serving step): a layer's protected time is the unprotected chain's per-layer time plus
    the measured change of the whole chain's time when only that layer is protected."""
    if in_chain:
        return _profile_layers_in_chain(weights, batch, dtype, tiling, iters)
    n = len(weights)
    chains = {s: ProtectedChain(weights, batch, [s] * n, dtype, tiling) for s in
              (Scheme.UNPROTECTED, Scheme.GLOBAL_ABFT, Scheme.THREAD_ONE_SIDED)}
    entries = {}
    for i in range(n):
        # the three schemes' launches of layer i, timed in interleaved rounds
        keys, graphs = [], []
        for s, ch in chains.items():
            L = ch.layers[i]
            a = ch.x if i == 0 else ch.acts[i - 1]
            kw = ch._gemm_kwargs(i, L)
            keys.append((i, s))
            graphs.append(capture_graph(lambda: kernels.gemm(a, a.stride(0), L.pw.bt, L.pw.ldbt, batch, L.n, L.k,
                                                             dtype, ch.numeric, L.scheme, ck_rows=L.ck_rows, **kw),
                                        iters))
        for key, tm in zip(keys, interleaved_min_us(graphs, iters)):
            entries[key] = tm
    # the chain's deferred verification runs in the last CTA of its last launch (no extra launch),
    # so a layer's global-ABFT time is its kernel time
    out = {}
    for i in range(n):
        out[(i, Scheme.UNPROTECTED)] = entries[(i, Scheme.UNPROTECTED)] * 1e-6
        out[(i, Scheme.GLOBAL_ABFT)] = entries[(i, Scheme.GLOBAL_ABFT)] * 1e-6
        out[(i, Scheme.THREAD_ONE_SIDED)] = entries[(i, Scheme.THREAD_ONE_SIDED)] * 1e-6
    return MeasuredTimings(entries=out)


def _profile_layers_in_chain(weights, batch, dtype, tiling, iters) -> MeasuredTimings:
    t = D.torch()
    n = len(weights)
    S = Scheme

    def chain_us(schemes):
        nl = len(schemes)
        block = t.zeros(16 * nl + 16, dtype=t.uint8, device="cuda")
        partials = t.zeros((nl, max(1, D.sm_count()), 2), dtype=t.float64, device="cuda")   # as in a ChainGroup
        shared = (block[:16 * nl].view(t.float64).view(nl, 2), block[16 * nl:16 * nl + 8].view(t.int32),
                  block[16 * nl + 8:16 * nl + 12].view(t.int32), partials)
        ch = ProtectedChain(weights, batch, list(schemes), dtype, tiling, shared=shared)
        return graph_time_us(ch.forward, iters)

    base = chain_us([S.UNPROTECTED] * n)
    # split the unprotected chain time over its layers by their standalone kernel times
    alone = profile_layers(weights, batch, dtype, tiling, iters).entries
    un = [alone[(i, S.UNPROTECTED)] for i in range(n)]
    scale = base * 1e-6 / sum(un)
    out = {}
    for i in range(n):
        t_un = un[i] * scale
        out[(i, S.UNPROTECTED)] = t_un
        for s in (S.GLOBAL_ABFT, S.THREAD_ONE_SIDED):
            sch = [S.UNPROTECTED] * n
            sch[i] = s
            out[(i, s)] = max(t_un + (chain_us(sch) - base) * 1e-6, 1e-9)
    return MeasuredTimings(entries=out)
