"""Intensity-guided scheme selection for a whole protected network (configs C3-C5) from B200
measurements ("measure each layer under both schemes").

``profile`` times every linear layer of a ``ProtectedNetwork`` on its real buffers under
unprotected / global / one-sided ABFT (CUDA-graph replayed, CUDA events) and returns the
reference's ``MeasuredTimings`` (cost.py:131-171); ``select_ig`` feeds them to the unchanged
reference ``select`` (cost.py:174-238) and applies the per-layer plan.

T_o (the overhead denominator) is the MINIMUM over the kernel's plans: the
unprotected layer is timed with the planner's tile and with the tiles the protected schemes
use, and the fastest becomes the unprotected configuration — a protected plan can never look
cheaper than the best unprotected one.  The network's one verification launch is measured
and charged to its global layers.
"""

from __future__ import annotations

from typing import Dict

from . import device as D
from . import kernels
from .cost import MeasuredTimings, select
from .profiler import capture_graph, graph_time_us, interleaved_min_us
from .protected_network import GLOBAL_DOT, GLOBAL_FUSED, SELECTABLE, GraphedNetwork, PoolProducer, ProtectedNetwork
from .schemes import Scheme
from .shapes import DeviceProfile


# plan hints tried: none, no k-block pairs, double output staging, both; direct (unstaged) output
# stores; the chunk-split epilogue for narrow tiles; 64-byte-row output stores; per-tap im2col
# instead of halo windows (stride-1 convs); CTA pairs (2-CTA clusters, M = 256 cta_group::2 MMAs),
# alone and over per-tap im2col
PLAN_FLAGS = (0, 1, 4, 5, 8, 16, 512, 2048, 4096, 6144)


def _batched_share(L) -> float:
    """A fused consumer's share (us) of the forward's two batched launches (ProtectedNetwork.fused_batch):
    its producer's border pixels at ~3 TB/s for a 3x3 consumer, plus its window-lhs CTAs."""
    x = L.x
    border_px = x.n * ((2 * x.w + 2 * x.h) if L.r == 3 else 0)
    return border_px * x.cp * 2 / 3e6 + 0.5


def profile(net: ProtectedNetwork, iters: int = 10, best_unprotected: bool = True,
            global_variants: bool = True) -> MeasuredTimings:
    S = Scheme
    out: Dict = {}
    t_ver = graph_time_us(lambda: kernels.verify_partials(net.partials, net.ks, len(net.layers), net.numeric,
                                                          out=net.verdict_buf, detected_count=net.counters[1:2]),
                          iters)
    # what a producer's epilogue pays for accumulating its consumers' window sums (charged to the
    # consumer's fused global variant; measured on the producer's unprotected launch)
    ws_cost = {}
    if global_variants:
        for P in net.producers():
            if isinstance(P, PoolProducer):
                t_off = graph_time_us(P.run, iters)
                P.ws_active = True
                t_on = graph_time_us(P.run, iters)
                P.ws_active = False
            else:
                it = iters if P.flops() < 2e11 else max(3, iters // 3)
                t_off = graph_time_us(lambda: net.launch(P, S.UNPROTECTED), it)
                P.ws_active = True
                P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
                t_on = graph_time_us(lambda: net.launch(P, S.UNPROTECTED), it)
                P.ws_active = False
                P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
            ws_cost[id(P)] = max(0.0, t_on - t_off)
    for L in net.layers:
        it = iters if L.flops() < 2e11 else max(3, iters // 3)
        # every candidate launch of the layer, captured with its own arguments, then timed in
        # interleaved rounds (the same clock / power state for all of them)
        cands = []          # (kind, config, extra_us, graph)

        def add(kind, config, fn, extra=0.0):
            cands.append((kind, config, extra, capture_graph(fn, it)))
        add("thread", None, lambda: net.launch(L, S.THREAD_ONE_SIDED))
        # unprotected: the planner's configuration and every tile / plan-hint alternative
        ucfgs = [(0, 0)]
        if best_unprotected:
            tiles = {net.plan_of(L, s)["tile_n"] for s in (S.GLOBAL_ABFT, S.THREAD_ONE_SIDED)}
            base_tile = net.plan_of(L, S.UNPROTECTED)["tile_n"]
            ucfgs += [(tn, fl) for tn in sorted(tiles - {base_tile}) + [0] for fl in PLAN_FLAGS if (tn, fl) != (0, 0)]
        for tn, fl in ucfgs:
            try:
                net.set_tile(L, S.UNPROTECTED, tn, fl)
            except Exception:     # noqa: BLE001 — a configuration the unprotected plan cannot take
                continue
            add("unprotected", (tn, fl), lambda: net.launch(L, S.UNPROTECTED))
        # global: the lhs source (checksum MMA slice, checksum-warp dot, producer-fused activation
        # checksum + its producer's window-sum cost and its share of the batched launches) x plan hints
        variants = [("slice", S.GLOBAL_ABFT), ("dot", GLOBAL_DOT)] if global_variants else [("slice", S.GLOBAL_ABFT)]
        if global_variants and L.producer is not None:
            variants.append(("fused", GLOBAL_FUSED))
        keep_var = L.gvar
        for var, key in variants:
            extra = ws_cost.get(id(L.producer), 0.0) + _batched_share(L) if var == "fused" else 0.0
            for fl in (PLAN_FLAGS if global_variants else (0,)):
                try:
                    net.set_tile(L, key, 0, fl)
                except Exception:      # noqa: BLE001
                    continue
                L.gvar = var           # (the launch key of the variant; window sums are not needed here)
                add("global", (var, fl), lambda: net.launch(L, S.GLOBAL_ABFT, deferred=True), extra)
                L.gvar = keep_var
        tms = interleaved_min_us([c[3] for c in cands], it)
        times = {}
        best = {}
        for (kind, cfg, extra, _), tm in zip(cands, tms):
            tt = tm + extra
            if kind not in best or tt < best[kind][0]:
                best[kind] = (tt, cfg)
        del cands
        times[S.THREAD_ONE_SIDED] = best["thread"][0]
        times[S.UNPROTECTED], (utn, ufl) = best["unprotected"]
        net.set_tile(L, S.UNPROTECTED, utn, ufl)
        times[S.GLOBAL_ABFT], (gvar, gfl) = best["global"]
        for var, key in variants:
            net.set_tile(L, key, 0, gfl if var == gvar else 0)
        net.set_global_variant(L, gvar)
        out[(L.index, S.UNPROTECTED)] = times[S.UNPROTECTED] * 1e-6
        out[(L.index, S.GLOBAL_ABFT)] = (times[S.GLOBAL_ABFT] + t_ver / len(net.layers)) * 1e-6
        out[(L.index, S.THREAD_ONE_SIDED)] = times[S.THREAD_ONE_SIDED] * 1e-6
    return MeasuredTimings(entries=out)


def select_ig(net: ProtectedNetwork, device: DeviceProfile, measured: MeasuredTimings):
    """The reference selector over the network's layers with B200 timings; applies the plan."""
    plan = select(net.gemm_layers(), net.dtype, device, net.tiling, measured=measured)
    net.set_schemes([lp.chosen for lp in plan.layers])
    return plan


def _forward_ms(graphs, reps: int):
    """Interleaved replays of several captured forwards -> median ms of each."""
    import statistics
    t = D.torch()
    res = [[] for _ in graphs]
    for _ in range(reps):
        for i, g in enumerate(graphs):
            e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            t.cuda.synchronize()
            res[i].append(e0.elapsed_time(e1))
    return [statistics.median(r) for r in res]


def refine_in_network(net: ProtectedNetwork, measured: MeasuredTimings, window: float = 0.08, reps: int = 11,
                      min_gain: float = 5e-3) -> list:
    """In-network A/B of the selector's close calls.  Isolated per-layer timings (each kernel
    replayed alone, its operands L2-warm) favour the thread-level epilogue slightly; where the two
    protected schemes are within `window` of each other, the whole forward is timed with the layer
    under each scheme (interleaved replays, medians) and the faster kept — thread-level only when it
    wins by more than `min_gain` of the forward (ties go to global, cost.py:186).  Returns the
    layers switched."""
    S = Scheme
    switched = []
    cur = GraphedNetwork(net, warmup=1)
    for L in net.layers:
        tg, tt = measured.get(L.index, S.GLOBAL_ABFT), measured.get(L.index, S.THREAD_ONE_SIDED)
        if abs(tt - tg) > window * min(tg, tt):
            continue
        keep = L.scheme
        alt = S.GLOBAL_ABFT if keep is S.THREAD_ONE_SIDED else S.THREAD_ONE_SIDED
        L.scheme = alt
        net._refresh_window_sums()      # a fused global consumer needs its producer's window sums
        g_alt = GraphedNetwork(net, warmup=1)
        t_cur, t_alt = _forward_ms([cur.graph, g_alt.graph], reps)
        # thread-level only when it is faster alone AND in the network; global on ties
        better = (tt < tg and t_alt < t_cur * (1 - min_gain)) if alt is S.THREAD_ONE_SIDED \
            else t_alt <= t_cur * (1 + min_gain)
        if better:
            cur = g_alt
            switched.append((L.index, keep.value, alt.value, round(t_cur, 4), round(t_alt, 4)))
        else:
            L.scheme = keep
            net._refresh_window_sums()
    return switched


def refine_unprotected_in_network(net: ProtectedNetwork, reps: int = 9, min_gain: float = 1e-3) -> list:
    """T_o as the minimum over plans, decided where it counts: where the isolated search (``profile``)
    moved a layer's unprotected launch off the planner's configuration, the all-unprotected forward
    is timed with each of the two (interleaved replays, medians) and the faster kept."""
    S = Scheme
    keep_schemes = net.schemes()
    net.set_schemes(S.UNPROTECTED)
    changed = []
    cur = GraphedNetwork(net, warmup=1, verify=False)
    for L in net.layers:
        chosen = net.config_of(L, S.UNPROTECTED)
        if chosen == (0, 0):
            continue
        net.set_tile(L, S.UNPROTECTED, 0, 0)
        g_def = GraphedNetwork(net, warmup=1, verify=False)
        t_cur, t_def = _forward_ms([cur.graph, g_def.graph], reps)
        if t_def <= t_cur * (1 + min_gain):
            changed.append((L.index, chosen, (0, 0), round(t_cur, 4), round(t_def, 4)))
            cur = g_def
        else:
            net.set_tile(L, S.UNPROTECTED, *chosen)
    net.set_schemes(keep_schemes)
    return changed


def policy_graphs(net: ProtectedNetwork, plan_schemes, verify: bool = True) -> Dict[str, GraphedNetwork]:
    """One captured forward per policy: unprotected / global / thread (always one scheme) and ig."""
    S = Scheme
    pols = {"unprotected": [S.UNPROTECTED] * len(net.layers), "global": [S.GLOBAL_ABFT] * len(net.layers),
            "thread": [S.THREAD_ONE_SIDED] * len(net.layers), "ig": list(plan_schemes)}
    graphs = {}
    for name, sch in pols.items():
        net.set_schemes(sch)
        graphs[name] = GraphedNetwork(net, verify=verify)
    net.set_schemes(plan_schemes)
    return graphs


def capture(fn, warmup: int = 2):
    """fn() captured once in a CUDA graph (after `warmup` eager calls on the capture stream)."""
    t = D.torch()
    s = t.cuda.Stream()
    s.wait_stream(t.cuda.current_stream())
    with t.cuda.stream(s):
        for _ in range(warmup):
            fn()
    t.cuda.current_stream().wait_stream(s)
    t.cuda.synchronize()
    g = t.cuda.CUDAGraph()
    with t.cuda.graph(g, stream=s):
        fn()
    t.cuda.synchronize()
    return g


def device_profile(peaks: dict) -> DeviceProfile:
    return DeviceProfile(name="B200", tensor_throughput=peaks["bf16_tflops"] * 1e12,
                         alu_throughput=148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6,
                         memory_bandwidth=peaks["hbm_gbs"] * 1e9, verification_launch_latency=0.0)


def fold_bn_model(model):
    """A copy of `model` with every Conv2d -> BatchNorm2d pair fused (eval statistics); module
    definition order pairs them in torchvision's ResNet / ShuffleNet blocks and Sequentials."""
    import copy

    import torch.nn as nn
    from torch.nn.utils.fusion import fuse_conv_bn_eval
    m = copy.deepcopy(model).eval()

    def fold(mod):
        names = list(mod._modules)
        for i, nm in enumerate(names):
            child = mod._modules[nm]
            if isinstance(child, nn.Conv2d) and i + 1 < len(names) and \
                    isinstance(mod._modules[names[i + 1]], nn.BatchNorm2d):
                mod._modules[nm] = fuse_conv_bn_eval(child, mod._modules[names[i + 1]])
                mod._modules[names[i + 1]] = nn.Identity()
            elif child is not None:
                fold(child)
    fold(m)
    return m


def vendor_forward(model, batch: int, h: int = 224, w: int = 224):
    """The same network with BN folded (torch.nn.utils.fusion) in fp16 channels_last through
    torch / cuDNN: the vendor denominator beside the unprotected sm_100a pipeline.
    Returns (fn, input) with fn() running one forward."""
    import torch
    m = fold_bn_model(model)
    m = m.half().cuda().to(memory_format=torch.channels_last)
    x = torch.zeros((batch, 3, h, w), dtype=torch.float16, device="cuda").to(memory_format=torch.channels_last)
    torch.backends.cudnn.benchmark = True

    def fn():
        with torch.no_grad():
            return m(x)
    return fn, x
