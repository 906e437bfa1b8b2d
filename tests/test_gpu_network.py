"""Whole-network protected inference (config C5) on the GPU: every protected conv / FC layer
of a real (BN-folded) torchvision CNN against an fp32 checker of the same layer on the same
input, the network's logits against the torch fp32 forward of the original model, zero false
positives on clean runs under every scheme, and injected faults flagged at exactly the layer
that holds them (deferred verification, checksum.py:198-237; fault model tiled.py:197-200)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NETS = ["resnet50", "vgg16", "squeezenet1_0", "shufflenet_v2_x1_0", "alexnet"]


@pytest.fixture(scope="module")
def PN():
    from paper_2104_09455_b200 import device, protected_network
    device.require_device()
    return protected_network


def _logical(act):
    """Act -> NCHW fp32 tensor of its logical channels."""
    import torch
    idx = torch.as_tensor(act.phys_map(), device=act.buf.device, dtype=torch.long)
    return act.buf.index_select(3, idx).float().permute(0, 3, 1, 2)


def check_layer(L):
    """The layer's output vs torch fp32 conv of ITS input with the fp16-rounded folded weights:
    fp32-accumulation reordering + one fp16 rounding of the output."""
    import torch
    import torch.nn.functional as F
    x = _logical(L.x)
    wq = L.weight.half().float()
    bias = L.bias if L.bias is not None else None
    if L.kind == "fc":
        x = x.reshape(x.shape[0], -1, 1, 1)
    ref = F.conv2d(x, wq, bias, stride=L.stride, padding=L.pad)
    bound = F.conv2d(x.abs(), wq.abs(), None, stride=L.stride, padding=L.pad)
    if bias is not None:
        bound = bound + bias.abs().view(1, -1, 1, 1)
    if L.residual is not None:
        r = _logical(L.residual)
        ref = ref + r
        bound = bound + r.abs()
    if L.relu:
        ref = torch.relu(ref)
    out = _logical(L.out)
    if L.kind == "fc":
        out = out.reshape(ref.shape)
    tol = 2e-5 * bound + ref.abs() * 2.0 ** -10 + 1e-6
    err = (out - ref).abs()
    bad = (err > tol)
    assert not bool(bad.any()), (f"{L.name}: {int(bad.sum())} of {bad.numel()} outside tolerance, "
                                 f"max err {float(err.max()):.3e}, max |ref| {float(ref.abs().max()):.3e}")
    return float((err / (tol)).max())


def _input(batch, seed=0, h=224, w=224):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.rand((batch, 3, h, w), generator=g, device="cuda") * 2 - 1).half()


@pytest.mark.parametrize("name", NETS)
def test_network_layers_logits_and_clean_flags(PN, name):
    import torch
    S = PN.Scheme
    model = PN.build_model(name)
    batch = 2
    net = PN.ProtectedNetwork(model, batch)
    x = _input(batch)
    # reference: the original (unfolded) model in fp32 on the same fp16-rounded input, and the
    # torch fp16 forward as the yardstick for fp16 storage error
    with torch.no_grad():
        ref32 = model.float().cuda()(x.float()).float()
        ref16 = model.half().cuda()(x).float()
    model.float()
    for scheme in (S.UNPROTECTED, S.GLOBAL_ABFT, S.THREAD_ONE_SIDED):
        net.set_schemes(scheme)
        out = net.forward(x).float()
        torch.cuda.synchronize()
        assert net.flags() == (0, 0), (scheme, net.flags())
        for L in net.layers:
            check_layer(L)
        err = float((out - ref32).abs().max().detach())
        err16 = float((ref16 - ref32).abs().max())
        scale = float(ref32.abs().max())
        assert err <= 4 * err16 + 2e-3 * scale, (scheme, err, err16, scale)
        if scheme is S.GLOBAL_ABFT:
            vs = net.verdicts()
            assert all(v is not None and not v.detected for v in vs)
            # lhs and rhs agree far inside tau on clean runs (bias correction exact)
            assert max(abs(v.lhs - v.rhs) / v.tolerance_used for v in vs) < 0.05


@pytest.mark.parametrize("name", ["noscope_coral", "noscope_roundabout", "noscope_taipei", "noscope_amsterdam"])
def test_noscope_networks_at_batch_64(PN, name):
    """The specialised NoScope CNNs (50x50 frames at batch 64): every layer against the
    fp32 checker, logits against the torch fp32 forward, zero false positives under each scheme, and
    a fault in the first conv flagged at that layer only."""
    import torch
    from paper_2104_09455_b200 import noscope
    S = PN.Scheme
    model = PN.build_model(name)
    net = PN.ProtectedNetwork(model, noscope.BATCH, noscope.HW, noscope.HW)
    x = _input(noscope.BATCH, seed=4, h=noscope.HW, w=noscope.HW)
    with torch.no_grad():
        ref32 = model.float().cuda()(x.float()).float()
        ref16 = model.half().cuda()(x).float()
    model.float()
    for scheme in (S.UNPROTECTED, S.GLOBAL_ABFT, S.THREAD_ONE_SIDED):
        net.set_schemes(scheme)
        out = net.forward(x).float()
        torch.cuda.synchronize()
        assert net.flags() == (0, 0), (scheme, net.flags())
        for L in net.layers:
            check_layer(L)
        err = float((out - ref32).abs().max())
        err16 = float((ref16 - ref32).abs().max())
        assert err <= 4 * err16 + 2e-3 * float(ref32.abs().max()), (scheme, err, err16)
    net.set_schemes(S.GLOBAL_ABFT)
    net.forward(x)
    L0 = net.layers[0]
    tau = net.verdicts()[L0.index].tolerance_used
    net.inject({L0.index: [(L0.m // 3, 7, 8.0 * tau + 64.0)]})
    net.forward(x)
    assert [i for i, v in enumerate(net.verdicts()) if v.detected] == [L0.index]
    net.inject({})


@pytest.mark.parametrize("scheme", ["global-abft", "thread-one-sided"])
def test_network_fault_flags_the_right_layer(PN, scheme):
    """A single-element fault in one layer (K < 1024: above that the reference tau of
    checksum.py:143-148 grows with the fault itself) is flagged at that layer only."""
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model("resnet50"), 2, schemes=S(scheme))
    x = _input(2)
    net.forward(x)
    clean = net.verdicts()
    targets = [L for L in net.layers if L.k_ref <= 600 and L.kind == "conv"][:6]
    assert targets
    for L in targets:
        tau = 1.0
        if scheme == "global-abft":
            tau = clean[L.index].tolerance_used
        delta = 8.0 * tau + 64.0
        row, col = (L.m * 3) // 7, (L.oc * 5) // 9
        net.inject({L.index: [(row, col, delta)]})
        net.forward(x)
        fired, flagged = net.flags()
        if scheme == "global-abft":
            vs = net.verdicts()
            got = [i for i, v in enumerate(vs) if v.detected]
            assert got == [L.index], (L.name, got)
            assert flagged == 1 and fired == 0
        else:
            assert fired >= 1 and flagged == 0, (L.name, fired, flagged)
    net.inject({})
    net.forward(x)
    assert net.flags() == (0, 0)


def test_network_real_extents_resnet50_b32(PN):
    """ResNet-50 at batch 32: the stem's explicit-im2col mode, halo-reuse 3x3 layers at
    56x56x64, strided downsamples and the 2048->1000 FC at a real batch, layer by layer."""
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model("resnet50"), 32)
    x = _input(32, seed=1)
    for scheme in (S.GLOBAL_ABFT, S.THREAD_ONE_SIDED):
        net.set_schemes(scheme)
        net.forward(x)
        assert net.flags() == (0, 0)
        for L in net.layers:
            check_layer(L)


def test_network_graph_replay_matches_eager(PN):
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model("squeezenet1_0"), 4, schemes=S.GLOBAL_ABFT)
    x = _input(4, seed=2)
    eager = net.forward(x).clone()
    g = PN.GraphedNetwork(net)
    net.load_input(x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(net.logits(), eager)
    assert net.flags() == (0, 0)


@pytest.mark.parametrize("name,layers", [
    ("resnet50", ["conv1", "layer1.0.conv2", "layer3.0.downsample"]),     # stem (explicit im2col), halo 3x3 56x56x64
    ("vgg16", ["features.2", "features.24", "classifier.0"]),             # conv1_2 at 224^2, a 256-wide tile, FC 25088->4096
])
def test_benchmarked_layers_at_batch_256(PN, name, layers):
    """The layers the bench's dominant kernels run, at the bench's batch 256, against the fp32
    checker, under global and one-sided ABFT: zero false positives, and a fault in the stem /
    first conv is flagged at that layer."""
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model(name), 256)
    x = _input(256, seed=3)
    byname = {L.name: L for L in net.layers}
    for scheme in (S.GLOBAL_ABFT, S.THREAD_ONE_SIDED):
        net.set_schemes(scheme)
        net.forward(x)
        torch.cuda.synchronize()
        assert net.flags() == (0, 0), scheme
        for nm in layers:
            check_layer(byname[nm])
            torch.cuda.empty_cache()
    L0 = byname[layers[0]]
    net.set_schemes(S.GLOBAL_ABFT)
    net.forward(x)
    tau = net.verdicts()[L0.index].tolerance_used
    net.inject({L0.index: [(L0.m - 3, 5, 8.0 * tau + 64.0)]})
    net.forward(x)
    assert [i for i, v in enumerate(net.verdicts()) if v.detected] == [L0.index]


@pytest.mark.parametrize("name", ["vgg16", "resnet50"])
def test_fused_window_checksums(PN, name):
    """Global ABFT with the producer-fused activation checksum: a producer's epilogue
    accumulates window sums of its stored output, the consumer runs only the output summation and
    abft_window_lhs rebuilds colck(im2col(x)) . rowck(B) (+ M * sum(bias)).  Clean runs agree far
    inside tau on every fused layer; a fault in a fused consumer is flagged there and only there,
    and a fault in its producer is flagged at the producer only (the consumer's checksum comes from
    the faulty activation it really reads, as in run_protected_pipeline, checksum.py:207-237)."""
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model(name), 2, schemes=S.GLOBAL_ABFT)
    fused = [L for L in net.layers if L.producer is not None]
    assert len(fused) >= (12 if name == "vgg16" else 20), [L.name for L in fused]
    for L in fused:
        net.set_global_variant(L, "fused")
    assert all(L.producer.ws_active for L in fused)
    x = _input(2, seed=5)
    net.forward(x)
    torch.cuda.synchronize()
    assert net.flags() == (0, 0)
    vs = net.verdicts()
    for L in net.layers:
        check_layer(L)
        v = vs[L.index]
        assert not v.detected and abs(v.lhs - v.rhs) < 0.05 * v.tolerance_used, (L.name, v)
    C = next(L for L in fused if L.k_ref <= 600 and isinstance(L.producer, PN.LinearLayer))
    P = C.producer
    for target in (C, P):
        tau = vs[target.index].tolerance_used
        net.inject({target.index: [(target.m // 2, 3, 8.0 * tau + 64.0)]})
        net.forward(x)
        got = [i for i, v in enumerate(net.verdicts()) if v.detected]
        assert got == [target.index], (target.name, got)
    net.inject({})
    # a consumer fed by a max-pooling glue op (its window sums come from the pool kernel)
    pooled = [L for L in fused if isinstance(L.producer, PN.PoolProducer)]
    assert pooled, "no pool-fed fused consumer"
    Lp = pooled[0]
    tau = vs[Lp.index].tolerance_used
    net.inject({Lp.index: [(Lp.m // 3, 1, 8.0 * tau + 64.0)]})
    net.forward(x)
    assert [i for i, v in enumerate(net.verdicts()) if v.detected] == [Lp.index]
    net.inject({})
    # switching the consumer away from the fused lhs stops the producer's window sums
    net.set_global_variant(C, "slice")
    assert not P.ws_active or any(L.gvar == "fused" for L in net.fused_consumers(P))


@pytest.mark.parametrize("name", ["vgg16", "resnet50"])
def test_per_tap_im2col_plan_flag(PN, name):
    """plan_flags bit 11 (per-tap im2col boxes instead of halo windows on stride-1 convs, a plan the
    profiler times): every layer still matches the fp32 checker under every scheme and global
    variant, clean runs flag nothing, and a fault in a 3x3 layer on that plan is flagged there."""
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model(name), 2)
    x = _input(2, seed=6)
    convs = [L for L in net.layers if L.kind == "conv" and L.r == 3 and L.stride == 1 and L.x.c >= 48]
    assert convs
    for L in convs:
        for key in net.keys_of(L):
            net.set_tile(L, key, 0, 2048)
    for scheme, variant in ((S.UNPROTECTED, None), (S.GLOBAL_ABFT, "slice"), (S.GLOBAL_ABFT, "dot"),
                            (S.GLOBAL_ABFT, "fused"), (S.THREAD_ONE_SIDED, None)):
        net.set_schemes(scheme)
        if variant:
            for L in convs:
                if variant != "fused" or L.producer is not None:
                    net.set_global_variant(L, variant)
        net.forward(x)
        torch.cuda.synchronize()
        assert net.flags() == (0, 0), (scheme, variant, net.flags())
        for L in net.layers:
            check_layer(L)
        if scheme is S.GLOBAL_ABFT:
            vs = net.verdicts()
            assert all(not v.detected and abs(v.lhs - v.rhs) < 0.05 * v.tolerance_used for v in vs), variant
    net.set_schemes(S.GLOBAL_ABFT)
    for L in convs:
        net.set_global_variant(L, "slice")
    net.forward(x)
    # (K <= 600: above ~1024 the reference tau grows with the fault itself, checksum.py:143-148)
    T = [L for L in convs if L.k_ref <= 600][-1]
    tau = net.verdicts()[T.index].tolerance_used
    net.inject({T.index: [(T.m // 5, 2, 8.0 * tau + 64.0)]})
    net.forward(x)
    assert [i for i, v in enumerate(net.verdicts()) if v.detected] == [T.index]
    net.inject({})


@pytest.mark.parametrize("name,pflags", [("vgg16", 4096 | 2048), ("resnet50", 4096 | 2048), ("vgg16", 4096),
                                         ("resnet50", 4096)])
def test_cta_pair_plans_in_network(PN, name, pflags):
    """CTA pairs (plan_flags bit 12) on every layer whose unprotected / global-slice launch takes
    them (3x3 stride-1 convs through per-tap im2col with bit 11, else through paired halo windows):
    layers match the fp32 checker, clean runs flag nothing, a fault in a paired layer is flagged
    there only, and paired producers feed fused consumers their window sums."""
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model(name), 2)
    x = _input(2, seed=7)
    paired = {S.UNPROTECTED: [], S.GLOBAL_ABFT: []}
    for L in net.layers:
        for key in paired:
            try:
                net.set_tile(L, key, 0, pflags)
                paired[key].append(L)
            except Exception:      # noqa: BLE001 — a plan the pairs do not take (stems, strided, thin)
                pass
    assert len(paired[S.UNPROTECTED]) >= 8 and len(paired[S.GLOBAL_ABFT]) >= 8, \
        {k.value: [L.name for L in v] for k, v in paired.items()}
    for scheme in paired:
        net.set_schemes(scheme)
        net.forward(x)
        torch.cuda.synchronize()
        assert net.flags() == (0, 0), scheme
        for L in net.layers:
            check_layer(L)
        if scheme is S.GLOBAL_ABFT:
            vs = net.verdicts()
            assert all(not v.detected and abs(v.lhs - v.rhs) < 0.05 * v.tolerance_used for v in vs)
    T = [L for L in paired[S.GLOBAL_ABFT] if L.k_ref <= 600][-1]
    tau = net.verdicts()[T.index].tolerance_used
    net.inject({T.index: [(T.m // 3, 1, 8.0 * tau + 64.0)]})
    net.forward(x)
    assert [i for i, v in enumerate(net.verdicts()) if v.detected] == [T.index]
    net.inject({})
    # fused consumers: paired producers accumulate window sums in their epilogues
    for L in net.layers:
        if L.producer is not None:
            net.set_tile(L, PN.GLOBAL_FUSED, 0, pflags) if L in paired[S.GLOBAL_ABFT] else None
            net.set_global_variant(L, "fused")
    assert any(P.ws_active and P in paired[S.UNPROTECTED] for P in net.producers() if isinstance(P, PN.LinearLayer))
    net.forward(x)
    torch.cuda.synchronize()
    assert net.flags() == (0, 0)
    vs = net.verdicts()
    for L in net.layers:
        check_layer(L)
        assert not vs[L.index].detected and abs(vs[L.index].lhs - vs[L.index].rhs) < 0.05 * vs[L.index].tolerance_used


@pytest.mark.parametrize("name", ["squeezenet1_0", "shufflenet_v2_x1_0", "resnet50"])
def test_deferred_fused_lhs_batch_all_networks(PN, name):
    """Every fused-eligible consumer on the producer-fused checksum: the forward leaves the border
    buckets and window lhs of all of them to two batched launches after the layers; each layer's lhs
    still equals its output summation far inside tau (no activation was overwritten meanwhile), in
    eager runs and in a replayed graph."""
    import torch
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model(name), 2, schemes=S.GLOBAL_ABFT)
    fused = [L for L in net.layers if L.producer is not None]
    assert fused
    for L in fused:
        net.set_global_variant(L, "fused")
    x = _input(2, seed=9)
    net.forward(x)
    torch.cuda.synchronize()
    assert net.flags() == (0, 0)
    vs = net.verdicts()
    for L in net.layers:
        check_layer(L)
        v = vs[L.index]
        assert not v.detected and abs(v.lhs - v.rhs) < 0.05 * v.tolerance_used, (L.name, v)
    g = PN.GraphedNetwork(net)
    net.load_input(x)
    g.replay()
    torch.cuda.synchronize()
    assert net.flags() == (0, 0)
    vs2 = net.verdicts()
    # (fp32 window sums accumulate by atomics: replays agree to rounding, far inside tau)
    assert all(abs(a.lhs - b.lhs) < 0.05 * a.tolerance_used and not b.detected for a, b in zip(vs, vs2))


def test_profiler_selects_and_applies_plans(PN):
    """netprofile.profile on a small network: every layer gets unprotected / global / one-sided
    timings from interleaved candidate rounds, the chosen variant and plan hints are applied, and
    the IG-selected forward still matches the fp32 checker with zero false positives."""
    import torch
    from paper_2104_09455_b200 import netprofile as NP
    from paper_2104_09455_b200.shapes import DeviceProfile
    S = PN.Scheme
    net = PN.ProtectedNetwork(PN.build_model("squeezenet1_0"), 2)
    x = _input(2, seed=11)
    net.load_input(x)
    net.forward()
    torch.cuda.synchronize()
    meas = NP.profile(net, iters=2)
    for L in net.layers:
        for s in PN.SELECTABLE:
            assert meas.get(L.index, s) > 0, (L.name, s)
        assert meas.get(L.index, S.UNPROTECTED) <= meas.get(L.index, S.GLOBAL_ABFT) * 1.5
    dev = DeviceProfile(name="B200", tensor_throughput=1.65e15, alu_throughput=74e12, memory_bandwidth=6.5e12)
    NP.select_ig(net, dev, meas)
    net.forward(x)
    torch.cuda.synchronize()
    assert net.flags() == (0, 0)
    for L in net.layers:
        check_layer(L)
