"""CPU-only checks of the boundary and the host logic (no GPU, no kernel launches).

* the in-tree C-ABI library loads and exports every entry point include/abft_b200.h declares;
* the product path has no CPU fallback: without a GPU it raises instead of computing;
* the product package never imports the oracle;
* host-side logic that mirrors the reference (selector, cost model, roofline, shapes,
  tiling / fault validation, fault localisation, Table-1 op counts) against the
  reference's golden vectors and its own unit-test known answers.
"""

import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "abft_b200.h")
PKG = os.path.join(ROOT, "paper_2104_09455_b200")


def _declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|int64_t|const char\*)\s+(abft_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = _declared_symbols()
    for name in ("abft_gemm", "abft_colsum", "abft_global_verify", "abft_verify_sums", "abft_last_error"):
        assert name in syms, name


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2104_09455_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load()
    missing = [s for s in _declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED_SYMBOLS) == set(_declared_symbols())
    assert lib.abft_version() == 100
    # the ctypes mirrors of the header's structs have the C layout's size
    import ctypes
    for which, cls in enumerate((_lib.GemmArgs, _lib.ConvArgs, _lib.GlobalTask, _lib.VerdictC, _lib.ThreadVerdictC,
                                 _lib.Fault)):
        assert lib.abft_struct_size(which) == ctypes.sizeof(cls), cls.__name__
    # pure host query: no device in this container
    assert lib.abft_device_sms() in (0, 148) or lib.abft_device_sms() > 0


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import _lib
    a = np.ones((8, 8), dtype=np.float16)
    with pytest.raises(_lib.AbftLibraryError):
        P.execute(a, a, P.TilingConfig(), P.Scheme.GLOBAL_ABFT)
    with pytest.raises(_lib.AbftLibraryError):
        P.run_protected_pipeline(a, [a])


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace("oracle of", ""), f


# ----------------------------------------------------------------- selector / cost model
def _select_cases():
    with open(os.path.join(ROOT, "tests", "golden", "select_cases.json")) as fh:
        return json.load(fh)


def _devices(P):
    return {
        "T4": P.DeviceProfile(name="T4", tensor_throughput=65e12, alu_throughput=65e12 / 8, memory_bandwidth=320e9),
        "B200": P.DeviceProfile(name="B200", tensor_throughput=1670.1e12, alu_throughput=74e12,
                                memory_bandwidth=6372.2e9, verification_launch_latency=0.0),
    }


def test_cost_model_matches_reference_golden():
    import paper_2104_09455_b200 as P
    devs = _devices(P)
    n = 0
    for case in _select_cases():
        if case["kind"] != "square":
            continue
        dev = devs[case["device"]]
        shape = P.GemmShape(*case["shape"])
        assert P.base_time(shape, P.BINARY16, dev) == pytest.approx(case["base"], rel=1e-12)
        for name, t in case["times"].items():
            assert P.scheme_time(shape, P.BINARY16, dev, P.Scheme(name)) == pytest.approx(t, rel=1e-12), name
        n += 1
    assert n == 22


def test_selector_matches_reference_golden():
    import paper_2104_09455_b200 as P
    devs = _devices(P)
    n = 0
    for case in _select_cases():
        if case["kind"] != "plan":
            continue
        layers = [(i, P.GemmShape(m, nn, k)) for i, m, nn, k in case["layers"]]
        plan = P.select(layers, P.BINARY16, devs[case["device"]])
        assert [lp.chosen.value for lp in plan.layers] == case["chosen"]
        assert plan.aggregate_base_time == pytest.approx(case["agg_base"], rel=1e-12)
        assert plan.aggregate_protected_time == pytest.approx(case["agg_prot"], rel=1e-12)
        n += 1
    assert n == 20


def test_selector_measured_override_and_ties_to_global():
    import paper_2104_09455_b200 as P
    dev = _devices(P)["B200"]
    layers = [(0, P.GemmShape(64, 64, 64)), (1, P.GemmShape(2048, 2048, 2048))]
    csv_text = ("layer_index,scheme,time_us\n0,unprotected,10\n0,global-abft,12\n0,thread-one-sided,11\n"
                "1,unprotected,100\n1,global-abft,101\n1,thread-one-sided,101\n")
    meas = P.MeasuredTimings.from_csv_text(csv_text)
    plan = P.select(layers, P.BINARY16, dev, measured=meas)
    assert [lp.chosen for lp in plan.layers] == [P.Scheme.THREAD_ONE_SIDED, P.Scheme.GLOBAL_ABFT]
    assert plan.aggregate_overhead_pct == pytest.approx(100 * (11 + 101 - 110) / 110)


def test_crossover_on_t4_profile_is_1280():
    # test_output.txt:25 of the reference: the T4 model crossover S* = 1280
    import paper_2104_09455_b200 as P
    dev = _devices(P)["T4"]
    sizes = [16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 640, 768, 896, 1024, 1280, 1536, 2048, 3072, 4096]
    prefer_global = [P.select([(0, P.GemmShape(s, s, s))], P.BINARY16, dev).layers[0].chosen is P.Scheme.GLOBAL_ABFT
                     for s in sizes]
    flips = sum(1 for a, b in zip(prefer_global, prefer_global[1:]) if a != b)
    assert flips == 1 and sizes[prefer_global.index(True)] == 1280


# ----------------------------------------------------------------- roofline / shapes
def test_roofline_known_answers():
    import paper_2104_09455_b200 as P
    # test_roofline.py:38-41 of the reference
    assert P.arithmetic_intensity(P.GemmShape(2048, 2048, 2048), P.BINARY16) == pytest.approx(682.67, abs=5e-3)
    assert P.arithmetic_intensity(P.GemmShape(32, 32, 32), P.BINARY16) == pytest.approx(10.67, abs=5e-3)
    assert P.gemm_flops(P.GemmShape(2, 3, 4)) == 48
    dev = _devices(P)["T4"]
    assert P.cmr(dev) == pytest.approx(203.1, abs=0.05)


def test_dlrm_aggregate_intensity():
    # test_acceptance.py:70-82: DLRM MLP-Bottom / Top at b1 and b2048, x8 padding
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200.shapes import PaddingPolicy

    def agg(dims, b):
        shapes = [P.pad_gemm(P.GemmShape(b, dims[i + 1], dims[i]), PaddingPolicy.MULTIPLE_OF_8)
                  for i in range(len(dims) - 1)]
        return P.aggregate_intensity(shapes, P.BINARY16)
    assert agg([13, 512, 256, 64], 1) == pytest.approx(7.4, abs=0.05)
    assert agg([512, 512, 256, 1], 1) == pytest.approx(7.7, abs=0.05)
    assert agg([13, 512, 256, 64], 2048) == pytest.approx(92.0, abs=0.05)
    assert agg([512, 512, 256, 1], 2048) == pytest.approx(175.8, abs=0.05)


def test_conv_lowering():
    import paper_2104_09455_b200 as P
    conv = P.ConvLayer(out_channels=64, kernel_h=7, kernel_w=7, stride_h=2, stride_w=2, pad_h=3, pad_w=3)
    assert P.conv_output_shape(224, 224, conv) == (112, 112)
    g = P.layer_to_gemm(1, 224, 224, 3, conv)
    assert (g.m, g.n, g.k) == (112 * 112, 64, 147)


# ----------------------------------------------------------------- tiling / faults
def test_tiling_validation():
    import paper_2104_09455_b200 as P
    P.TilingConfig()
    with pytest.raises(ValueError):
        P.TilingConfig(thread_m=3, warp_m=3, tb_m=3)
    with pytest.raises(ValueError):
        P.TilingConfig(tb_m=100)
    with pytest.raises(ValueError):
        P.TilingConfig(k_step=0)


def test_fault_validation_and_localisation():
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200.schemes import fault_cell, validate_faults
    t64 = P.TilingConfig(tb_m=64, tb_n=64, warp_m=32, warp_n=32, thread_m=16, thread_n=8, k_step=2)
    with pytest.raises(ValueError):
        P.OutputFault(row=0, col=0, delta=0.0)
    shape = P.GemmShape(64, 64, 64)
    with pytest.raises(ValueError):
        validate_faults([P.OutputFault(row=64, col=0, delta=1.0)], shape, t64)
    # ThreadMmaFault(2, 5, step=7, local=11) -> cell (2*16 + 11//8, 5*8 + 11%8)  (tiled.py:386-397)
    f = P.ThreadMmaFault(thread_row=2, thread_col=5, step=7, local_index=11, delta=3.0)
    validate_faults([f], shape, t64)
    assert fault_cell(f, t64)[:2] == (2 * 16 + 1, 5 * 8 + 3)
    with pytest.raises(ValueError):
        validate_faults([P.ThreadMmaFault(thread_row=2, thread_col=5, step=32, local_index=0, delta=1.0)], shape, t64)


def test_op_count_closed_forms():
    # test_tiled.py:261-271 of the reference (64^3, T64 tiling)
    import paper_2104_09455_b200 as P
    t64 = P.TilingConfig(tb_m=64, tb_n=64, warp_m=32, warp_n=32, thread_m=16, thread_n=8, k_step=2)
    g = P.GemmShape(64, 64, 64)
    assert P.count_redundant_ops(P.Scheme.THREAD_ONE_SIDED, t64, g).redundant_mma_count == 8192
    assert P.count_redundant_ops(P.Scheme.THREAD_TWO_SIDED, t64, g).redundant_mma_count == 1024
    assert P.count_redundant_ops(P.Scheme.THREAD_REPLICATION_FULL, t64, g).redundant_mma_count == 65536
    assert P.count_redundant_ops(P.Scheme.GLOBAL_ABFT, t64, g).checksum_op_count == 64 * 64 + 64 + 64 * 64
    # cli check --m 32 --n 32 --k 32 --scheme two-sided (test_output.txt:87-101)
    # -> 32^3 padded to 128x128x32 by the default tiling
    c = P.count_redundant_ops(P.Scheme.THREAD_TWO_SIDED, P.TilingConfig(), P.GemmShape(128, 128, 32))
    assert (c.base_mma_count, c.redundant_mma_count, c.checksum_op_count) == (131072, 2048, 90112)


def test_scheme_names_and_abi_codes():
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import _lib
    from paper_2104_09455_b200.schemes import SCHEME_CODE
    assert [s.value for s in P.Scheme] == ["unprotected", "global-abft", "thread-one-sided", "thread-two-sided",
                                            "thread-replication-full", "thread-replication-single-acc"]
    assert SCHEME_CODE[P.Scheme.GLOBAL_ABFT] == _lib.GLOBAL
    assert SCHEME_CODE[P.Scheme.THREAD_REPLICATION_SINGLE_ACC] == _lib.REPL_SINGLE
    with pytest.raises(ValueError):
        P.Scheme("bogus")


def test_network_layer_lists_reproduce_paper_fig4():
    # PAPER.md:284-291 (Fig 4): aggregate FP16 AI at 1080x1920, batch 1, x8 padding
    pytest.importorskip("torchvision")
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import networks
    from paper_2104_09455_b200.shapes import PaddingPolicy
    fig4 = {"squeezenet1_0": 71.1, "shufflenet_v2_x1_0": 76.6, "resnet50": 122.0, "alexnet": 125.5, "vgg16": 155.5,
            "densenet161": 79.0, "resnext50_32x4d": 220.8, "wide_resnet50_2": 220.8}
    for name, ai in fig4.items():
        layers = networks.capture(name, 1, 1080, 1920)
        agg = P.aggregate_intensity([P.pad_gemm(l.gemm(), PaddingPolicy.MULTIPLE_OF_8) for l in layers], P.BINARY16)
        assert agg == pytest.approx(ai, abs=0.05), name
    assert len(networks.capture("resnet50", 1, 224, 224)) == 54


def test_noscope_layer_lists_reproduce_paper_aggregate_intensity():
    # PAPER.md:679-735 / BASELINE.md 1.2: FP16 aggregate AI of the NoScope CNNs at batch 64, x8 padding;
    # 2-4 conv layers of 16-64 channels, <= 2 FC layers, 50x50 frames
    pytest.importorskip("torchvision")
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import networks, noscope
    from paper_2104_09455_b200.shapes import PaddingPolicy
    for name, ai in noscope.PAPER_AI.items():
        layers = networks.capture(name, noscope.BATCH, noscope.HW, noscope.HW)
        convs = [l for l in layers if l.kind == "conv"]
        fcs = [l for l in layers if l.kind == "fc"]
        assert 2 <= len(convs) <= 4 and len(fcs) <= 2, name
        assert all(16 <= l.oc <= 64 for l in convs), name
        agg = P.aggregate_intensity([P.pad_gemm(l.gemm(), PaddingPolicy.MULTIPLE_OF_8) for l in layers], P.BINARY16)
        assert agg == pytest.approx(ai, abs=0.35), name


def test_fitted_device_profile_recovers_model_choices():
    """calibrate.fit_device_profile: on timings generated by a known device model, the fitted
    profile's model-only choices agree with the measured choices on every layer."""
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import calibrate
    from paper_2104_09455_b200.cost import scheme_time
    truth = P.DeviceProfile(name="truth", tensor_throughput=400e12, alu_throughput=20e12,
                            memory_bandwidth=3000e9, verification_launch_latency=1e-6)
    shapes = [P.GemmShape(m, n, k) for m in (1, 64, 2048, 50176) for n in (64, 512) for k in (16, 512, 2304)]
    S = P.Scheme
    rows = [calibrate.LayerTiming(s, *(scheme_time(s, P.BINARY16, truth, sch) for sch in
                                       (S.UNPROTECTED, S.GLOBAL_ABFT, S.THREAD_ONE_SIDED))) for s in shapes]
    peaks = P.DeviceProfile(name="B200", tensor_throughput=1600e12, alu_throughput=80e12, memory_bandwidth=6000e9,
                            verification_launch_latency=0.0)
    fit = calibrate.fit_device_profile(rows, P.BINARY16, peaks)
    assert fit.agreement == 1.0
    assert fit.model_plan_time == pytest.approx(fit.measured_plan_time)
