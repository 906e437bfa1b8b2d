"""Parity of the sm_100a path against the reference's golden vectors and the oracle.

Bar: exact-int mode is bit-exact (outputs, verdict values, flags); binary16
outputs agree with the fp32-accumulate reference within GEMM_ATOL (summation
order only) and fault flags agree exactly for faults outside [0.5 tau, 2 tau].
"""

import numpy as np
import pytest

from oracle import abft_oracle as O

pytestmark = pytest.mark.gpu

GEMM_RTOL = 2e-5      # fp32-accumulate reordering, relative to sum |a_ik b_kj|
VERDICT_RTOL = 1e-2   # tau values: same formula on lhs/rhs that differ by rounding


@pytest.fixture(scope="module")
def P():
    import paper_2104_09455_b200 as pkg
    from paper_2104_09455_b200 import device
    device.require_device()
    return pkg


def _tiling(P, meta):
    f = meta["tiling_fields"]
    return P.TilingConfig(**f)


def _faults(P, meta):
    out = []
    for f in meta["faults"]:
        if f[0] == "output":
            out.append(P.OutputFault(row=f[1], col=f[2], delta=f[3]))
        else:
            out.append(P.ThreadMmaFault(thread_row=f[1], thread_col=f[2], step=f[3], local_index=f[4], delta=f[5]))
    return out


def _abs_bound(a, b):
    return np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))


def test_execute_golden_cases(P, execute_cases):
    failures = []
    for meta, arr in execute_cases:
        dtype = P.BINARY16 if meta["dtype"] == "binary16" else None
        scheme = P.Scheme(meta["scheme"])
        rep = P.execute(arr["a"], arr["b"], _tiling(P, meta), scheme, _faults(P, meta), dtype)
        name = meta["name"]
        exact = np.issubdtype(arr["a"].dtype, np.integer)
        if exact:
            if not np.array_equal(rep.output, arr["out"]):
                failures.append(f"{name}: output mismatch")
        else:
            bound = _abs_bound(arr["a"], arr["b"])
            err = np.abs(rep.output.astype(np.float64) - arr["out"])
            if not (err <= GEMM_RTOL * bound + 1e-6).all():
                failures.append(f"{name}: output err {err.max()}")
        if rep.detected != meta["detected"]:
            failures.append(f"{name}: detected {rep.detected} vs {meta['detected']}")
        if scheme is P.Scheme.GLOBAL_ABFT:
            v = rep.verdicts[0]
            det, lhs, rhs, tol = meta["global"]
            if v.detected != det:
                failures.append(f"{name}: global flag")
            if exact and (v.lhs, v.rhs, v.tolerance_used) != (lhs, rhs, tol):
                failures.append(f"{name}: global values {(v.lhs, v.rhs)} vs {(lhs, rhs)}")
            if not exact and abs(v.tolerance_used - tol) > VERDICT_RTOL * tol:
                failures.append(f"{name}: global tol {v.tolerance_used} vs {tol}")
        elif scheme is not P.Scheme.UNPROTECTED:
            tv = arr["tv"]
            if len(rep.verdicts) != len(tv):
                failures.append(f"{name}: {len(rep.verdicts)} verdicts vs {len(tv)}")
                continue
            for v, ref in zip(rep.verdicts, tv):
                if (v.thread_row, v.thread_col, v.detected) != (int(ref[0]), int(ref[1]), bool(ref[2])):
                    failures.append(f"{name}: verdict {(v.thread_row, v.thread_col, v.detected)} vs {ref[:3]}")
                    break
                if exact and (v.max_abs_diff, v.tolerance_used) != (ref[3], ref[4]):
                    failures.append(f"{name}: verdict values {(v.max_abs_diff, v.tolerance_used)} vs {ref[3:]}")
                    break
                if not exact and v.detected and abs(v.max_abs_diff - ref[3]) > VERDICT_RTOL * max(ref[3], 1):
                    failures.append(f"{name}: fired diff {v.max_abs_diff} vs {ref[3]}")
                    break
        op = rep.op_counts
        if [op.base_mma_count, op.redundant_mma_count, op.checksum_op_count] != meta["op_counts"]:
            failures.append(f"{name}: op counts")
    assert not failures, "\n".join(failures[:40])


def _exact_fp16_overflow(a0, ws, faults) -> bool:
    """Whether the exact-int pipeline leaves the range the tensor-core path computes exactly
    (device.guard_exact: |values| <= 2048 in fp16 storage, K*max|a|*max|b| < 2**24 in fp32) —
    the reference computes these cases in int64 (checksum.py:65-74); the B200 path raises
    ExactOverflowError instead.  Mirrors checksum.run_protected_pipeline's guards."""
    a = np.asarray(a0, dtype=np.int64)
    if np.abs(a).max() > 2048:
        return True
    for idx, w in enumerate(ws):
        w = np.asarray(w, dtype=np.int64)
        ma, mw = max(int(np.abs(a).max()), 1), max(int(np.abs(w).max()), 1)
        if mw > 2048 or a.shape[1] * ma * mw >= 2 ** 24:
            return True
        c = a @ w
        for r, col, d in faults.get(idx, ()):
            c[int(r), int(col)] += int(d)
        a = np.maximum(c, 0)
        if np.abs(a).max() > 2048:
            return True
    return False


def test_pipeline_golden_cases(P, pipeline_cases):
    """Every golden pipeline case runs; exact-int cases outside the tensor-core exact range must
    raise ExactOverflowError — an explicit, predicted list, never a silent skip."""
    from paper_2104_09455_b200.errors import ExactOverflowError
    ran, skipped = 0, []
    for meta, arr in pipeline_cases:
        ws = [arr[f"w{j}"] for j in range(len(meta["verdicts"]))]
        faults = {int(k): [tuple(x) for x in v] for k, v in meta["faults"].items()}
        P.checksum.clear_weight_checksum_cache()
        expect_overflow = meta["exact"] and _exact_fp16_overflow(arr["a0"], ws, faults)
        if expect_overflow:
            with pytest.raises(ExactOverflowError):
                P.run_protected_pipeline(arr["a0"], ws, dtype=None, faults=faults)
            skipped.append(meta["name"])
            continue
        vs = P.run_protected_pipeline(arr["a0"], ws, dtype=None if meta["exact"] else P.BINARY16, faults=faults)
        ran += 1
        for v, (det, lhs, rhs, tol) in zip(vs, meta["verdicts"]):
            assert v.detected == det, meta["name"]
            if meta["exact"]:
                assert (v.lhs, v.rhs) == (lhs, rhs), meta["name"]
            else:
                assert abs(v.tolerance_used - tol) <= VERDICT_RTOL * tol, meta["name"]
                assert abs(v.lhs - lhs) <= 1e-3 * tol and abs(v.rhs - rhs) <= 1e-3 * tol, meta["name"]
    assert ran + len(skipped) == len(pipeline_cases)
    assert len(skipped) <= 4, skipped          # the golden set's exact cases mostly fit fp16


@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (1, 512, 13), (2048, 512, 512), (300, 200, 1000),
                                   (4096, 4096, 4096)])
def test_unprotected_gemm_matches_torch(P, m, n, k):
    import torch
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = (torch.rand((m, k), generator=g, device="cuda") * 2 - 1).half()
    b = (torch.rand((k, n), generator=g, device="cuda") * 2 - 1).half()
    rep = P.execute(a, b)
    ref = a.float() @ b.float()
    bound = a.float().abs() @ b.float().abs()
    assert ((rep.output - ref).abs() <= GEMM_RTOL * bound + 1e-6).all()


@pytest.mark.parametrize("scheme", ["thread-one-sided", "thread-two-sided", "global-abft"])
@pytest.mark.parametrize("m,n,k", [(2048, 512, 512), (4096, 1024, 768), (8192, 2048, 1000)])
def test_no_false_positives_and_detection_at_scale(P, scheme, m, n, k):
    """Full-size property test (K < 1024 so that r*K < 1 and a fault is detectable)."""
    import torch
    sch = P.Scheme(scheme)
    g = torch.Generator(device="cuda").manual_seed(7)
    a = (torch.rand((m, k), generator=g, device="cuda") - 0.5).half()
    b = (torch.rand((k, n), generator=g, device="cuda") - 0.5).half()
    tiling = P.TilingConfig()
    clean = P.execute(a, b, tiling, sch)
    assert clean.detected is False
    row, col = m // 2 + 3, n // 3 + 1
    if sch is P.Scheme.GLOBAL_ABFT:
        v = clean.verdicts[0]
        lhs = max(abs(v.lhs), abs(v.rhs))
    else:
        v = clean.verdicts[(row // 16) * (n // 8) + col // 8]
        lhs = v.tolerance_used / (2.0 ** -10 * k)        # max(|lhs|,|rhs|,1) of the worst row
    # the tolerance grows with |rhs| (which includes the fault): pick delta well past the fixed point
    rk = 2.0 ** -10 * k
    delta = 3.0 * (rk * (lhs + 64.0)) / (1.0 - rk) + 64.0
    faulty = P.execute(a, b, tiling, sch, [P.OutputFault(row=row, col=col, delta=delta)])
    assert faulty.detected is True
    if sch is not P.Scheme.GLOBAL_ABFT:
        fired = [(v.thread_row, v.thread_col) for v in faulty.verdicts if v.detected]
        assert fired == [(row // 16, col // 8)]
    diff = faulty.output - clean.output
    assert float(diff[row, col]) == pytest.approx(delta, rel=1e-5)
    assert float(diff.abs().sum()) == pytest.approx(delta, rel=1e-5)


def test_reference_tolerance_is_vacuous_for_k_at_least_1024(P):
    """tau = 2^-10 K max(|lhs|,|rhs|,1) >= |delta| once K >= 1024 (checksum.py:143-148):
    no single fault is detectable — on the reference and, by parity, here."""
    import torch
    m, n, k = 1024, 512, 2304
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    for sch in (P.Scheme.THREAD_ONE_SIDED, P.Scheme.GLOBAL_ABFT):
        for delta in (1.0, 1e3, 1e6):
            rep = P.execute(a, b, P.TilingConfig(), sch, [P.OutputFault(row=5, col=7, delta=delta)])
            assert rep.detected is False


@pytest.mark.parametrize("source", ["onchip", "offline", "aug"])
@pytest.mark.parametrize("tiling", [dict(thread_m=16, thread_n=8), dict(thread_m=6, thread_n=6, warp_m=24, warp_n=24,
                                                                        tb_m=48, tb_n=48, k_step=3),
                                    dict(thread_m=32, thread_n=16, warp_m=64, warp_n=64)])
def test_checksum_sources_agree(P, source, tiling):
    """On-chip and offline checksum rows give the same verdicts (same fp32 sum order)."""
    rng = np.random.default_rng(11)
    a = rng.integers(-8, 9, size=(700, 200), dtype=np.int64)
    b = rng.integers(-8, 9, size=(200, 300), dtype=np.int64)
    t = P.TilingConfig(**tiling)
    faults = [P.OutputFault(row=5, col=7, delta=3), P.OutputFault(row=650, col=290, delta=-11)]
    out_ref, v_ref = O.execute(a, b, O.Tiling(tb_m=t.tb_m, tb_n=t.tb_n, thread_m=t.thread_m, thread_n=t.thread_n,
                                              k_step=t.k_step), "thread-one-sided",
                               [("output", 5, 7, 3), ("output", 650, 290, -11)])
    for scheme in (P.Scheme.THREAD_ONE_SIDED, P.Scheme.THREAD_TWO_SIDED):
        rep = P.execute(a, b, t, scheme, faults, ck_source=source)
        assert np.array_equal(rep.output, out_ref)
        fired = [(v.thread_row, v.thread_col) for v in rep.verdicts if v.detected]
        assert fired == [(v.thread_row, v.thread_col) for v in v_ref if v.detected]
    xf = rng.uniform(-1, 1, size=(600, 320)).astype(np.float16)
    wf = rng.uniform(-1, 1, size=(320, 256)).astype(np.float16)
    r1 = P.execute(xf, wf, t, P.Scheme.THREAD_ONE_SIDED, ck_source="onchip")
    r2 = P.execute(xf, wf, t, P.Scheme.THREAD_ONE_SIDED, ck_source="offline" if source == "onchip" else source)
    assert [(v.detected, v.max_abs_diff, v.tolerance_used) for v in r1.verdicts] == \
           [(v.detected, v.max_abs_diff, v.tolerance_used) for v in r2.verdicts]


def test_bf16_path(P):
    import torch
    a = (torch.rand((512, 384), device="cuda") - 0.5).bfloat16()
    b = (torch.rand((384, 256), device="cuda") - 0.5).bfloat16()
    rep = P.execute(a, b, P.TilingConfig(), P.Scheme.THREAD_ONE_SIDED)
    ref = a.float() @ b.float()
    bound = a.float().abs() @ b.float().abs()
    assert ((rep.output - ref).abs() <= GEMM_RTOL * bound + 1e-6).all()
    assert rep.detected is False


def test_checksum_helpers_match_oracle(P):
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, size=(300, 72)).astype(np.float16)
    b = rng.uniform(-1, 1, size=(72, 40)).astype(np.float16)
    assert np.allclose(P.column_checksum(a), O.colck(a), rtol=1e-5, atol=1e-4)
    assert np.allclose(P.row_checksum(b), O.rowck(b), rtol=1e-5, atol=1e-4)
    ai = rng.integers(-8, 9, size=(50, 30), dtype=np.int64)
    assert P.column_checksum(ai).tolist() == O.colck(ai).tolist()
    assert P.checksum_dot(np.array([4, 6]), np.array([3, 7])) == 54
    c = O.matmul(ai, ai.T[:, :20].copy() if False else rng.integers(-8, 9, size=(30, 20), dtype=np.int64))
    assert P.output_summation(c) == O.total(c)
    v = P.global_abft_check(np.array([[1, 2], [3, 4]]), np.array([[5, 6], [7, 8]]), np.array([[19, 22], [43, 50]]))
    assert v.detected is False and v.lhs == 134 and v.rhs == 134


def test_shape_errors_map_to_reference_exceptions(P):
    from paper_2104_09455_b200.errors import ShapeMismatchError
    with pytest.raises(ShapeMismatchError):
        P.execute(np.ones((4, 5), dtype=np.int64), np.ones((4, 5), dtype=np.int64))
    with pytest.raises(ValueError):
        P.execute(np.ones((16, 16), dtype=np.int64), np.ones((16, 16), dtype=np.int64), P.TilingConfig(),
                  P.Scheme.GLOBAL_ABFT, [P.OutputFault(row=16, col=0, delta=1)])


@pytest.mark.parametrize("m,n,k", [(700, 300, 200), (1, 512, 13), (300, 1000, 72), (2048, 512, 512)])
def test_global_lhs_variants_agree(P, m, n, k):
    """Global lhs from the checksum N-slice (appended or separate checksum rows) and from the
    checksum warps' dot of the staged A tiles with rowck(B): exact-int verdict values equal the
    oracle's (colck(A) . rowck(B) and the output summation, checksum.py:108-127)."""
    rng = np.random.default_rng(m + n + k)
    a = rng.integers(-8, 9, size=(m, k), dtype=np.int64)
    b = rng.integers(-8, 9, size=(k, n), dtype=np.int64)
    fr = [("output", m // 2, n - 1, 13)]
    out_ref, v_ref = O.execute(a, b, O.Tiling(), "global-abft", fr)
    faults = [P.OutputFault(row=m // 2, col=n - 1, delta=13)]
    for src in ("aug", "offline", "dot", "auto"):
        rep = P.execute(a, b, P.TilingConfig(), P.Scheme.GLOBAL_ABFT, faults, ck_source=src)
        assert np.array_equal(rep.output, out_ref), src
        v = rep.verdicts[0]
        assert (v.detected, v.lhs, v.rhs, v.tolerance_used) == \
            (v_ref[0].detected, v_ref[0].lhs, v_ref[0].rhs, v_ref[0].tolerance_used), src
    # binary16: the dot and the slice agree to fp32-accumulation rounding, no false positive
    af = rng.uniform(-1, 1, size=(m, k)).astype(np.float16)
    bf = rng.uniform(-1, 1, size=(k, n)).astype(np.float16)
    r1 = P.execute(af, bf, P.TilingConfig(), P.Scheme.GLOBAL_ABFT, ck_source="aug")
    r2 = P.execute(af, bf, P.TilingConfig(), P.Scheme.GLOBAL_ABFT, ck_source="dot")
    assert r1.detected is False and r2.detected is False
    assert r1.verdicts[0].rhs == pytest.approx(r2.verdicts[0].rhs, rel=1e-6, abs=1e-6)
    assert r1.verdicts[0].lhs == pytest.approx(r2.verdicts[0].lhs, rel=1e-4, abs=1e-3)


@pytest.mark.parametrize("scheme", ["global-abft", "thread-one-sided", "thread-two-sided"])
@pytest.mark.parametrize("m,n,k", [(700, 600, 300), (300, 256, 1000)])
def test_augmented_weights_with_full_width_tile(P, scheme, m, n, k):
    """tile_n = 256 with augmented weights: the checksum rows no longer fit the one MMA
    (N <= 256), so they come by their own box into their own N-slice (single-buffered
    accumulator).  Exact-int outputs and verdicts equal the oracle's."""
    rng = np.random.default_rng(m * 3 + n + k)
    a = rng.integers(-8, 9, size=(m, k), dtype=np.int64)
    b = rng.integers(-8, 9, size=(k, n), dtype=np.int64)
    fr = [("output", m - 2, n - 3, -9), ("output", 17, 255, 4)]
    out_ref, v_ref = O.execute(a, b, O.Tiling(), scheme, fr)
    faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in fr]
    rep = P.execute(a, b, P.TilingConfig(), P.Scheme(scheme), faults, ck_source="aug", tile_n=256)
    assert np.array_equal(rep.output, out_ref)
    if scheme == "global-abft":
        v = rep.verdicts[0]
        assert (v.detected, v.lhs, v.rhs) == (v_ref[0].detected, v_ref[0].lhs, v_ref[0].rhs)
    else:
        assert [(v.thread_row, v.thread_col) for v in rep.verdicts if v.detected] == \
            [(v.thread_row, v.thread_col) for v in v_ref if v.detected]
        assert len([v for v in rep.verdicts if v.detected]) == 2


@pytest.mark.parametrize("scheme", ["unprotected", "global-abft", "thread-one-sided"])
@pytest.mark.parametrize("m,n,k", [(300, 200, 1000), (2048, 64, 576), (130, 120, 136)])
def test_kblock_pairs_match_single_kblock_stages(P, monkeypatch, scheme, m, n, k):
    """Pipeline stages of two k-blocks (default for narrow tiles; odd k-block counts end with a
    single one) and single k-block stages (ABFT_KPAIR=0) give the oracle's exact-int results."""
    rng = np.random.default_rng(m + 7 * n + k)
    a = rng.integers(-8, 9, size=(m, k), dtype=np.int64)
    b = rng.integers(-8, 9, size=(k, n), dtype=np.int64)
    fr = [("output", m - 1, n // 2, 5)] if scheme != "unprotected" else []
    out_ref, v_ref = O.execute(a, b, O.Tiling(), scheme, fr)
    faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in fr]
    for kp in ("0", "2"):
        monkeypatch.setenv("ABFT_KPAIR", kp)
        rep = P.execute(a, b, P.TilingConfig(), P.Scheme(scheme), faults)
        assert np.array_equal(rep.output, out_ref), kp
        assert rep.detected == any(v.detected for v in v_ref), kp


@pytest.mark.parametrize("scheme", ["unprotected", "global-abft"])
@pytest.mark.parametrize("m,n,k", [(700, 300, 200), (300, 256, 1000), (2048, 64, 576), (130, 120, 136),
                                   (1, 512, 13), (4096, 512, 320)])
def test_cta_pairs_match_oracle(P, scheme, m, n, k):
    """CTA pairs (plan_flags bit 12): 2-CTA clusters running one M = 256 cta_group::2 MMA per
    k-step, each CTA staging its own 128 A rows and half of the B rows (odd M-block counts end with
    an out-of-range tile).  Exact-int outputs and global verdicts equal the oracle's, with a fault;
    binary16 outputs equal the single-CTA kernel's."""
    rng = np.random.default_rng(m + 5 * n + k)
    a = rng.integers(-8, 9, size=(m, k), dtype=np.int64)
    b = rng.integers(-8, 9, size=(k, n), dtype=np.int64)
    fr = [("output", m - 1, n // 2, 5)] if scheme != "unprotected" else []
    out_ref, v_ref = O.execute(a, b, O.Tiling(), scheme, fr)
    faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in fr]
    # (global with tile_n 256: the checksum rows by their own half boxes into their own pair slice)
    for tn in ((0, 256) if scheme == "global-abft" and n >= 256 else (0,)):
        rep = P.execute(a, b, P.TilingConfig(), P.Scheme(scheme), faults, plan_flags=4096, tile_n=tn)
        assert np.array_equal(rep.output, out_ref), tn
        if scheme == "global-abft":
            v = rep.verdicts[0]
            assert (v.detected, v.lhs, v.rhs) == (v_ref[0].detected, v_ref[0].lhs, v_ref[0].rhs), tn
            assert v.detected
    af = rng.uniform(-1, 1, size=(m, k)).astype(np.float16)
    bf = rng.uniform(-1, 1, size=(k, n)).astype(np.float16)
    r1 = P.execute(af, bf, P.TilingConfig(), P.Scheme(scheme), plan_flags=4096)
    r0 = P.execute(af, bf, P.TilingConfig(), P.Scheme(scheme))
    assert np.allclose(np.asarray(r1.output), np.asarray(r0.output), rtol=1e-5, atol=1e-5)
    assert r1.detected is False
