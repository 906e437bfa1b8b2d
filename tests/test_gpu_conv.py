"""Parity of the implicit-GEMM convolution path (TMA im2col) against the oracle.

The reference checks a conv as the GEMM of its im2col lowering (shapes.py:156-180); the
oracle restates that lowering (im2col_nhwc, K ordered (r, s, c)) and runs the reference
execute / global check on it.  Bar: exact-int bit-exact (outputs, verdict values, flags);
binary16 outputs within the fp32-accumulate reordering bound, flags identical for faults
far outside tau.
"""

import numpy as np
import pytest

from oracle import abft_oracle as O

pytestmark = pytest.mark.gpu

GEMM_RTOL = 2e-5

# (n, h, w, c, oc, r, s, stride, pad): every A-load mode of the kernel
CASES = [
    (2, 20, 22, 3, 64, 7, 7, 2, 3),      # ResNet stem: gathered (tap, 4-channel) A tiles (mode 5)
    (2, 17, 19, 3, 64, 3, 3, 1, 1),      # VGG stem (mode 5, one k-block)
    (3, 15, 13, 3, 24, 3, 3, 2, 1),      # ShuffleNet stem: N = 24 (mode 5, 32-wide tile)
    (1, 23, 21, 3, 96, 7, 7, 2, 0),      # SqueezeNet stem: N = 96, no padding (mode 5)
    (2, 13, 11, 64, 48, 3, 3, 1, 1),     # 64-channel chunks, SW128 (mode 1)
    (3, 9, 10, 16, 40, 3, 3, 2, 1),      # strided, 8-channel columns
    (2, 12, 12, 32, 24, 1, 1, 1, 0),     # pointwise = plain GEMM of the NHWC matrix (mode 0)
    (2, 14, 14, 64, 32, 1, 1, 2, 0),     # strided pointwise (downsample) through im2col
    (1, 35, 33, 3, 16, 11, 11, 4, 2),    # AlexNet stem geometry
    (2, 9, 9, 24, 136, 5, 5, 1, 2),      # several 8-channel chunks per tap, N > one CTA tile
    (1, 8, 8, 128, 64, 3, 3, 1, 1),      # two 64-channel chunks per tap
    # halo reuse (mode 4): stride 1 and Q divisible into 64..128-pixel row tiles
    (1, 6, 64, 64, 48, 3, 3, 1, 1),      # Qt = 64
    (2, 5, 112, 96, 80, 3, 3, 1, 1),     # Qt = 112 (16 junk MMA rows), C = 96 -> 2 zero-padded chunks
    (1, 4, 128, 64, 32, 5, 5, 1, 2),     # Qt = 128, 5x5 taps
    (1, 3, 96, 64, 144, 3, 3, 1, 1),     # Qt = 96, two N tiles
]


@pytest.fixture(scope="module")
def P():
    import paper_2104_09455_b200 as pkg
    from paper_2104_09455_b200 import device
    device.require_device()
    return pkg


def _data(case, exact, seed=0):
    n, h, w, c, oc, r, s, st, pd = case
    rng = np.random.default_rng(seed)
    if exact:
        x = rng.integers(-3, 4, size=(n, h, w, c)).astype(np.int64)
        wt = rng.integers(-3, 4, size=(oc, c, r, s)).astype(np.int64)
    else:
        x = rng.uniform(-1, 1, size=(n, h, w, c)).astype(np.float16)
        wt = rng.uniform(-1, 1, size=(oc, c, r, s)).astype(np.float16)
    cols = O.im2col_nhwc(x, r, s, st, pd)
    wmat = np.ascontiguousarray(wt.transpose(2, 3, 1, 0).reshape(r * s * c, oc))
    return x, wt, cols, wmat


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme", ["unprotected", "global-abft", "thread-one-sided"])
def test_conv_exact_int_bit_exact(P, case, scheme):
    n, h, w, c, oc, r, s, st, pd = case
    x, wt, cols, wmat = _data(case, exact=True)
    tiling = P.TilingConfig()
    m = cols.shape[0]
    faults_ref = [("output", m // 2, oc - 1, 5)] if scheme != "unprotected" else []
    faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in faults_ref]
    rep = P.conv2d(x, wt, stride=st, padding=pd, tiling=tiling, scheme=P.Scheme(scheme), faults=faults)
    out, verdicts = O.execute(cols, wmat, O.Tiling(), scheme, faults_ref)
    assert rep.output.shape == (n, (h + 2 * pd - r) // st + 1, (w + 2 * pd - s) // st + 1, oc)
    assert np.array_equal(rep.output.reshape(m, oc), out)
    assert (rep.shape.m, rep.shape.n, rep.shape.k) == (m, oc, c * r * s)
    if scheme == "global-abft":
        v, rv = rep.verdicts[0], verdicts[0]
        assert (v.detected, v.lhs, v.rhs, v.tolerance_used) == (rv.detected, rv.lhs, rv.rhs, rv.tolerance_used)
    elif scheme == "thread-one-sided":
        got = [(v.thread_row, v.thread_col, v.detected) for v in rep.verdicts]
        ref = [(v.thread_row, v.thread_col, v.detected) for v in verdicts]
        assert got == ref
    assert rep.detected == any(v.detected for v in verdicts)


@pytest.mark.parametrize("case", CASES)
def test_conv_binary16_outputs_and_flags(P, case):
    x, wt, cols, wmat = _data(case, exact=False, seed=1)
    n, h, w, c, oc, r, s, st, pd = case
    m = cols.shape[0]
    ref_out, _ = O.execute(cols, wmat, O.Tiling(), "unprotected", [], "binary16")
    bound = np.abs(cols.astype(np.float64)) @ np.abs(wmat.astype(np.float64))
    for scheme in ("unprotected", "global-abft", "thread-one-sided"):
        rep = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme(scheme), dtype=P.BINARY16)
        err = np.abs(rep.output.reshape(m, oc).astype(np.float64) - ref_out)
        assert (err <= GEMM_RTOL * bound + 1e-6).all(), scheme
        assert rep.detected is False, scheme          # zero false positives on clean runs
    # a fault far above tau is flagged by both schemes, at the same thread tile as the oracle
    g = O.global_check(cols, wmat, ref_out, "binary16")
    delta = float(50 * g.tolerance_used + 1)
    row, col = m - 1, oc // 2
    for scheme in ("global-abft", "thread-one-sided"):
        rep = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme(scheme),
                       faults=[P.OutputFault(row=row, col=col, delta=delta)], dtype=P.BINARY16)
        _, ref_v = O.execute(cols, wmat, O.Tiling(), scheme, [("output", row, col, delta)], "binary16")
        # the reference tau 2^-10 * K * max(|lhs|, |rhs|, 1) (global AND per-row) cannot fire for K >= 1024
        assert rep.detected == any(v.detected for v in ref_v)
        if c * r * s < 1024:
            assert rep.detected is True
        if scheme == "thread-one-sided":
            assert [(v.thread_row, v.thread_col) for v in rep.verdicts if v.detected] == \
                [(v.thread_row, v.thread_col) for v in ref_v if v.detected]


def test_conv_colck_is_the_im2col_column_sum(P):
    import torch
    from paper_2104_09455_b200 import conv as C, kernels
    for case in CASES:
        n, h, w, c, oc, r, s, st, pd = case
        x, wt, cols, _ = _data(case, exact=True, seed=2)
        xd = C.upload_nhwc(x, P.EXACT_INT)
        geom = C.geometry(xd, r, s, st, pd, c)
        out = torch.empty(r * s * xd.shape[3], dtype=torch.float32, device="cuda")
        kernels.conv_colck(xd, geom, P.EXACT_INT, out)
        ref = O.colck(O.im2col_nhwc(np.pad(x, ((0, 0), (0, 0), (0, 0), (0, xd.shape[3] - c))), r, s, st, pd))
        assert np.array_equal(out.cpu().numpy().astype(np.int64), ref), case


@pytest.mark.parametrize("case", CASES)
def test_conv_global_fused_and_standalone_checksums_agree(P, case):
    """The in-kernel activation checksum (from the staged A tiles) equals the standalone pass."""
    n, h, w, c, oc, r, s, st, pd = case
    x, wt, cols, wmat = _data(case, exact=True, seed=3)
    m = cols.shape[0]
    for faults in ([], [P.OutputFault(row=m // 3, col=1, delta=7)]):
        b = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme.GLOBAL_ABFT, faults=faults,
                     colck_source="standalone")
        vb = b.verdicts[0]
        assert vb.detected == bool(faults)
        # checksum N-slice, checksum-warp dot with rowck(B), and the default choice between them
        for src in ("slice", "dot", "fused"):
            a = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme.GLOBAL_ABFT, faults=faults, colck_source=src)
            va = a.verdicts[0]
            assert (va.detected, va.lhs, va.rhs) == (vb.detected, vb.lhs, vb.rhs), src
            assert np.array_equal(a.output, b.output), src


@pytest.mark.parametrize("mode", ["1", "2", "3", "4"])
def test_conv_every_a_load_mode_bit_exact(P, mode, monkeypatch):
    """Each A-load mode (64-channel TMA im2col, 8-channel TMA im2col, explicit im2col) on the
    same non-pointwise cases gives the oracle's exact-int outputs and verdicts."""
    monkeypatch.setenv("ABFT_CONV_MODE", mode)
    for case in CASES:
        n, h, w, c, oc, r, s, st, pd = case
        if r == 1 and s == 1 and st == 1 and pd == 0:
            continue
        x, wt, cols, wmat = _data(case, exact=True, seed=4)
        m = cols.shape[0]
        for scheme in ("unprotected", "global-abft", "thread-one-sided"):
            faults_ref = [("output", m - 1, 0, 9)] if scheme != "unprotected" else []
            faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in faults_ref]
            out, verdicts = O.execute(cols, wmat, O.Tiling(), scheme, faults_ref)
            for src in (("slice", "dot") if scheme == "global-abft" else ("fused",)):
                rep = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme(scheme), faults=faults,
                               colck_source=src)
                assert np.array_equal(rep.output.reshape(m, oc), out), (mode, case, scheme, src)
                assert rep.detected == any(v.detected for v in verdicts), (mode, case, scheme, src)
                if scheme == "global-abft":
                    v, rv = rep.verdicts[0], verdicts[0]
                    assert (v.lhs, v.rhs) == (rv.lhs, rv.rhs), (mode, case, src)


@pytest.mark.parametrize("case", [(1, 6, 64, 64, 256, 3, 3, 1, 1),      # halo (Qt = 64), N = one 256 tile
                                  (2, 7, 9, 64, 300, 3, 3, 1, 1),       # 64-channel im2col, two N tiles
                                  (2, 12, 12, 32, 260, 1, 1, 1, 0)])    # pointwise
@pytest.mark.parametrize("scheme", ["global-abft", "thread-one-sided"])
@pytest.mark.parametrize("faulted", [True, False])
def test_conv_full_width_tile_checksum_slice(P, case, scheme, faulted):
    """tile_n = 256: the checksum rows of the augmented weights go through their own box and
    MMA N-slice (ck_mode 4), in every A-load mode.  Exact-int parity with the oracle.  Without
    faults (and with 16-bit outputs, below) the global scheme runs the lean epilogue with the
    split accumulator tail (columns 240..255 + the checksum slice in a shared TMEM tail)."""
    n, h, w, c, oc, r, s, st, pd = case
    x, wt, cols, wmat = _data(case, exact=True, seed=5)
    m = cols.shape[0]
    fr = [("output", m - 1, oc - 1, 6), ("output", 3, 130, -2)] if faulted else []
    faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in fr]
    rep = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme(scheme), faults=faults, tile_n=256)
    out, verdicts = O.execute(cols, wmat, O.Tiling(), scheme, fr)
    assert np.array_equal(rep.output.reshape(m, oc), out)
    if scheme == "global-abft":
        v, rv = rep.verdicts[0], verdicts[0]
        assert (v.detected, v.lhs, v.rhs) == (rv.detected, rv.lhs, rv.rhs)
    else:
        assert [(v.thread_row, v.thread_col) for v in rep.verdicts if v.detected] == \
            [(v.thread_row, v.thread_col) for v in verdicts if v.detected]


@pytest.mark.parametrize("flags", [0, 512])
def test_gemm_full_width_global_lean_exact(P, flags):
    """Global ABFT on a 256-wide tile with 16-bit outputs (the lean epilogue, the 272-column
    accumulator with its own checksum N-slice), with 128-byte-row and (plan_flags bit 9) 64-byte-row
    bulk stores: the exact outputs and the exact global lhs / rhs of the reference
    (checksum.py:108-127)."""
    import torch
    from paper_2104_09455_b200 import _lib, kernels
    from paper_2104_09455_b200 import device as D
    rng = np.random.default_rng(7)
    m, n, k = 777, 512, 192
    a = rng.integers(-3, 4, size=(m, k)).astype(np.int64)
    b = rng.integers(-3, 4, size=(k, n)).astype(np.int64)
    ad = torch.from_numpy(a.astype(np.float16)).cuda()
    pw = D.prepare_weight(torch.from_numpy(b.astype(np.float16)).cuda(), P.EXACT_INT)
    out = torch.zeros((m, n), dtype=torch.float16, device="cuda")
    sums = torch.zeros(2, dtype=torch.float64, device="cuda")
    kw = dict(out=out, ldc=n, out_kind="f16", out_sum=sums[1:2], out_lhs=sums[0:1], tile_n=256, plan_flags=flags)
    plan = kernels.gemm(ad, k, pw.bt, pw.ldbt, m, n, k, P.EXACT_INT, _lib.NUM_EXACT, P.Scheme.GLOBAL_ABFT,
                        plan_only=True, ck_layout=1, **kw)
    kw["ck_rows"] = kernels.global_ck_rows(pw.bt, n, k, P.EXACT_INT, plan)
    kernels.gemm(ad, k, pw.bt, pw.ldbt, m, n, k, P.EXACT_INT, _lib.NUM_EXACT, P.Scheme.GLOBAL_ABFT, **kw)
    torch.cuda.synchronize()
    c = a @ b
    assert np.array_equal(out.float().cpu().numpy().astype(np.int64), c)
    lhs, rhs = sums.cpu().numpy()
    assert int(round(rhs)) == int(c.sum())
    assert int(round(lhs)) == int(a.sum(axis=0) @ b.sum(axis=1))


@pytest.mark.parametrize("depth", [3, 5, 7])
def test_gathered_stem_copy_depths_bit_exact(P, depth):
    """The gathered stem (a_mode 5) with 3, 5 and 7 k-blocks of copies in flight (plan_flags bits
    6-8): exact-int outputs and global verdict values equal the oracle's."""
    from paper_2104_09455_b200 import conv as C
    case = (2, 20, 22, 3, 64, 7, 7, 2, 3)
    n, h, w, c, oc, r, s, st, pd = case
    x, wt, cols, wmat = _data(case, exact=True, seed=9)
    out, verdicts = O.execute(cols, wmat, O.Tiling(), "global-abft", [])
    rep = C.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme.GLOBAL_ABFT, plan_flags=depth << 6)
    assert np.array_equal(rep.output.reshape(cols.shape[0], oc), out)
    v, rv = rep.verdicts[0], verdicts[0]
    assert (v.detected, v.lhs, v.rhs) == (rv.detected, rv.lhs, rv.rhs)


@pytest.mark.parametrize("n,h,w,c,ld", [(3, 28, 28, 512, 512), (5, 1, 7, 64, 72), (2, 2, 1, 8, 8), (4, 56, 56, 64, 64),
                                        (7, 13, 9, 24, 32), (1, 224, 224, 64, 64)])
def test_border_sums_buckets(n, h, w, c, ld):
    """abft_nhwc_border_sums: buckets 1..8 (rows 0 / H-1, columns 0 / W-1, the four corners) of the
    activation's border pixels, accumulated onto wsum (bucket 0 untouched), against fp64 sums."""
    import torch
    from paper_2104_09455_b200 import BINARY16, kernels
    g = torch.Generator(device="cuda").manual_seed(n * h + w)
    x = (torch.rand((n, h, w, ld), generator=g, device="cuda") * 2 - 1).half()
    wsum = torch.ones((9, c + 8), dtype=torch.float32, device="cuda")
    kernels.border_sums(x, n, h, w, c, ld, BINARY16, wsum, c + 8)
    torch.cuda.synchronize()
    xd = x[..., :c].double()
    want = [xd[:, 0].sum((0, 1)), xd[:, -1].sum((0, 1)), xd[:, :, 0].sum((0, 1)), xd[:, :, -1].sum((0, 1)),
            xd[:, 0, 0].sum(0), xd[:, 0, -1].sum(0), xd[:, -1, 0].sum(0), xd[:, -1, -1].sum(0)]
    got = wsum.double()
    assert torch.equal(got[0], torch.ones_like(got[0]))
    for b, ref in enumerate(want):
        err = (got[b + 1, :c] - 1.0 - ref).abs().max().item()
        assert err <= 1e-5 * (1 + n * max(h, w)), (b + 1, err)
        assert torch.equal(got[b + 1, c:], torch.ones_like(got[b + 1, c:]))


@pytest.mark.parametrize("case", [(2, 9, 64, 64, 64, 3, 3, 1, 1),       # halo windows, Qt = 64, N = 64
                                  (3, 6, 112, 64, 128, 3, 3, 1, 1),     # Qt = 112 (partial quadrant), N = 128
                                  (1, 5, 80, 128, 96, 3, 3, 1, 1),      # two 64-channel chunks, odd tile count
                                  (2, 11, 13, 64, 200, 3, 3, 1, 1),     # no halo tile: per-tap im2col
                                  (2, 12, 12, 64, 48, 1, 1, 1, 0)])     # pointwise
@pytest.mark.parametrize("flags", [4096, 4096 | 2048])
def test_conv_cta_pairs_exact(P, case, flags):
    """CTA pairs on the conv A-load modes (halo windows with resident or streamed weights, per-tap
    im2col, pointwise): exact-int outputs and global verdicts equal the oracle's, faults flagged."""
    n, h, w, c, oc, r, s, st, pd = case
    x, wt, cols, wmat = _data(case, exact=True, seed=8)
    m = cols.shape[0]
    for scheme in ("unprotected", "global-abft"):
        fr = [("output", m - 1, oc - 1, 6), ("output", 3, oc // 2, -2)] if scheme != "unprotected" else []
        faults = [P.OutputFault(row=f[1], col=f[2], delta=f[3]) for f in fr]
        rep = P.conv2d(x, wt, stride=st, padding=pd, scheme=P.Scheme(scheme), faults=faults, plan_flags=flags)
        out, verdicts = O.execute(cols, wmat, O.Tiling(), scheme, fr)
        assert np.array_equal(rep.output.reshape(m, oc), out), (case, flags, scheme)
        if scheme == "global-abft":
            v, rv = rep.verdicts[0], verdicts[0]
            assert (v.detected, v.lhs, v.rhs) == (rv.detected, rv.lhs, rv.rhs)
            assert v.detected
