"""The protected multi-layer chain (per-layer schemes, fused deferred verification, graph replay)
against the reference's run_protected_pipeline semantics (checksum.py:198-237) via the oracle."""

import numpy as np
import pytest

from oracle import abft_oracle as O

pytestmark = pytest.mark.gpu

DIMS = [16, 512, 256, 64]      # DLRM MLP-Bottom, K padded 13 -> 16


@pytest.fixture(scope="module")
def P():
    import paper_2104_09455_b200 as pkg
    from paper_2104_09455_b200 import device
    device.require_device()
    return pkg


def _weights(exact, seed=0):
    rng = np.random.default_rng(seed)
    if exact:
        # layer 0 dense, deeper layers sparse: every activation stays inside fp16's exact integers
        w0 = rng.integers(-2, 3, size=(DIMS[0], DIMS[1])).astype(np.int64)
        rest = [rng.choice([-1, 0, 1], p=[0.02, 0.96, 0.02], size=(DIMS[i], DIMS[i + 1])).astype(np.int64)
                for i in (1, 2)]
        return [w0] + rest
    return [rng.uniform(-0.5, 0.5, size=(DIMS[i], DIMS[i + 1])).astype(np.float16) for i in range(3)]


def _verdicts(chain):
    raw = chain.verdict_buf.cpu().numpy().view(np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"),
                                                         ("det", "<i4"), ("k", "<i4")]))
    return raw


@pytest.mark.parametrize("batch", [1, 64, 300])
def test_chain_global_matches_pipeline_exact(P, batch):
    import torch
    from paper_2104_09455_b200.network import ProtectedChain
    ws = _weights(True)
    rng = np.random.default_rng(batch)
    x = rng.integers(-2, 3, size=(batch, DIMS[0])).astype(np.int64)
    S = P.Scheme
    faults = {1: [(batch - 1, 7, 11.0)]}
    ch = ProtectedChain([torch.from_numpy(w.astype(np.float16)).cuda() for w in ws], batch, [S.GLOBAL_ABFT] * 3,
                        P.EXACT_INT, faults=faults)
    ch.forward(torch.from_numpy(x.astype(np.float16)).cuda())
    torch.cuda.synchronize()
    ref = O.pipeline(x, ws, None, {1: [(batch - 1, 7, 11)]})
    raw = _verdicts(ch)
    for i, v in enumerate(ref):
        assert (int(round(raw[i]["lhs"])), int(round(raw[i]["rhs"])), bool(raw[i]["det"])) == \
            (v.lhs, v.rhs, v.detected), i
    assert ch.flags() == (0, 1)
    # the last activation equals the reference chain's (ReLU on every layer, exact)
    a = x
    for i, w in enumerate(ws):
        c = a @ w
        if i == 1:
            c[batch - 1, 7] += 11
        a = np.maximum(c, 0)
    assert np.array_equal(ch.acts[-1].float().cpu().numpy().astype(np.int64), a)


def test_chain_mixed_schemes_graph_replay_binary16(P):
    import torch
    from paper_2104_09455_b200.network import GraphedForward, ProtectedChain
    S = P.Scheme
    ws = [torch.from_numpy(w).cuda() for w in _weights(False, 1)]
    batch = 256
    x = (torch.rand((batch, DIMS[0]), device="cuda") - 0.5).half()
    clean = ProtectedChain(ws, batch, [S.GLOBAL_ABFT, S.THREAD_ONE_SIDED, S.GLOBAL_ABFT])
    clean.x.copy_(x)
    g = GraphedForward(clean)
    for _ in range(3):                 # replays reuse the self-resetting verification counter
        g.replay()
        torch.cuda.synchronize()
        assert clean.flags() == (0, 0)
    # a large fault in the one-sided layer fires exactly one thread tile; in a global layer one layer
    big = {1: [(5, 9, 1000.0)]}
    ch = ProtectedChain(ws, batch, [S.GLOBAL_ABFT, S.THREAD_ONE_SIDED, S.GLOBAL_ABFT], faults=big)
    ch.forward(x)
    torch.cuda.synchronize()
    assert ch.flags() == (1, 0)
    ch2 = ProtectedChain(ws, batch, [S.GLOBAL_ABFT, S.THREAD_ONE_SIDED, S.GLOBAL_ABFT], faults={2: [(3, 1, 1e4)]})
    ch2.forward(x)
    torch.cuda.synchronize()
    assert ch2.flags() == (0, 1)


def test_sharded_partials_reduce_to_full_batch_verdict(P):
    """Batch sharding on one device: two half-batch chains' (lhs, rhs) partials
    summed give the full-batch chain's verdicts exactly in exact-int mode."""
    import torch
    from paper_2104_09455_b200.network import ProtectedChain
    from paper_2104_09455_b200 import sharding
    S = P.Scheme
    ws = [torch.from_numpy(w.astype(np.float16)).cuda() for w in _weights(True, 2)]
    batch = 200
    x = torch.from_numpy(np.random.default_rng(9).integers(-2, 3, size=(batch, DIMS[0])).astype(np.float16)).cuda()
    full = ProtectedChain(ws, batch, [S.GLOBAL_ABFT] * 3, P.EXACT_INT)
    full.forward(x)
    parts = []
    for r in range(2):
        lo, hi = sharding.shard_rows(batch, r, 2)
        ch = ProtectedChain(ws, hi - lo, [S.GLOBAL_ABFT] * 3, P.EXACT_INT)
        ch.forward(x[lo:hi])
        torch.cuda.synchronize()
        parts.append(ch.global_partials().clone())
    red = parts[0] + parts[1]
    torch.cuda.synchronize()
    assert torch.equal(red, full.global_partials())
    vs = sharding.verdicts_from_sums(red.cpu(), [16, 512, 256], P.EXACT_INT)
    assert not any(v.detected for v in vs)


def test_chain_group_batched_verification_matches_members(P):
    """A ChainGroup (one memset, members on their own streams, ONE verification launch) gives
    the same per-layer verdict values as each member's fused deferred verification, counts the
    flagged global layers of all members, and the fired thread tiles."""
    import torch
    from paper_2104_09455_b200.network import ChainGroup, ProtectedChain
    ws = _weights(True)
    wt = [torch.from_numpy(w.astype(np.float16)).cuda() for w in ws]
    S = P.Scheme
    specs = [(wt, 1, [S.GLOBAL_ABFT] * 3), (wt, 64, [S.GLOBAL_ABFT, S.THREAD_ONE_SIDED, S.GLOBAL_ABFT]),
             (wt, 300, [S.UNPROTECTED, S.GLOBAL_ABFT, S.THREAD_ONE_SIDED])]
    faults = [None, {0: [(5, 3, 9.0)], 1: [(60, 100, 7.0)]}, {1: [(299, 2, 5.0)]}]
    rng = np.random.default_rng(3)
    xs = [torch.from_numpy(rng.integers(-2, 3, size=(b, DIMS[0])).astype(np.float16)).cuda() for _, b, _ in specs]
    grp = ChainGroup([(w, b, s) for (w, b, s) in specs], dtype=P.EXACT_INT)
    for ch, f, x in zip(grp.chains, faults, xs):
        ch.faults = f
        ch._fault_dev = {int(i): P.device.faults_tensor(list(v)) for i, v in (f or {}).items()}
        ch.x.copy_(x)
    for _ in range(2):                        # replayable: the accumulators are cleared each time
        grp.forward()
        torch.cuda.synchronize()
    raw = grp.verdicts.cpu().numpy().view(np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"),
                                                   ("det", "<i4"), ("k", "<i4")]))
    o = 0
    n_global_flagged = 0
    for (w, b, sch), f, x in zip(specs, faults, xs):
        solo = ProtectedChain(w, b, sch, P.EXACT_INT, faults=f)
        solo.forward(x)
        torch.cuda.synchronize()
        sv = _verdicts(solo)
        for i in range(3):
            if sch[i] is S.GLOBAL_ABFT:
                assert (raw[o + i]["lhs"], raw[o + i]["rhs"], raw[o + i]["det"]) == \
                    (sv[i]["lhs"], sv[i]["rhs"], sv[i]["det"]), (b, i)
                n_global_flagged += int(sv[i]["det"])
            else:
                assert raw[o + i]["det"] == 0
        o += 3
    fired, flagged = grp.flags()
    assert flagged == n_global_flagged == 2
    assert fired == 1                          # the one thread-level fault, one tile
