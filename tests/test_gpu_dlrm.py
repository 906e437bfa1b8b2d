"""Parity of the benchmarked C2 workload itself: all 24 DLRM chains (MLP-Bottom 13-512-256-64
and MLP-Top 512-512-256-1 at batch 1..2048, x8 padded, the N = 1 -> 8 output layer included) as
ONE ChainGroup — the configuration bench.py times — against the reference pipeline
(checksum.py:198-237, oracle.pipeline): every layer's output on the layer's own input, every
global layer's (lhs, rhs) and flag, bit-exact in exact-int mode, under always-global,
always-thread-level and mixed plans, clean and with injected faults."""

import numpy as np
import pytest

from oracle import abft_oracle as O

pytestmark = pytest.mark.gpu

GEMM_RTOL = 2e-5
VERDICT_DTYPE = np.dtype([("lhs", "<f8"), ("rhs", "<f8"), ("tol", "<f8"), ("det", "<i4"), ("k", "<i4")])


@pytest.fixture(scope="module")
def P():
    import paper_2104_09455_b200 as pkg
    from paper_2104_09455_b200 import device
    device.require_device()
    return pkg


def _workload(exact):
    from tools import dlrm_secondary as W
    mlps, inputs = W.workload()
    if exact:
        rng = np.random.default_rng(5)
        for name, ws in mlps.items():
            # first layer dense small integers, deeper layers sparse: activations stay in fp16's exact range
            mlps[name] = [np.where(w != 0, rng.integers(-2, 3, size=w.shape), 0).astype(np.float16) if i == 0 else
                          np.where(w != 0, rng.choice([-1, 0, 1], p=[0.03, 0.94, 0.03], size=w.shape), 0)
                          .astype(np.float16) for i, w in enumerate(ws)]
        for k, x in inputs.items():
            inputs[k] = np.where(x != 0, rng.integers(-2, 3, size=x.shape), 0).astype(np.float16)
    return mlps, inputs, W.BATCHES


def _plan(policy, S, key):
    if policy == "global":
        return [S.GLOBAL_ABFT] * 3
    if policy == "thread":
        return [S.THREAD_ONE_SIDED] * 3
    # mixed: what the IG selector produces on other boxes / sizes
    return [S.GLOBAL_ABFT, S.THREAD_ONE_SIDED, S.GLOBAL_ABFT] if key[1] % 2 else \
        [S.THREAD_ONE_SIDED, S.GLOBAL_ABFT, S.UNPROTECTED]


@pytest.mark.parametrize("grouped", [False, True])
@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("policy", ["global", "thread", "mixed"])
def test_dlrm_24_chains_match_reference(P, policy, exact, grouped):
    """(grouped: every layer depth of the 24 chains as grouped launches, one per depth and scheme.)"""
    import torch
    from paper_2104_09455_b200.network import ChainGroup
    S = P.Scheme
    mlps, inputs, batches = _workload(exact)
    keys = [(n, b) for n in ("bottom", "top") for b in batches]
    wt = {n: [torch.from_numpy(w).cuda() for w in ws] for n, ws in mlps.items()}
    plans = {k: _plan(policy, S, k) for k in keys}
    grp = ChainGroup([(wt[k[0]], k[1], plans[k]) for k in keys], dtype=P.EXACT_INT if exact else P.BINARY16,
                     ck_split=True, grouped=grouped)
    if grouped:
        assert len(grp._groups) <= 9
    for k, ch in zip(keys, grp.chains):
        ch.x.copy_(torch.from_numpy(inputs[k]).cuda())
    grp.forward()
    torch.cuda.synchronize()
    assert grp.flags() == (0, 0)
    raw = grp.verdicts.cpu().numpy().view(VERDICT_DTYPE)
    o = 0
    for k, ch in zip(keys, grp.chains):
        ws = mlps[k[0]]
        a = inputs[k]
        for i, w in enumerate(ws):
            out = ch.acts[i].float().cpu().numpy()
            if exact:
                ref = np.maximum(a.astype(np.int64) @ w.astype(np.int64), 0)
                assert np.array_equal(out.astype(np.int64), ref), (k, i)
            else:
                c = a.astype(np.float32) @ w.astype(np.float32)
                ref = np.maximum(c, 0).astype(np.float16).astype(np.float32)
                bound = np.abs(a.astype(np.float64)) @ np.abs(w.astype(np.float64))
                err = np.abs(out - ref)
                assert (err <= GEMM_RTOL * bound + np.abs(ref) * 2.0 ** -10 + 1e-6).all(), (k, i, err.max())
            if plans[k][i] is S.GLOBAL_ABFT:
                ai, wi = (a.astype(np.int64), w.astype(np.int64)) if exact else (a, w)
                v = O.global_check(ai, wi, O.matmul(ai, wi), O.EXACT if exact else "binary16")
                g = raw[o + i]
                assert bool(g["det"]) == v.detected == False  # noqa: E712
                if exact:
                    assert (int(round(g["lhs"])), int(round(g["rhs"]))) == (v.lhs, v.rhs), (k, i)
                else:
                    assert abs(g["lhs"] - v.lhs) <= 1e-3 * v.tolerance_used, (k, i)
                    assert abs(g["rhs"] - v.rhs) <= 1e-3 * v.tolerance_used, (k, i)
            a = ch.acts[i].cpu().numpy().astype(np.float16)       # the next layer's input as the GPU has it
        o += 3


@pytest.mark.parametrize("policy", ["global", "thread"])
def test_dlrm_24_chains_fault_flags(P, policy):
    """One injected fault per chain (exact-int, so detection is exact): every global fault flags
    its layer, every thread-level fault fires exactly one thread tile, across all 24 chains."""
    import torch
    from paper_2104_09455_b200.network import ChainGroup
    S = P.Scheme
    mlps, inputs, batches = _workload(True)
    keys = [(n, b) for n in ("bottom", "top") for b in batches]
    wt = {n: [torch.from_numpy(w).cuda() for w in ws] for n, ws in mlps.items()}
    plans = {k: _plan(policy, S, k) for k in keys}
    grp = ChainGroup([(wt[k[0]], k[1], plans[k]) for k in keys], dtype=P.EXACT_INT)
    for j, (k, ch) in enumerate(zip(keys, grp.chains)):
        layer = j % 3
        n_out = mlps[k[0]][layer].shape[1]
        f = {layer: [(k[1] - 1, (7 * j) % min(n_out, 64), 5.0)]}
        ch.faults = f
        ch._fault_dev = {int(i): P.device.faults_tensor(list(v)) for i, v in f.items()}
        ch.x.copy_(torch.from_numpy(inputs[k]).cuda())
    grp.forward()
    torch.cuda.synchronize()
    fired, flagged = grp.flags()
    if policy == "global":
        assert (fired, flagged) == (0, len(keys))
    else:
        assert (fired, flagged) == (len(keys), 0)
