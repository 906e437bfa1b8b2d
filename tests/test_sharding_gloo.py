"""Multi-process (gloo, world_size 2) check of the batch-sharded verification path.

Each rank takes its contiguous batch shard, forms its per-layer global-ABFT partials
(lhs_s = colck(A_s) . rowck(B), rhs_s = sum C_s — computed here by the oracle as the
checker, the GPU epilogue produces them on the box) plus its fired-tile counter, and
the product's ``allreduce_partials`` + ``verdicts_from_sums`` turn them into verdicts.
They must equal the reference's FULL-batch verdict bit for bit (exact-int), and agree on
flags for binary16 with faults far from tau.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import abft_oracle as O  # noqa: E402

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(mode, seed):
    rng = np.random.default_rng(seed)
    m, k, n = 37, 24, 19
    if mode == "exact":
        a = rng.integers(-8, 9, size=(m, k)).astype(np.int64)
        b = rng.integers(-8, 9, size=(k, n)).astype(np.int64)
    else:
        a = rng.uniform(-1, 1, size=(m, k)).astype(np.float16)
        b = rng.uniform(-1, 1, size=(k, n)).astype(np.float16)
    c = O.matmul(a, b)
    return a, b, c


def _worker(rank, port, mode, fault, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2104_09455_b200 as P
        from paper_2104_09455_b200 import sharding
        a, b, c = _case(mode, 11)
        c = c.copy()
        if fault is not None:
            c[fault[0], fault[1]] += fault[2]
        lo, hi = sharding.shard_rows(a.shape[0], rank, WORLD)
        a_s, c_s = a[lo:hi], c[lo:hi]
        lhs = O.dot(O.colck(a_s), O.rowck(b))
        rhs = O.total(c_s)
        sums = torch.tensor([[float(lhs), float(rhs)]], dtype=torch.float64)
        fired = torch.tensor([1 if (fault is not None and lo <= fault[0] < hi) else 0, 0], dtype=torch.int32)
        red, cnt = sharding.allreduce_partials(sums, fired)
        dtype = P.EXACT_INT if mode == "exact" else P.BINARY16
        v = sharding.verdicts_from_sums(red, [a.shape[1]], dtype)[0]
        q.put((rank, v.detected, v.lhs, v.rhs, v.tolerance_used, cnt.tolist()))
    finally:
        dist.destroy_process_group()


def _run(mode, fault):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mode, fault, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("fault", [None, (30, 4, 3)])
def test_sharded_exact_verdict_equals_full_batch(fault):
    a, b, c = _case("exact", 11)
    c = c.copy()
    if fault is not None:
        c[fault[0], fault[1]] += fault[2]
    ref = O.global_check(a, b, c)
    out = _run("exact", fault)
    for rank, det, lhs, rhs, tol, cnt in out:
        assert (det, lhs, rhs, tol) == (ref.detected, ref.lhs, ref.rhs, ref.tolerance_used)
        assert cnt == [1 if fault else 0, 0]


def test_sharded_binary16_flags_match_full_batch():
    a, b, c = _case("binary16", 11)
    ref_clean = O.global_check(a, b, c, "binary16")
    delta = 50.0 * ref_clean.tolerance_used
    out_clean = _run("binary16", None)
    out_fault = _run("binary16", (5, 7, delta))
    for rank, det, lhs, rhs, tol, _ in out_clean:
        assert det is False and det == ref_clean.detected
        assert lhs == pytest.approx(ref_clean.lhs, rel=1e-5, abs=1e-4)
        assert tol == pytest.approx(ref_clean.tolerance_used, rel=1e-5)
    for rank, det, *_ in out_fault:
        assert det is True


def test_shard_rows_cover_the_batch():
    from paper_2104_09455_b200.sharding import shard_rows
    for batch in (0, 1, 7, 64, 257):
        for world in (1, 2, 4, 8):
            spans = [shard_rows(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)
