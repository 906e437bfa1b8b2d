"""Batch sharding of protected inference across GPUs.

The reference is single-process (checksum.py:198-237 runs one chain); on B200 a
network forward is split by batch rows — the GEMM M dimension — one process per
GPU.  Nothing on the per-layer hot path communicates:

* thread-level verdicts are row-local (a (row, column-group) check only involves
  that row), so a shard's verdicts are exactly the full-batch verdicts of its rows;
* global verdicts are linear in the rows: lhs = sum_s colck(A_s) . rowck(B) and
  rhs = sum_s sum(C_s).  Each rank keeps per-layer fp64 [lhs_s, rhs_s]; ONE
  all-reduce (sum) at the end of the forward — a few hundred bytes over NVLink —
  gives the full-batch (lhs, rhs), and the reference's tau rule
  (checksum.py:143-153) applied to the reduced pair is exactly the full-batch
  verdict.  Checking each shard alone would use a smaller tau and could flag
  differently, so the reduction is what keeps flag parity bit-exact.

The flag counters (fired thread tiles, flagged global layers) ride in the same
all-reduce.  The functions here are backend-agnostic: NCCL with CUDA tensors on the
GPU box, gloo with CPU tensors in the CPU test-suite.
"""

from __future__ import annotations

from typing import Sequence

from .checksum import Verdict, make_verdict
from .shapes import DType


def shard_rows(batch: int, rank: int, world: int) -> tuple:
    """Contiguous [start, stop) batch rows of `rank` (first `batch % world` ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if batch < 0:
        raise ValueError("batch must be >= 0")
    q, r = divmod(batch, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def pack_partials(sums, counters):
    """[L, 2] fp64 (lhs, rhs) partials + int counters -> one fp64 message [2L + len(counters)].

    Counters are small integers, exact in fp64, so one collective carries both."""
    import torch
    flat = sums.reshape(-1).to(torch.float64)
    cnt = counters.reshape(-1).to(device=flat.device, dtype=torch.float64)
    return torch.cat([flat, cnt])


def allreduce_partials(sums, counters, group=None):
    """Sum the per-rank global-ABFT partials and flag counters over all ranks (one collective).

    Returns (reduced sums [L, 2] fp64, reduced counters int64) on the input's device."""
    import torch
    import torch.distributed as dist
    msg = pack_partials(sums, counters)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(msg, op=dist.ReduceOp.SUM, group=group)
    n = sums.numel()
    return msg[:n].view(sums.shape), msg[n:].round().to(torch.int64)


def verdicts_from_sums(sums, ks: Sequence[int], dtype: DType) -> list:
    """Host-side verdicts of reduced (lhs, rhs) pairs with the reference tau rule.

    Same rule as the device verification kernel (abft_verify_sums); used where the
    reduced pairs are already on the host (one small D2H read at the end of a forward)."""
    rows = sums.tolist() if hasattr(sums, "tolist") else list(sums)
    if len(rows) != len(ks):
        raise ValueError(f"{len(rows)} partial pairs for {len(ks)} layers")
    out = []
    for (lhs, rhs), k in zip(rows, ks):
        if dtype.is_exact:
            lhs, rhs = int(round(lhs)), int(round(rhs))
        out.append(make_verdict(dtype, int(k), lhs, rhs))
    return out


def any_detected(verdicts: Sequence[Verdict], counters) -> bool:
    return any(v.detected for v in verdicts) or int(counters[0]) > 0
