"""Batch-sharded protected inference through the real GPU code path (the deferred
verdict of checksum.py:237): two ranks (gloo, both on GPU 0 — the box has one GPU) each run
half the batch through ProtectedNetwork, their per-layer checksum sums and flag counters go
out in ONE all-reduce (verify_sharded_many, the call bench.py --gpus N makes over NCCL), and
the resulting verdicts must equal the single-process full-batch verdicts — same flags, same
(lhs, rhs) up to fp64 summation order — clean and with a fault injected on one shard."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NET, BATCH = "squeezenet1_0", 4


def _run(rank, world, port, fault, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2104_09455_b200 import protected_network as PN
    net = _build(PN, BATCH // world)
    x = _input(BATCH)[rank * (BATCH // world):(rank + 1) * (BATCH // world)]
    if fault is not None and rank == fault[0]:
        net.inject({fault[1]: [fault[2]]})
    net.forward(x, verify=False)
    PN.verify_sharded_many([net])
    torch.cuda.synchronize()
    vs = net.verdicts()
    if rank == 0:
        np.save(out_path, np.array([[v.lhs, v.rhs, v.tolerance_used, float(v.detected)] for v in vs]))
        with open(out_path + ".flags", "w") as fh:
            fh.write("%d %d" % net.flags())
    dist.destroy_process_group()


def _build(PN, batch):
    return PN.ProtectedNetwork(PN.build_model(NET), batch, schemes=PN.Scheme.GLOBAL_ABFT)


def _input(batch):
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    return (torch.rand((batch, 3, 224, 224), generator=g, device="cuda") * 2 - 1).half()


def _sharded(tmp_path, fault, port):
    import torch.multiprocessing as mp
    out = str(tmp_path / f"v{port}.npy")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_run, args=(r, 2, port, fault, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    with open(out + ".flags") as fh:
        flags = tuple(int(v) for v in fh.read().split())
    return np.load(out), flags


@pytest.mark.parametrize("with_fault", [False, True])
def test_sharded_verdicts_equal_full_batch(tmp_path, with_fault):
    import torch
    from paper_2104_09455_b200 import protected_network as PN
    full = _build(PN, BATCH)
    layer = 3
    half = BATCH // 2
    fault = None
    if with_fault:
        full.forward(_input(BATCH))
        delta = 8.0 * full.verdicts()[layer].tolerance_used + 64.0    # well above tau (K = 144 < 1024)
        L = full.layers[layer]
        rows_per_image = L.m // BATCH
        # a fault on rank 1's first image: row index (shard-local) 5, full-batch row half*rows + 5
        fault = (1, layer, (5, 11, delta))
        full.inject({layer: [(half * rows_per_image + 5, 11, delta)]})
    full.forward(_input(BATCH))
    torch.cuda.synchronize()
    ref = np.array([[v.lhs, v.rhs, v.tolerance_used, float(v.detected)] for v in full.verdicts()])
    got, flags = _sharded(tmp_path, fault, 29630 + int(with_fault))
    assert np.array_equal(got[:, 3], ref[:, 3])
    assert flags == full.flags() == ((0, 1) if with_fault else (0, 0))
    if with_fault:
        assert got[layer, 3] == 1.0
    # the same sums up to rounding: a shard's launch may plan other CTA tiles than the full batch's,
    # which regroups the fp32 per-tile checksum columns; far inside tau either way
    # (layers past a huge injected fault see inf/NaN activations on both sides alike)
    fin = np.isfinite(ref[:, :3]).all(axis=1)
    assert np.array_equal(fin, np.isfinite(got[:, :3]).all(axis=1))
    assert fin[:layer + 1].all()
    g, r = got[fin], ref[fin]
    assert (np.abs(g[:, 0] - r[:, 0]) <= 1e-5 * np.maximum(r[:, 2], 1)).all()
    assert (np.abs(g[:, 1] - r[:, 1]) <= 1e-5 * np.maximum(r[:, 2], 1)).all()
