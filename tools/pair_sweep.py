"""CTA pairs (plan_flags bit 12) against the single-CTA kernel and cuBLAS on plain GEMMs, unprotected
and global ABFT (checksum slice), graph-replayed:  python tools/pair_sweep.py [M N K ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import device as D, kernels  # noqa: E402
from paper_2104_09455_b200.profiler import graph_time_us  # noqa: E402

SHAPES = [(4096, 4096, 4096), (8192, 8192, 8192), (16384, 4096, 4096), (802816, 256, 2304), (200704, 512, 4608),
          (12845056, 64, 576), (3211264, 128, 1152), (2048, 512, 512)]


def run(m, n, k):
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    osum = torch.zeros(1, dtype=torch.float64, device="cuda")
    lhs = torch.zeros(1, dtype=torch.float64, device="cuda")
    base = dict(out=out, ldc=n, out_kind="f16", relu=True)
    gkw = dict(base, out_sum=osum, out_lhs=lhs)
    it = 20 if m * n * k < 2 ** 36 else 5
    res = {"cublas": graph_time_us(lambda: torch.matmul(a, b), it)}
    plans = {}
    for fl in (0, 4096):
        u = dict(base, plan_flags=fl)
        plans[f"u{fl}"] = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.UNPROTECTED,
                                       plan_only=True, **u)
        res[f"unprot{'_pair' if fl else ''}"] = graph_time_us(
            lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.UNPROTECTED, **u), it)
        g = dict(gkw, plan_flags=fl)
        gplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.GLOBAL_ABFT, plan_only=True,
                             ck_layout=1, **g)
        plans[f"g{fl}"] = gplan
        gck = kernels.global_ck_rows(pw.bt, n, k, P.BINARY16, gplan)
        res[f"global{'_pair' if fl else ''}"] = graph_time_us(
            lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.GLOBAL_ABFT, ck_rows=gck,
                                 **g), it)
    # global with the lhs outside the GEMM (plan_flags bit 10): colck(A) by one column-sum pass,
    # dotted with the weights' offline rowck(B) (checksum.py:108-117), the GEMM only sums its output
    rowck = kernels.weight_rowck(pw.bt, n, k, P.BINARY16)
    colck = torch.zeros(k, dtype=torch.float32, device="cuda")
    sums = torch.zeros(2, dtype=torch.float64, device="cuda")
    tasks = kernels.global_tasks([(colck, rowck, None, k)])
    ekw = dict(base, out_sum=sums[1:2], plan_flags=1024 | 4096)

    def ext():
        kernels.colsum(a, m, k, k, P.BINARY16, colck)
        kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.GLOBAL_ABFT, **ekw)
        kernels.global_lhs(tasks, 1, sums)
    res["global_ext_pair"] = graph_time_us(ext, it)
    # the same with the column-sum pass on a second stream, overlapping the (compute-bound) GEMM
    side = torch.cuda.Stream()

    def ext_overlap():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            kernels.colsum(a, m, k, k, P.BINARY16, colck)
        kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.GLOBAL_ABFT, **ekw)
        cur.wait_stream(side)
        kernels.global_lhs(tasks, 1, sums)
    res["global_ext_pair_overlap"] = graph_time_us(ext_overlap, it)
    tf = {key: 2 * m * n * k / (v * 1e-6) / 1e12 for key, v in res.items()}
    print(f"{m:8d} {n:5d} {k:5d} | " + " ".join(f"{key}={v:9.2f}us({tf[key]:6.0f})" for key, v in res.items()) +
          " | tiles " + " ".join(f"{key}={pl['tile_n']}/{pl['stages']}st" for key, pl in plans.items()), flush=True)
    del a, b, out, pw
    torch.cuda.empty_cache()


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] if args else SHAPES
    for s in shapes:
        run(*s)
