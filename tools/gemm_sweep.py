"""Per-shape timing of the sm_100a protected GEMM vs cuBLAS (torch.matmul), graph-replayed.

usage: python tools/gemm_sweep.py   -> one line per shape:
  M N K | cuBLAS us | unprotected | global | one-sided(on-chip) | one-sided(offline ck) | TFLOP/s of unprotected
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import _lib, device as D, kernels  # noqa: E402
from paper_2104_09455_b200.profiler import graph_time_us  # noqa: E402

SHAPES = [(1, 512, 16), (64, 512, 16), (2048, 512, 16), (2048, 256, 512), (2048, 64, 256), (2048, 512, 512),
          (2048, 8, 256), (256, 256, 256), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096),
          (8192, 8192, 8192), (50176, 64, 576), (200704, 64, 64), (12544, 256, 2304)]


def run(m, n, k):
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    osum = torch.zeros(1, dtype=torch.float64, device="cuda")
    lhs = torch.zeros(1, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    base = dict(out=out, ldc=n, out_kind="f16", relu=True)
    one = dict(base, fired_count=cnt, m_ext=-(-m // 16) * 16, n_ext=-(-n // 8) * 8)
    plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.THREAD_ONE_SIDED, plan_only=True,
                        **one)
    uplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.UNPROTECTED, plan_only=True, **base)
    ckr = kernels.ck_rows(pw.bt, n, k, P.BINARY16, plan, 8, False)
    aplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.THREAD_ONE_SIDED, plan_only=True,
                         ck_layout=1, **one)
    augw = kernels.aug_weights(pw.bt, n, k, P.BINARY16, aplan, 8, False)
    gkw = dict(base, out_sum=osum, out_lhs=lhs)
    gplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.GLOBAL_ABFT, plan_only=True,
                         ck_layout=1, **gkw)
    gck = kernels.global_ck_rows(pw.bt, n, k, P.BINARY16, gplan)
    it = 50 if m * n * k < 2 ** 33 else 10
    bt = b.t().contiguous()
    res = {"cublas": graph_time_us(lambda: torch.matmul(a, b), it)}
    res["unprot"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                       P.Scheme.UNPROTECTED, **base), it)
    res["global"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                       P.Scheme.GLOBAL_ABFT, ck_rows=gck, **gkw), it)
    rowck = kernels.weight_rowck(pw.bt, n, k, P.BINARY16)
    res["global_dot"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                           P.Scheme.GLOBAL_ABFT, lhs_rowck=rowck, **gkw), it)
    res["one_chip"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                         P.Scheme.THREAD_ONE_SIDED, **one), it)
    res["one_off"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                        P.Scheme.THREAD_ONE_SIDED, ck_rows=ckr, **one), it)
    res["one_aug"] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                        P.Scheme.THREAD_ONE_SIDED, ck_rows=augw, **one), it)
    del bt
    tf = 2 * m * n * k / (res["unprot"] * 1e-6) / 1e12
    gbs = 2 * (m * k + k * n + m * n) / (res["unprot"] * 1e-6) / 1e9
    print(f"{m:6d} {n:5d} {k:5d} | " + " ".join(f"{key}={v:8.2f}" for key, v in res.items()) +
          f" | unprot {tf:7.1f} TF/s {gbs:7.1f} GB/s | plan u={uplan['tile_n']}/{uplan['stages']}st grid {uplan['grid']}"
          f" one={plan['tile_n']}/{plan['stages']}st aug={aplan['tile_n']}/{aplan['stages']}st"
          f" glob={gplan['tile_n']}/{gplan['stages']}st", flush=True)


if __name__ == "__main__":
    for s in SHAPES:
        run(*s)
