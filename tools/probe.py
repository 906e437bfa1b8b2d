"""Time protected-GEMM variants: python tools/probe.py "M N K scheme tile_n [debug] [acolck|dot|gck]" ..."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels
from paper_2104_09455_b200.profiler import graph_time_us

cache = {}
for spec in sys.argv[1:]:
    f = spec.split()
    m, n, k, sch, tn = int(f[0]), int(f[1]), int(f[2]), P.Scheme(f[3]), int(f[4])
    dbg = int(f[5]) if len(f) > 5 else 0
    acol = len(f) > 6 and f[6] == "acolck"
    key = (m, n, k)
    if key not in cache:
        a = (torch.rand((m, k), device="cuda") - 0.5).half()
        b = (torch.rand((k, n), device="cuda") - 0.5).half()
        cache.clear()
        cache[key] = (a, D.prepare_weight(b, P.BINARY16), torch.empty((m, n), dtype=torch.float16, device="cuda"))
    a, pw, out = cache[key]
    kw = dict(out=out, ldc=n, out_kind="f16", relu=True, tile_n=tn)
    if sch is P.Scheme.GLOBAL_ABFT:
        kw["out_sum"] = torch.zeros(1, dtype=torch.float64, device="cuda")
        if acol:
            kw["a_colck"] = torch.zeros(k, dtype=torch.float32, device="cuda")
        elif len(f) > 6 and f[6] == "dot":
            kw["out_lhs"] = torch.zeros(1, dtype=torch.float64, device="cuda")
            kw["lhs_rowck"] = kernels.weight_rowck(pw.bt, n, k, P.BINARY16)
        elif len(f) > 6 and f[6] == "gck":
            kw["out_lhs"] = torch.zeros(1, dtype=torch.float64, device="cuda")
            gplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, plan_only=True, ck_layout=1, **kw)
            kw["ck_rows"] = kernels.global_ck_rows(pw.bt, n, k, P.BINARY16, gplan)
    elif sch is not P.Scheme.UNPROTECTED:
        kw.update(fired_count=torch.zeros(1, dtype=torch.int32, device="cuda"), m_ext=-(-m // 16) * 16,
                  n_ext=-(-n // 8) * 8)
        if len(f) > 6 and f[6] == "aug":
            tplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, plan_only=True, ck_layout=1, **kw)
            kw["ck_rows"] = kernels.aug_weights(pw.bt, n, k, P.BINARY16, tplan, 8, False)
    os.environ["ABFT_DEBUG"] = str(dbg)
    try:
        plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, plan_only=True, **kw)
        us = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, **kw),
                           10 if m * n * k > 2 ** 34 else 30)
        print(f"{spec:45s} {us:9.2f} us  {2*m*n*k/us/1e6:8.1f} TF/s  plan {plan}", flush=True)
    except Exception as e:
        print(f"{spec:45s} ERROR {e}", flush=True)
    os.environ.pop("ABFT_DEBUG")
