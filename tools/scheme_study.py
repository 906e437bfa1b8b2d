"""All six schemes of the reference on the sm_100a kernel (the paper's Fig-10-style study,
SURVEY 8f item 2): graph-replayed time and overhead against the unprotected kernel.
usage: python tools/scheme_study.py [--out FILE]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import device as D, kernels  # noqa: E402
from paper_2104_09455_b200.profiler import graph_time_us  # noqa: E402

SHAPES = [(256, 256, 256), (2048, 512, 512), (64, 512, 512), (2048, 2048, 2048), (4096, 4096, 4096),
          (12544, 256, 2304), (200704, 64, 64)]


def run(m, n, k):
    S = P.Scheme
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    base = dict(out=out, ldc=n, out_kind="f16", relu=True)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    sums = torch.zeros(2, dtype=torch.float64, device="cuda")
    t = P.TilingConfig()
    thread = dict(base, thread_m=t.thread_m, thread_n=t.thread_n, m_ext=-(-m // 16) * 16, n_ext=-(-n // 8) * 8,
                  fired_count=cnt)
    calls = {S.UNPROTECTED: dict(base)}
    g = dict(base, out_sum=sums[1:2], out_lhs=sums[0:1])
    plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, S.GLOBAL_ABFT, plan_only=True, ck_layout=1, **g)
    g["ck_rows"] = kernels.global_ck_rows(pw.bt, n, k, P.BINARY16, plan)
    calls[S.GLOBAL_ABFT] = g
    for sch in (S.THREAD_ONE_SIDED, S.THREAD_TWO_SIDED):
        kw = dict(thread)
        plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, plan_only=True, ck_layout=1, **kw)
        kw["ck_rows"] = kernels.aug_weights(pw.bt, n, k, P.BINARY16, plan, t.thread_n, False)
        calls[sch] = kw
    for sch in (S.THREAD_REPLICATION_FULL, S.THREAD_REPLICATION_SINGLE_ACC):
        calls[sch] = dict(thread)
    it = 50 if m * n * k < 2 ** 33 else 10
    res = {}
    for sch, kw in calls.items():
        res[sch.value] = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, **kw), it)
    u = res["unprotected"]
    row = dict(m=m, n=n, k=k, us=res, overhead_pct={s: round(100 * (v / u - 1), 1) for s, v in res.items()})
    print(json.dumps(row), flush=True)
    return row


if __name__ == "__main__":
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "gpurun_out/scheme_study.jsonl"
    rows = [run(*s) for s in SHAPES]
    with open(out, "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
