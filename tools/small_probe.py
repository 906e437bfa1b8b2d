"""Graph-replayed timing of small protected GEMMs under the ABFT_DEBUG knob (bring-up)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels
from tools.perf_probe_lib import bench
m, n, k = (int(x) for x in sys.argv[1:4])
a = (torch.rand((m, k), device="cuda") - 0.5).half()
b = (torch.rand((k, n), device="cuda") - 0.5).half()
pw = D.prepare_weight(b, P.BINARY16)
out = torch.empty((m, n), dtype=torch.float16, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
base = dict(out=out, ldc=n, out_kind="f16", relu=True)
one = dict(base, fired_count=cnt, m_ext=-(-m // 16) * 16, n_ext=-(-n // 8) * 8)
plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.THREAD_ONE_SIDED, plan_only=True, **one)
ckr = kernels.ck_rows(pw.bt, n, k, P.BINARY16, plan, 8, False)
res = []
for name, sch, kw in [("unprot", P.Scheme.UNPROTECTED, base), ("onesided", P.Scheme.THREAD_ONE_SIDED, one),
                      ("offline", P.Scheme.THREAD_ONE_SIDED, dict(one, ck_rows=ckr))]:
    res.append(f"{name} {bench(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, **kw)):.2f}")
print(m, n, k, "plan", plan, " | ".join(res))
