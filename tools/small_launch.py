"""Back-to-back launches of small protected GEMMs (for ncu launch-duration lists)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels, _lib
m, n, k = 1, 512, 16
a = (torch.rand((m, k), device="cuda") - 0.5).half()
b = (torch.rand((k, n), device="cuda") - 0.5).half()
pw = D.prepare_weight(b, P.BINARY16)
out = torch.empty((m, n), dtype=torch.float16, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
osum = torch.zeros(1, dtype=torch.float64, device="cuda")
base = dict(out=out, ldc=n, out_kind="f16", relu=True)
one = dict(base, fired_count=cnt, m_ext=16, n_ext=512)
plan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.THREAD_ONE_SIDED, plan_only=True, **one)
ckr = kernels.ck_rows(pw.bt, n, k, P.BINARY16, plan, 8, False)
cfgs = [("unprot", P.Scheme.UNPROTECTED, base), ("global", P.Scheme.GLOBAL_ABFT, dict(base, out_sum=osum)),
        ("onesided", P.Scheme.THREAD_ONE_SIDED, one), ("offline", P.Scheme.THREAD_ONE_SIDED, dict(one, ck_rows=ckr)),
        ("onesided_noflag", P.Scheme.THREAD_ONE_SIDED, dict(base, m_ext=16, n_ext=512))]
for name, sch, kw in cfgs:
    for _ in range(6):
        kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, **kw)
    torch.cuda.synchronize()
print("done")
