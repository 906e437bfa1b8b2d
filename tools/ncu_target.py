"""Launch one protected GEMM configuration a few times (target for ncu captures).
usage: python tools/ncu_target.py M N K scheme [reps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels, _lib

m, n, k = (int(x) for x in sys.argv[1:4])
sch = P.Scheme(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
k8 = D.round8(k)
a = (torch.rand((m, k8), device="cuda") - 0.5).half()
b = (torch.rand((k8, n), device="cuda") - 0.5).half()
pw = D.prepare_weight(b, P.BINARY16)
out = torch.empty((m, D.round8(n)), dtype=torch.float16, device="cuda")
osum = torch.zeros(1, dtype=torch.float64, device="cuda")
colck = torch.zeros(D.round8(n), dtype=torch.float32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
kw = {}
if sch is P.Scheme.GLOBAL_ABFT:
    # the product's global scheme: output summation + the lhs checksum slice
    lhs = torch.zeros(1, dtype=torch.float64, device="cuda")
    kw = dict(out_sum=osum, out_lhs=lhs)
    plan = kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                        ldc=out.stride(0), out_kind="f16", relu=True, plan_only=True, ck_layout=1, **kw)
    kw["ck_rows"] = kernels.global_ck_rows(pw.bt, n, k8, P.BINARY16, plan)
elif sch is not P.Scheme.UNPROTECTED:
    kw = dict(fired_count=cnt, m_ext=-(-m // 16) * 16, n_ext=-(-n // 8) * 8)
    if len(sys.argv) <= 6 or sys.argv[6] == "aug":
        plan = kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                            ldc=out.stride(0), out_kind="f16", relu=True, plan_only=True, ck_layout=1, **kw)
        kw["ck_rows"] = kernels.aug_weights(pw.bt, n, k8, P.BINARY16, plan, 8, False)
    elif sys.argv[6] == "offline":
        plan = kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                            ldc=out.stride(0), out_kind="f16", relu=True, plan_only=True, **kw)
        kw["ck_rows"] = kernels.ck_rows(pw.bt, n, k8, P.BINARY16, plan, 8, False)
torch.cuda.synchronize()
for _ in range(reps):
    kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                 ldc=out.stride(0), out_kind="f16", relu=True, **kw)
torch.cuda.synchronize()
print("done", m, n, k, sch.value)
