"""Per-CTA %globaltimer stamps (ABFT_DEBUG bit 2048) of small protected GEMMs: where the time goes."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import _lib, device as D, kernels
lib = _lib.load()
m, n, k = (int(x) for x in sys.argv[1:4])
a = (torch.rand((m, k), device="cuda") - 0.5).half()
b = (torch.rand((k, n), device="cuda") - 0.5).half()
pw = D.prepare_weight(b, P.BINARY16)
out = torch.empty((m, n), dtype=torch.float16, device="cuda")
S = P.Scheme
base = dict(out=out, ldc=n, out_kind="f16", relu=True)
osum = torch.zeros(2, dtype=torch.float64, device="cuda")
gkw = dict(base, out_sum=osum[1:2], out_lhs=osum[0:1])
gplan = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, S.GLOBAL_ABFT, plan_only=True, **gkw)
gkw["ck_rows"] = kernels.global_ck_rows(pw.bt, n, k, P.BINARY16, gplan)
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
okw = dict(base, fired_count=cnt, m_ext=-(-m // 16) * 16, n_ext=-(-n // 8) * 8)
buf = (ctypes.c_ulonglong * (160 * 8))()
os.environ["ABFT_DEBUG"] = "2048"
for name, sch, kw in [("unprot", S.UNPROTECTED, base), ("global", S.GLOBAL_ABFT, gkw), ("onesided", S.THREAD_ONE_SIDED, okw)]:
    rows = []
    for it in range(6):
        kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, **kw)
        torch.cuda.synchronize()
        lib.abft_debug_timestamps(buf)
        ts = np.frombuffer(buf, dtype=np.uint64).reshape(160, 8).astype(np.int64)
        g = kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, plan_only=True, **kw)["grid"]
        ts = ts[:g]
        rel = ts[:, :7] - ts[:, 0].min()
        rows.append(np.median(rel, axis=0))
    med = np.median(np.array(rows[2:]), axis=0).astype(int).tolist()
    print(f"{name:9s} {m}x{n}x{k}: entry,setup,tfull0,epi_end,exit,ld0,tile0_done (ns) {med}", flush=True)
