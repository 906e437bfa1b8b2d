"""Which epilogue step bounds a bandwidth-bound GEMM: ABFT_DEBUG bits x grid size x stages."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels
from paper_2104_09455_b200.profiler import graph_time_us

BITS = {"full": 0, "no_sts": 131072, "no_tma": 262144, "no_store": 16384, "no_epi": 32768, "direct": 8192,
        "nosplit": 65536}
for (m, n, k) in [(200704, 256, 64), (200704, 64, 64), (12544, 256, 2304)]:
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    fn = lambda sms=0: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, P.Scheme.UNPROTECTED, out=out,
                                    ldc=n, out_kind="f16", relu=True, num_sms=sms)
    res = []
    for name, bit in BITS.items():
        os.environ["ABFT_DEBUG"] = str(bit)
        res.append(f"{name}={graph_time_us(fn, 20):.1f}")
    os.environ.pop("ABFT_DEBUG")
    for sms in (37, 74, 111):
        res.append(f"sms{sms}={graph_time_us(lambda: fn(sms), 20):.1f}")
    for cap in (140, 190):
        os.environ["ABFT_SMEM_CAP"] = str(cap)
        try:
            res.append(f"cap{cap}={graph_time_us(fn, 20):.1f}")
        except Exception:
            res.append(f"cap{cap}=ERR")
    os.environ.pop("ABFT_SMEM_CAP")
    res.append(f"fill={graph_time_us(lambda: out.fill_(1.0), 20):.1f}")
    res.append(f"copy={graph_time_us(lambda: out.copy_(out.flip(0)) if False else torch.add(out, 1, out=out), 20):.1f}")
    print(m, n, k, " ".join(res), flush=True)
