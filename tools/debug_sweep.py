"""Time a few GEMM shapes under ABFT_DEBUG bring-up bits (which part of the kernel bounds it)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels
from paper_2104_09455_b200.profiler import graph_time_us

BITS = {"full": 0, "no_store": 16384, "no_epi": 32768, "no_tmastore": 8192}
for (m, n, k) in [(200704, 256, 64), (2048, 512, 512), (200704, 64, 576), (8192, 8192, 8192), (12544, 256, 2304)]:
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    res = []
    for name, bit in BITS.items():
        os.environ["ABFT_DEBUG"] = str(bit)
        for tn in (0, 64, 128, 256):
            if tn and tn > n:
                continue
            try:
                us = graph_time_us(lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1,
                                                        P.Scheme.UNPROTECTED, out=out, ldc=n, out_kind="f16",
                                                        relu=True, tile_n=tn), 10 if m * n * k > 2**33 else 30)
                res.append(f"{name}/tn{tn}={us:.1f}")
            except Exception as e:
                res.append(f"{name}/tn{tn}=ERR")
    os.environ.pop("ABFT_DEBUG")
    print(m, n, k, " ".join(res), flush=True)
    del a, b, pw, out
