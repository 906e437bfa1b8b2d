"""Output-store throughput of the unprotected kernel on write-bound shapes (tiny K), against a
torch device copy of the same bytes: python tools/store_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import _lib, kernels, profiler  # noqa: E402
from paper_2104_09455_b200 import device as D  # noqa: E402

for m, n, k in ((12845056, 64, 16), (3211264, 256, 16), (802816, 256, 64), (3211264, 64, 64), (3211264, 128, 16)):
    a = (torch.rand((m, k), device="cuda") - 0.5).half()
    b = (torch.rand((k, n), device="cuda") - 0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    nbytes = out.numel() * 2 + a.numel() * 2
    for flags in (0, 16, 8):
        def run():
            kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, _lib.NUM_BINARY16, P.Scheme.UNPROTECTED,
                         out=out, ldc=n, out_kind="f16", relu=True, plan_flags=flags)
        us = profiler.graph_time_us(run, 10)
        print(f"gemm M={m} N={n} K={k} flags={flags}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s", flush=True)
    src = torch.empty_like(out)
    us = profiler.graph_time_us(lambda: out.copy_(src), 10)
    print(f"torch copy {out.numel() * 2 / 1e6:.0f} MB: {us:.1f} us  {2 * out.numel() * 2 / us / 1e3:.0f} GB/s (r+w)",
          flush=True)
    us = profiler.graph_time_us(lambda: out.fill_(1.0), 10)
    print(f"torch fill {out.numel() * 2 / 1e6:.0f} MB: {us:.1f} us  {out.numel() * 2 / us / 1e3:.0f} GB/s (w)", flush=True)
    del a, b, out, src
    torch.cuda.empty_cache()
