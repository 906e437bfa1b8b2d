"""Do independent launches overlap as parallel CUDA-graph branches?  24 branches of (a) one small
abft GEMM each, (b) one small torch matmul each, against the same launches on one stream.
  python tools/concurrency_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import _lib, kernels  # noqa: E402
from paper_2104_09455_b200 import device as D  # noqa: E402

NB = 24
m, n, k = 64, 512, 512
As = [(torch.rand((m, k), device="cuda") - 0.5).half() for _ in range(NB)]
Ws = [D.prepare_weight((torch.rand((k, n), device="cuda") - 0.5).half(), P.BINARY16) for _ in range(NB)]
Os = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _ in range(NB)]
Bt = [(torch.rand((k, n), device="cuda") - 0.5).half() for _ in range(NB)]


def abft(i):
    kernels.gemm(As[i], k, Ws[i].bt, Ws[i].ldbt, m, n, k, P.BINARY16, _lib.NUM_BINARY16, P.Scheme.UNPROTECTED,
                 out=Os[i], ldc=n, out_kind="f16")


def tmm(i):
    torch.matmul(As[i], Bt[i], out=Os[i])


def capture(fn, parallel):
    main = torch.cuda.Stream()
    streams = [torch.cuda.Stream() for _ in range(NB)]
    main.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(main):
        for i in range(NB):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        for i, s in enumerate(streams):
            if parallel:
                s.wait_stream(main)
                with torch.cuda.stream(s):
                    fn(i)
                main.wait_stream(s)
            else:
                fn(i)
    torch.cuda.synchronize()
    return g


def timeit(g, n=30):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


for name, fn in (("abft", abft), ("torch", tmm)):
    print(name, "24 parallel branches", round(timeit(capture(fn, True)), 1), "us;  one stream",
          round(timeit(capture(fn, False)), 1), "us", flush=True)
