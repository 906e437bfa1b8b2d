"""Max pooling with the consumer's column sums: pool + column-sum pass vs the pooling kernel that
accumulates them (abft_nhwc_maxpool_ws), graph-replayed:  python tools/pool_ws_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200 import kernels  # noqa: E402
from paper_2104_09455_b200.profiler import capture_graph, interleaved_min_us  # noqa: E402

for n, h, c in ((256, 224, 64), (256, 112, 128), (256, 56, 256), (256, 28, 512), (256, 112, 64)):
    x = (torch.rand((n, h, h, c), device="cuda") - 0.5).half()
    o = torch.empty((n, h // 2, h // 2, c), dtype=torch.float16, device="cuda")
    ws = torch.zeros((1, c), dtype=torch.float32, device="cuda")
    k, s = (2, 2) if h != 112 or c != 64 else (3, 2)
    pad = 1 if k == 3 else 0
    def pool():
        kernels.maxpool_nhwc(x, n, h, h, c, c, k, s, pad, False, P.BINARY16, o, c)
    def pool_col():
        pool()
        kernels.colsum(o, o.shape[0] * o.shape[1] * o.shape[2], c, c, P.BINARY16, ws, accumulate=True)
    def pool_ws():
        kernels.maxpool_nhwc_ws(x, n, h, h, c, c, k, s, pad, False, P.BINARY16, o, c, ws, c, 1)
    g = [capture_graph(f, 5) for f in (pool, pool_col, pool_ws)]
    t = interleaved_min_us(g, 5)
    gb = (x.numel() + o.numel()) * 2 / 1e9
    print(f"{n}x{h}x{h}x{c} k{k}: pool {t[0]:.1f} us ({gb / t[0] * 1e6 / 1e3:.2f} TB/s)  pool+colsum {t[1]:.1f}  "
          f"pool_ws {t[2]:.1f}", flush=True)
    del x, o
