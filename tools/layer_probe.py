"""Time one CNN layer's conv under each scheme / global variant, with the kernel plan traced.
usage: python tools/layer_probe.py NET CONFIG LAYER [tile_n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks, profiler
from paper_2104_09455_b200.convnet import LayerRunner

CONFIGS = {"hd1": (1, 1080, 1920), "b64": (64, 224, 224), "b256": (256, 224, 224)}
net, cfg, li = sys.argv[1], sys.argv[2], int(sys.argv[3])
b, h, w = CONFIGS[cfg]
spec = [s for s in networks.capture(net, b, h, w) if s.index == li][0]
print(spec, flush=True)
r = LayerRunner(spec)
S = P.Scheme
for name, fn in [("unprot", lambda: r.conv(S.UNPROTECTED)), ("global-slice", lambda: r.conv(S.GLOBAL_ABFT)),
                 ("global-dot", lambda: r.conv_variant("global-dot")), ("one-sided", lambda: r.conv(S.THREAD_ONE_SIDED))]:
    os.environ["ABFT_TRACE"] = "1"
    fn(); torch.cuda.synchronize()
    os.environ.pop("ABFT_TRACE")
    print(f"{name:14s} {profiler.graph_time_us(fn, 10):9.1f} us", flush=True)
