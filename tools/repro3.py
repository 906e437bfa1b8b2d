import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks, profiler
from paper_2104_09455_b200.convnet import LayerRunner
spec = networks.capture("vgg16", 64, 224, 224)[13]
r = LayerRunner(spec)
first, second = sys.argv[1], sys.argv[2]
S = {"un": P.Scheme.UNPROTECTED, "gl": P.Scheme.GLOBAL_ABFT, "one": P.Scheme.THREAD_ONE_SIDED}
if first == "torch":
    x = torch.ones(1000, device="cuda")
    print(profiler.graph_time_us(lambda: x.add_(1), 3), flush=True)
else:
    print(profiler.graph_time_us(lambda: r.conv(S[first]), 3), flush=True)
r.conv(S[second])
torch.cuda.synchronize()
print("second ok", flush=True)
