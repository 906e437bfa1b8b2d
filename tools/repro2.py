import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks, profiler
from paper_2104_09455_b200.convnet import LayerRunner
spec = networks.capture("vgg16", 64, 224, 224)[13]
r = LayerRunner(spec)
mode = sys.argv[1]
if mode == "graph":
    print("un", profiler.graph_time_us(lambda: r.conv(P.Scheme.UNPROTECTED), 3), flush=True)
elif mode == "eager":
    r.conv(P.Scheme.UNPROTECTED); torch.cuda.synchronize()
elif mode == "stream":
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        r.conv(P.Scheme.UNPROTECTED)
    torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    r.conv(P.Scheme.GLOBAL_ABFT)
torch.cuda.synchronize()
print("global ok", flush=True)
