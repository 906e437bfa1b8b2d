"""Run one network layer under a scheme (bring-up): python tools/repro_layer.py NET CFG IDX [scheme ...]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks
from paper_2104_09455_b200.convnet import LayerRunner
CONFIGS = {"hd1": (1, 1080, 1920), "b64": (64, 224, 224), "b8": (8, 224, 224), "b32": (32, 224, 224)}
net, cfg, idx = sys.argv[1], sys.argv[2], int(sys.argv[3])
b, h, w = CONFIGS[cfg]
spec = networks.capture(net, b, h, w)[idx]
print(spec, flush=True)
r = LayerRunner(spec)
print("plan", r.plan, flush=True)
for s in sys.argv[4:] or ["unprotected", "global-abft", "thread-one-sided"]:
    sch = P.Scheme(s)
    r.conv(sch)
    torch.cuda.synchronize()
    print("ok", s, flush=True)
r.global_standalone(); torch.cuda.synchronize(); print("ok standalone", flush=True)
