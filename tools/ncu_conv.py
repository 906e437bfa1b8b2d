"""Launch one network layer's protected conv a few times (target for ncu):
python tools/ncu_conv.py NET CFG IDX SCHEME [reps]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks
from paper_2104_09455_b200.convnet import LayerRunner
CONFIGS = {"hd1": (1, 1080, 1920), "b64": (64, 224, 224), "b256": (256, 224, 224), "b8": (8, 224, 224)}
net, cfg, idx, sch = sys.argv[1], sys.argv[2], int(sys.argv[3]), P.Scheme(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
r = LayerRunner(networks.capture(net, *CONFIGS[cfg])[idx])
print("plan", r.plan, flush=True)
for _ in range(reps):
    r.conv(sch)
torch.cuda.synchronize()
print("done", flush=True)
