"""A-load mode of every conv layer of the bench networks under each scheme's current arguments:
python tools/amode_probe.py [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

from paper_2104_09455_b200 import kernels  # noqa: E402
from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

S = PN.Scheme
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for name in ("resnet50", "vgg16", "squeezenet1_0", "shufflenet_v2_x1_0"):
    net = PN.ProtectedNetwork(PN.build_model(name), batch)
    for L in net.layers:
        kind, a = L.args[S.UNPROTECTED]
        if kind != "conv":
            continue
        pl = kernels.conv_plan(a)
        if pl["a_mode"] in (2, 3):
            print(name, L.name, "c", L.x.c, "k", L.r, "s", L.stride, "a_mode", pl["a_mode"], "ws MB",
                  round(pl["ws"] / 1e6, 1), flush=True)
