"""Time one network layer's unprotected conv under each A-load mode / debug bit (bring-up)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import networks, profiler
from paper_2104_09455_b200.convnet import LayerRunner
CONFIGS = {"hd1": (1, 1080, 1920), "b64": (64, 224, 224)}
net, cfg, idx = sys.argv[1], sys.argv[2], int(sys.argv[3])
r = LayerRunner(networks.capture(net, *CONFIGS[cfg])[idx])
for name, env in [("default", {}), ("halo_tiled4d", {"ABFT_DEBUG": "4194304"}), ("mode1", {"ABFT_CONV_MODE": "1"}), ("halo_nores", {"ABFT_DEBUG": "262144"}),
                  ("halo_nooff", {"ABFT_DEBUG": "2097152"}), ("halo_nostore", {"ABFT_DEBUG": "16384"}),
                  ("halo_noepi", {"ABFT_DEBUG": "32768"}), ("mode1_noepi", {"ABFT_CONV_MODE": "1", "ABFT_DEBUG": "32768"})]:
    old = dict(os.environ)
    os.environ.update(env)
    try:
        us = profiler.graph_time_us(lambda: r.conv(P.Scheme.UNPROTECTED), 5)
        print(f"{net} {cfg} {idx} {name:14s} {us:8.1f} us", flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True)
    os.environ.clear()
    os.environ.update(old)
