"""In-network per-layer cost of global ABFT: the all-unprotected forward vs the same forward with
only layer i under global ABFT (interleaved CUDA-graph replays, medians)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
from paper_2104_09455_b200 import protected_network as PN, netprofile as NP

name, b = sys.argv[1], int(sys.argv[2])
net = PN.ProtectedNetwork(PN.build_model(name), b)
net.load_input((torch.rand((b, 3, 224, 224), device="cuda") * 2 - 1).half())
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
meas = NP.profile(net, 10)
S = PN.Scheme
net.set_schemes(S.UNPROTECTED)
base = PN.GraphedNetwork(net, warmup=1, verify=False)
tot = 0.0
for L in net.layers:
    L.scheme = S.GLOBAL_ABFT
    g = PN.GraphedNetwork(net, warmup=1, verify=False)
    t0, t1 = NP._forward_ms([base.graph, g.graph], 9)
    L.scheme = S.UNPROTECTED
    tot += t1 - t0
    pu, pg = net.plan_of(L, S.UNPROTECTED), net.plan_of(L, S.GLOBAL_ABFT)
    print(f"{L.index:3d} {L.name:28s} M={L.m:8d} N={L.oc:5d} K={L.k_ref:5d} gvar={L.gvar:5s} cfgU={net.config_of(L, S.UNPROTECTED)} "
          f"delta_us={1e3 * (t1 - t0):8.1f} iso_un={meas.get(L.index, S.UNPROTECTED) * 1e6:8.1f} iso_gl={meas.get(L.index, S.GLOBAL_ABFT) * 1e6:8.1f} "
          f"tileU={pu['tile_n']}/{pu['stages']} tileG={pg['tile_n']}/{pg['stages']}", flush=True)
print("sum of deltas ms", tot, "base ms", NP._forward_ms([base.graph], 9)[0])
