"""Tile plans of a network's window-sum producers with and without the window sums (a producer's
cost jump when ws_active flips the plan): python tools/ws_plan_probe.py NET [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

S = PN.Scheme
name = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
net = PN.ProtectedNetwork(PN.build_model(name), batch)
for P in net.producers():
    if not isinstance(P, PN.LinearLayer):
        continue
    plans = []
    for on in (False, True):
        P.ws_active = on
        plans.append(net._plan(P, S.UNPROTECTED, net._kw(P, S.UNPROTECTED)))
    P.ws_active = False
    print(P.name, "flags", P.flags.get(S.UNPROTECTED), "\n  off", plans[0], "\n  on ", plans[1], flush=True)
