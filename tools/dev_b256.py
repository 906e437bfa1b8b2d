"""Bring-up: eager protected forwards at a given batch with a sync after every op (locates faults)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_09455_b200 import protected_network as PN
from paper_2104_09455_b200 import netprofile as NP

names = sys.argv[1].split(",")
b = int(sys.argv[2])
for name in names:
    net = PN.ProtectedNetwork(PN.build_model(name), b)
    net.load_input((torch.rand((b, 3, 224, 224), device="cuda") * 2 - 1).half())
    for sch in PN.SELECTABLE:
        net.set_schemes(sch)
        PN.kernels.zero(net._block)
        for op in net.ops:
            if isinstance(op, PN.LinearLayer):
                net.launch(op)
            else:
                op.fn()
            try:
                torch.cuda.synchronize()
            except Exception as e:
                print("FAIL", name, sch, getattr(op, "name", "?"), type(op).__name__,
                      getattr(op, "gemm_path", None), net.plan_of(op, sch) if isinstance(op, PN.LinearLayer) else "", e, flush=True)
                sys.exit(1)
        net.verify()
        torch.cuda.synchronize()
        print(name, sch.value, "ok flags", net.flags(), flush=True)
    meas = NP.profile(net, 3)
    torch.cuda.synchronize()
    print(name, "profile ok", flush=True)
    for pol, g in NP.policy_graphs(net, [PN.Scheme.GLOBAL_ABFT] * len(net.layers)).items():
        g.replay(); torch.cuda.synchronize(); print(name, "graph", pol, "ok", net.flags(), flush=True)
    g = NP.capture(net.forward_glue); g.replay(); torch.cuda.synchronize(); print("glue ok", flush=True)
