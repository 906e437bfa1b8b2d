"""Isolated timings of one network layer under several launch configurations (bring-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2104_09455_b200 import protected_network as PN
from paper_2104_09455_b200.profiler import graph_time_us

name, b, idx = sys.argv[1], int(sys.argv[2]), [int(v) for v in sys.argv[3].split(",")]
net = PN.ProtectedNetwork(PN.build_model(name), b)
net.load_input((torch.rand((b, 3, 224, 224), device="cuda") * 2 - 1).half())
net.forward(); torch.cuda.synchronize()
S = PN.Scheme
for i in idx:
    L = net.layers[i]
    print(L.name, L.m, L.oc, L.k_ref, flush=True)
    cfgs = [("un", S.UNPROTECTED, 0, 0), ("un-nokp", S.UNPROTECTED, 0, 1), ("un-dbl", S.UNPROTECTED, 0, 4), ("un-padb", S.UNPROTECTED, 0, 2), ("gl", S.GLOBAL_ABFT, 0, 0),
            ("gl-nokp", S.GLOBAL_ABFT, 0, 1), ("dot", PN.GLOBAL_DOT, 0, 0), ("one", S.THREAD_ONE_SIDED, 0, 0)]
    for t in (64, 128, 192, 256):
        cfgs.append((f"un-t{t}", S.UNPROTECTED, t, 0))
    res = {}
    for rep in range(3):
        for nm, key, tn, fl in cfgs:
            try:
                net.set_tile(L, key, tn, fl)
            except Exception as e:
                res.setdefault(nm, []).append(str(e)[:40]); continue
            try:
                res.setdefault(nm, []).append(round(graph_time_us(lambda: net.launch(L, key), 5), 1))
            except Exception as e:
                res.setdefault(nm, []).append(str(e)[:40])
                torch.cuda.synchronize()
    for nm, v in res.items():
        print(f"   {nm:10s} {v}", flush=True)
