"""Chain timing vs launch plumbing: PDL on/off, memset node on/off, single kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import network, kernels
from paper_2104_09455_b200.network import ProtectedChain
from paper_2104_09455_b200.profiler import graph_time_us

S = P.Scheme
mlps, inputs = bench.workload()
wt = {k: [torch.from_numpy(w).cuda() for w in ws] for k, ws in mlps.items()}
for key in [("top", 2048), ("bottom", 1)]:
    out = []
    for name in ["base", "nopdl", "nomemset", "nopdl-nomemset"]:
        network._NO_PDL = "nopdl" in name
        ch = ProtectedChain(wt[key[0]], key[1], [S.UNPROTECTED] * 3)
        ch.x.copy_(torch.from_numpy(inputs[key]).cuda())
        if "nomemset" in name:
            ch.scratch = None
        out.append(f"{name}={graph_time_us(ch.forward, 300):6.2f}")
    # single layers
    ch = ProtectedChain(wt[key[0]], key[1], [S.UNPROTECTED] * 3)
    for i, L in enumerate(ch.layers):
        kw = ch._gemm_kwargs(i, L)
        a = ch.x if i == 0 else ch.acts[i - 1]
        t = graph_time_us(lambda: kernels.gemm(a, a.stride(0), L.pw.bt, L.pw.ldbt, ch.batch, L.n, L.k, ch.dtype,
                                               ch.numeric, L.scheme, **kw), 300)
        out.append(f"L{i}={t:6.2f}")
    t = graph_time_us(lambda: kernels.zero(ch.scratch), 300)
    out.append(f"memset={t:5.2f}")
    print(key, " ".join(out), flush=True)
