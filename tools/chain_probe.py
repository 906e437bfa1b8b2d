"""Time single DLRM chains (bench.py workload) under several schemes / debug variants.
usage: python tools/chain_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_09455_b200 as P
from paper_2104_09455_b200.network import ProtectedChain
from paper_2104_09455_b200.profiler import graph_time_us

S = P.Scheme
mlps, inputs = bench.workload()
wt = {k: [torch.from_numpy(w).cuda() for w in ws] for k, ws in mlps.items()}
for key in [("top", 2048), ("bottom", 2048), ("top", 64), ("bottom", 1)]:
    res = {}
    for name, sch, env, noverify in [("unprot", S.UNPROTECTED, "", False), ("global", S.GLOBAL_ABFT, "", False),
                                     ("global-noverify", S.GLOBAL_ABFT, "", True),
                                     ("global-nolhsld", S.GLOBAL_ABFT, "524288", False),
                                     ("thread", S.THREAD_ONE_SIDED, "", False)]:
        if env:
            os.environ["ABFT_DEBUG"] = env
        ch = ProtectedChain(wt[key[0]], key[1], [sch] * 3)
        ch.x.copy_(torch.from_numpy(inputs[key]).cuda())
        if noverify:
            ch.global_ids = []
        res[name] = graph_time_us(ch.forward, 200)
        os.environ.pop("ABFT_DEBUG", None)
    base = res["unprot"]
    print(key, " ".join(f"{k}={v:6.2f}({100 * (v / base - 1):+5.1f}%)" for k, v in res.items()), flush=True)
