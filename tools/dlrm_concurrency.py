"""Do the 24 DLRM chains of the C2 step overlap as parallel graph branches?  Times the captured
step with the chains on parallel streams vs one stream, and a single chain alone.
  python tools/dlrm_concurrency.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09455_b200 as P  # noqa: E402
from paper_2104_09455_b200.network import ChainGroup  # noqa: E402
from tools import dlrm_secondary as DS  # noqa: E402

S = P.Scheme
mlps, inputs = DS.workload()
wt = {name: [torch.from_numpy(w).cuda() for w in ws] for name, ws in mlps.items()}
keys = list(inputs)


def capture(grp, parallel=True):
    main = torch.cuda.Stream()
    streams = [torch.cuda.Stream() for _ in grp.chains]
    main.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(main):
        grp.forward()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        grp.begin()
        for s, ch in zip(streams, grp.chains):
            if parallel:
                s.wait_stream(main)
                with torch.cuda.stream(s):
                    ch.forward()
                main.wait_stream(s)
            else:
                ch.forward()
        grp.end()
    torch.cuda.synchronize()
    return g


def timeit(g, n=30):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


for pol in (S.UNPROTECTED, S.GLOBAL_ABFT):
    grp = ChainGroup([(wt[k[0]], k[1], [pol] * 3) for k in keys])
    for k, ch in zip(keys, grp.chains):
        ch.x.copy_(torch.from_numpy(inputs[k]).cuda())
    print(pol.value, "parallel branches", round(timeit(capture(grp, True)), 1), "us", flush=True)
    print(pol.value, "one stream", round(timeit(capture(grp, False)), 1), "us", flush=True)
    one = ChainGroup([(wt["bottom"], 1, [pol] * 3)])
    print(pol.value, "one chain (bottom b1)", round(timeit(capture(one, False)), 1), "us", flush=True)
    big = ChainGroup([(wt["top"], 2048, [pol] * 3)])
    print(pol.value, "one chain (top b2048)", round(timeit(capture(big, False)), 1), "us", flush=True)
