"""Why a fused-global launch times slower than the unprotected one in graph replay: the same layer
and plan under variants of the global arguments.  python tools/fused_vs_unprot.py NET LAYER FLAGS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_09455_b200 import kernels, profiler  # noqa: E402
from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

S = PN.Scheme
name, lname, flags = sys.argv[1], sys.argv[2], int(sys.argv[3])
net = PN.ProtectedNetwork(PN.build_model(name), 256)
net.load_input((torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1).half())
L = {x.name: x for x in net.layers}[lname]
net.set_global_variant(L, "fused")
for key in (S.UNPROTECTED, PN.GLOBAL_FUSED):
    net.set_tile(L, key, 0, flags)
net.forward()
torch.cuda.synchronize()
osum = torch.zeros(1, dtype=torch.float64, device="cuda")
res = {}


def run(tag, scheme, kw):
    _, a, _ = net._launch_args(L, scheme, kw)
    res[tag] = profiler.graph_time_us(lambda: kernels.conv2d(a), 10)


run("unprotected", S.UNPROTECTED, net._kw(L, S.UNPROTECTED))
kw = net._kw(L, PN.GLOBAL_FUSED)
run("fused (out_partials)", S.GLOBAL_ABFT, kw)
kw2 = dict(kw)
kw2.pop("out_partials")
kw2["out_sum"] = osum
run("fused (out_sum atomics)", S.GLOBAL_ABFT, kw2)
run("unprotected again", S.UNPROTECTED, net._kw(L, S.UNPROTECTED))
print(lname, flags, {k: round(v, 1) for k, v in res.items()}, flush=True)
