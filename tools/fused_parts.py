"""Split a fused-global layer's time into its launches (the conv kernel with output summation only,
the producer's border buckets, the window lhs):  python tools/fused_parts.py NET LAYER [flags]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_09455_b200 import kernels, profiler  # noqa: E402
from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

S = PN.Scheme
name, lname = sys.argv[1], sys.argv[2]
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
net = PN.ProtectedNetwork(PN.build_model(name), 256)
net.load_input((torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1).half())
L = {x.name: x for x in net.layers}[lname]
net.set_global_variant(L, "fused")
for key in (S.UNPROTECTED, PN.GLOBAL_FUSED):
    net.set_tile(L, key, 0, flags)
net.forward()
torch.cuda.synchronize()
P, x = L.producer, L.x
kind, args = L.args[PN.GLOBAL_FUSED]
ukind, uargs = L.args[S.UNPROTECTED]
t = {
    "unprotected": profiler.graph_time_us(lambda: kernels.conv2d(uargs), 10),
    "fused kernel": profiler.graph_time_us(lambda: kernels.conv2d(args), 10),
    "border_sums": profiler.graph_time_us(lambda: kernels.border_sums(x.buf, x.n, x.h, x.w, x.cp, x.ld, net.dtype,
                                                                      P._wsum, P.out.cp), 10),
    "window_lhs": profiler.graph_time_us(lambda: kernels.window_lhs(P._wsum, P.out.cp, L.x.cp, L.r, L.s,
                                                                    L._k // (L.r * L.s), L._rowck, L._bias_dev,
                                                                    PN._r8(L.oc), L.m, net.partials[L.index, 0, 0:1]),
                                         10),
    "launch(fused)": profiler.graph_time_us(lambda: net.launch(L, PN.GLOBAL_FUSED), 10),
}
print(lname, flags, {k: round(v, 1) for k, v in t.items()}, flush=True)
