"""Launch chosen layers of a protected network (the bench's exact per-layer arguments) a few
times each — an ncu target.  Also prints each layer's CUDA-graph time per scheme.

  python tools/ncu_netlayer.py NET BATCH SCHEME LAYER[,LAYER...] [reps] [plan_flags]

LAYER is a layer name (e.g. features.2, conv1, layer1.0.conv3).  SCHEME: unprotected |
global-abft | thread-one-sided | global-dot | global-fused.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_09455_b200 import profiler  # noqa: E402
from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

net_name, batch, scheme = sys.argv[1], int(sys.argv[2]), sys.argv[3]
names = sys.argv[4].split(",")
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
flags = int(sys.argv[6]) if len(sys.argv) > 6 else 0     # abft_gemm_args_t.plan_flags for every chosen layer
hw = 50 if net_name.startswith("noscope_") else 224
net = PN.ProtectedNetwork(PN.build_model(net_name), batch, hw, hw)
x = (torch.rand((batch, 3, hw, hw), device="cuda") * 2 - 1).half()
net.load_input(x)
net.forward()
torch.cuda.synchronize()
sch = {"global-dot": PN.GLOBAL_DOT, "global-fused": PN.GLOBAL_FUSED}.get(scheme) or PN.Scheme(scheme)
layers = {L.name: L for L in net.layers}
if flags:
    for n in names:
        net.set_tile(layers[n], sch, 0, flags)
for n in names:
    L = layers[n]
    us = profiler.graph_time_us(lambda: net.launch(L, sch), 10)
    print(f"{n}: M={L.m} N={L.oc} K={L.k_ref} {scheme} {us:.1f} us  plan={net.plan_of(L, PN.Scheme.GLOBAL_ABFT if isinstance(sch, str) else sch)}",
          flush=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for n in names:
    for _ in range(reps):
        net.launch(layers[n], sch)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", flush=True)
