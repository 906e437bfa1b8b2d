"""Per fused-eligible layer of a network: the global variants' times and the producer's window-sum
cost (what netprofile.profile charges): python tools/fused_probe.py NET [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_09455_b200 import netprofile, profiler  # noqa: E402
from paper_2104_09455_b200 import protected_network as PN  # noqa: E402

S = PN.Scheme
name = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
net = PN.ProtectedNetwork(PN.build_model(name), batch)
net.load_input((torch.rand((batch, 3, 224, 224), device="cuda") * 2 - 1).half())
net.forward()
torch.cuda.synchronize()
for L in net.layers:
    if L.producer is None:
        continue
    t = {k: profiler.graph_time_us(lambda k=k: net.launch(L, k, deferred=True), 10)
         for k in (S.UNPROTECTED, S.GLOBAL_ABFT, PN.GLOBAL_DOT, PN.GLOBAL_FUSED)}
    P = L.producer
    if isinstance(P, PN.PoolProducer):
        t_off = profiler.graph_time_us(P.run, 10)
        P.ws_active = True
        t_on = profiler.graph_time_us(P.run, 10)
        P.ws_active = False
    else:
        t_off = profiler.graph_time_us(lambda: net.launch(P, S.UNPROTECTED), 10)
        P.ws_active = True
        P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
        t_on = profiler.graph_time_us(lambda: net.launch(P, S.UNPROTECTED), 10)
        P.ws_active = False
        P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
    print(f"{L.name:24s} unprot {t[S.UNPROTECTED]:8.1f} slice {t[S.GLOBAL_ABFT]:8.1f} dot {t[PN.GLOBAL_DOT]:8.1f} "
          f"fused {t[PN.GLOBAL_FUSED]:8.1f} (+batched {netprofile._batched_share(L):.1f})  producer {P.name} "
          f"{t_off:.1f} -> {t_on:.1f} (ws_mode {P.ws_mode})",
          flush=True)
