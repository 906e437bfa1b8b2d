timeout 600 python -m pytest tests/test_gpu_network.py -x -q -k fused > gpurun_out/t_15.log 2>&1; tail -2 gpurun_out/t_15.log
cat > /tmp/fz.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2104_09455_b200 import protected_network as PN, profiler
S = PN.Scheme
net = PN.ProtectedNetwork(PN.build_model("vgg16"), 256)
x = (torch.rand((256, 3, 224, 224), device="cuda") * 2 - 1).half()
net.load_input(x); net.forward(); torch.cuda.synchronize()
L = {l.name: l for l in net.layers}
for n in ("features.12", "features.14", "features.19"):
    l = L[n]
    for key in (S.UNPROTECTED, S.GLOBAL_ABFT, PN.GLOBAL_DOT, PN.GLOBAL_FUSED):
        us = profiler.graph_time_us(lambda: net.launch(l, key), 10)
        pl = net.plan_of(l, S.GLOBAL_ABFT if key != S.UNPROTECTED else key)
        print(n, key if isinstance(key, str) else key.value, round(us, 1), pl["tile_n"], pl["stages"], flush=True)
    P = l.producer
    t0 = profiler.graph_time_us(lambda: net.launch(P, S.UNPROTECTED), 10)
    P.ws_active = True; P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
    t1 = profiler.graph_time_us(lambda: net.launch(P, S.UNPROTECTED), 10)
    P.ws_active = False; P.args[S.UNPROTECTED] = net._make_args(P, S.UNPROTECTED)
    print("  producer", P.name, round(t0, 1), "with window sums", round(t1, 1), flush=True)
PY

ABFT_TRACE=1 timeout 600 python /tmp/fz.py 2>&1 | grep "^\[abft\]" | grep "N=256 K=2304\|N=256 K=1152" | sort -u | head
