"""Bring-up: per-layer global verdicts of a protected network vs torch-computed (lhs, rhs)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2104_09455_b200 import protected_network as PN
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_network import _logical, _input

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 2
net = PN.ProtectedNetwork(PN.build_model(name), b, schemes=PN.Scheme.GLOBAL_ABFT)
x = _input(b)
net.forward(x)
torch.cuda.synchronize()
vs = net.verdicts()
print("flags", net.flags())
for L, v in list(zip(net.layers, vs))[:12]:
    xi = _logical(L.x).double()
    if L.kind == "fc":
        xi = xi.reshape(xi.shape[0], -1, 1, 1)
    wq = L.weight.half().double()
    pre = F.conv2d(xi, wq, None, stride=L.stride, padding=L.pad)
    rhs0 = float(pre.sum())
    bsum = float(L.bias.double().sum()) * L.m if L.bias is not None else 0.0
    print(f"{L.index:3d} {L.name:24s} m={L.m} oc={L.oc} k={L.k_ref} gemm={L.gemm_path} | lhs {v.lhs:.6e} rhs {v.rhs:.6e} "
          f"tol {v.tolerance_used:.3e} det {v.detected} | torch sum(AW) {rhs0:.6e} + M*sum(b) {bsum:.6e} = {rhs0 + bsum:.6e}")
