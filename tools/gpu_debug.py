"""Stepwise GPU bring-up of the sm_100a kernels (run under `timeout`)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P

def check(m, n, k, scheme=P.Scheme.UNPROTECTED, tiling=P.TilingConfig(), dtype=torch.float16):
    g = torch.Generator(device="cuda").manual_seed(1)
    a = (torch.rand((m, k), generator=g, device="cuda") * 2 - 1).to(dtype)
    b = (torch.rand((k, n), generator=g, device="cuda") * 2 - 1).to(dtype)
    t0 = time.time()
    rep = P.execute(a, b, tiling, scheme)
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    err = (rep.output - ref).abs().max().item()
    print(f"{m}x{n}x{k} {scheme.value}: maxerr {err:.3e} detected {rep.detected} nverd {len(rep.verdicts)} "
          f"({time.time()-t0:.2f}s)", flush=True)
    if err > 1e-2:
        print("  ref[:2,:8]", ref[:2, :8].tolist()); print("  out[:2,:8]", rep.output[:2, :8].tolist())
    return err

check(128, 128, 64)
check(128, 128, 128)
check(256, 256, 256)
check(1, 512, 13)
check(300, 200, 1000)
check(2048, 2048, 2048)
for s in P.Scheme:
    check(256, 256, 256, s)
check(512, 384, 320, P.Scheme.THREAD_ONE_SIDED, dtype=torch.bfloat16)
print("DEBUG DONE")
