"""Quick per-shape timing of the sm_100a kernels vs cuBLAS (CUDA events, graph-replayed)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels, _lib

def bench(fn, iters=50):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / iters)
    return best

shapes = [(256,256,256),(1,512,16),(2048,512,16),(2048,256,512),(2048,512,512),(2048,1,256),
          (4096,4096,4096),(8192,8192,8192),(12544,64,147+5),(50176,64,576),(3136*64,256,64)]
for (m,n,k) in shapes:
    k8 = D.round8(k)
    a = (torch.rand((m,k8),device="cuda")-0.5).half()
    b = (torch.rand((k8,n),device="cuda")-0.5).half()
    pw = D.prepare_weight(b, P.BINARY16)
    out = torch.empty((m,D.round8(n)),dtype=torch.float16,device="cuda")
    osum = torch.zeros(1,dtype=torch.float64,device="cuda")
    colck = torch.zeros(D.round8(n),dtype=torch.float32,device="cuda")
    cnt = torch.zeros(1,dtype=torch.int32,device="cuda")
    res = {}
    for name, sch, kw in [("unprot", P.Scheme.UNPROTECTED, {}),
                          ("global", P.Scheme.GLOBAL_ABFT, dict(out_sum=osum, next_colck=colck)),
                          ("onesided", P.Scheme.THREAD_ONE_SIDED, dict(fired_count=cnt, m_ext=-(-m//16)*16, n_ext=-(-n//8)*8)),
                          ("onesided_split", P.Scheme.THREAD_ONE_SIDED, dict(fired_count=cnt, ck_split=True, m_ext=-(-m//16)*16, n_ext=-(-n//8)*8)),
                          ("onesided_off", P.Scheme.THREAD_ONE_SIDED, dict(fired_count=cnt, m_ext=-(-m//16)*16, n_ext=-(-n//8)*8, offline=True))]:
        offline = kw.pop("offline", False)
        if offline:
            plan = kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                                ldc=out.stride(0), out_kind="f16", relu=True, plan_only=True, **kw)
            kw["ck_rows"] = kernels.ck_rows(pw.bt, n, k8, P.BINARY16, plan, 8, False)
        fn = lambda: kernels.gemm(a, k8, pw.bt, pw.ldbt, m, n, k8, P.BINARY16, _lib.NUM_BINARY16, sch, out=out,
                                  ldc=out.stride(0), out_kind="f16", relu=True, **kw)
        res[name] = bench(fn)
    ref = bench(lambda: torch.matmul(a, b))
    fl = 2*m*n*k8
    print(f"{m}x{n}x{k8}: unprot {res['unprot']:.2f}us ({fl/res['unprot']/1e6:.0f} TF) global {res['global']:.2f} "
          f"({100*(res['global']/res['unprot']-1):+.1f}%) 1sided {res['onesided']:.2f} ({100*(res['onesided']/res['unprot']-1):+.1f}%) "
          f"split {res['onesided_split']:.2f} offline {res['onesided_off']:.2f} ({100*(res['onesided_off']/res['unprot']-1):+.1f}%) cublas {ref:.2f}us ({fl/ref/1e6:.0f} TF)", flush=True)
