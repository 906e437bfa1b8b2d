"""In-kernel %globaltimer stamps (ABFT_DEBUG=2048) for small protected GEMMs, eager and in a graph."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2104_09455_b200 as P
from paper_2104_09455_b200 import device as D, kernels, _lib
lib = _lib.load()
m, n, k = 1, 512, 16
a = (torch.rand((m, k), device="cuda") - 0.5).half(); b = (torch.rand((k, n), device="cuda") - 0.5).half()
pw = D.prepare_weight(b, P.BINARY16); out = torch.empty((m, n), dtype=torch.float16, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
buf = (ctypes.c_ulonglong * (160 * 8))()
for name, sch, kw in [("unprot", P.Scheme.UNPROTECTED, {}),
                      ("onesided", P.Scheme.THREAD_ONE_SIDED, dict(m_ext=16, n_ext=512, fired_count=cnt))]:
    fn = lambda: kernels.gemm(a, k, pw.bt, pw.ldbt, m, n, k, P.BINARY16, 1, sch, out=out, ldc=n, out_kind="f16",
                              relu=True, **kw)
    for it in range(4):
        fn(); fn(); torch.cuda.synchronize()
        lib.abft_debug_timestamps(buf)
        ts = np.frombuffer(buf, dtype=np.uint64).reshape(160, 8)[:8].astype(np.int64)
        t0 = ts[:, 0].min()
        rel = (ts[:, :7] - t0)
        print(name, it, "entry..setup..tfull..epi_done..exit..ld0..loopdone (ns, max over CTAs):", rel.max(axis=0).tolist(),
              "entry spread", int(rel[:, 0].max()))
    # back-to-back pair: second launch's entry relative to first's exit
