"""Network-level intensity-guided ABFT on B200 (configs C3-C5): per-layer timings under
unprotected / global / thread-one-sided, the reference selector (cost.select) fed with them,
and the per-network overhead of IG vs always-global vs always-thread-level.

usage: python tools/netbench.py [--nets resnet50,vgg16,...] [--configs hd1,b64,b256] [--out FILE]
Prints one JSON object per (network, config) and writes them all to --out.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"hd1": (1, 1080, 1920), "b1": (1, 224, 224), "b64": (64, 224, 224), "b256": (256, 224, 224)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", default="resnet50,vgg16,alexnet,squeezenet1_0,shufflenet_v2_x1_0")
    ap.add_argument("--configs", default="hd1,b64,b256")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cudnn", action="store_true", help="also time torch/cuDNN conv2d (channels_last fp16)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "netbench.jsonl"))
    ap.add_argument("--layers", default="", help="comma-separated layer indices (bring-up)")
    args = ap.parse_args()

    import torch
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import networks, profiler
    from paper_2104_09455_b200.convnet import LayerRunner
    from paper_2104_09455_b200.shapes import DeviceProfile

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6535.1, "bf16_tflops": 1636.2, "sm_max_mhz": 1965}
    dev = DeviceProfile(name="B200", tensor_throughput=peaks["bf16_tflops"] * 1e12,
                        alu_throughput=148 * 128 * 2 * peaks.get("sm_max_mhz", 1965) * 1e6,
                        memory_bandwidth=peaks["hbm_gbs"] * 1e9, verification_launch_latency=0.0)
    S = P.Scheme
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    results = []
    for net in args.nets.split(","):
        for cfg in args.configs.split(","):
            b, h, w = CONFIGS[cfg]
            specs = networks.capture(net, b, h, w)
            if args.layers:
                keep = {int(x) for x in args.layers.split(",")}
                specs = [sp for sp in specs if sp.index in keep]
            t0 = time.time()
            rows = []
            for spec in specs:
                print(f"# {net} {cfg} layer {spec.index}: {spec}", file=sys.stderr, flush=True)
                r = LayerRunner(spec)
                it = args.iters if r.flops() < 2e11 else max(3, args.iters // 4)
                t_un = profiler.graph_time_us(lambda: r.conv(S.UNPROTECTED), it)
                t_glf = profiler.graph_time_us(lambda: r.conv(S.GLOBAL_ABFT), it)        # checksum N-slice
                t_gld = profiler.graph_time_us(lambda: r.conv_variant("global-dot"), it)  # checksum-warp dot
                t_gls = profiler.graph_time_us(r.global_standalone, it)                  # + standalone pass
                t_ck = profiler.graph_time_us(r.colck_pass, it)
                t_gl = min(t_glf, t_gld, t_gls)
                t_one = profiler.graph_time_us(lambda: r.conv(S.THREAD_ONE_SIDED), it)
                row = dict(i=spec.index, kind=spec.kind, m=r.m, n=spec.oc, k=r.k_ref, r=spec.r, stride=spec.stride_h,
                           cin=spec.cin, t_un=t_un, t_gl=t_gl, t_gl_fused=t_glf, t_gl_standalone=t_gls, t_ck=t_ck,
                           t_gl_dot=t_gld, t_one=t_one,
                           global_variant=min((t_glf, "fused"), (t_gld, "dot"), (t_gls, "standalone"))[1])
                if args.cudnn:
                    x = torch.randn(spec.n, spec.cin, spec.h, spec.w, device="cuda", dtype=torch.float16) \
                        .to(memory_format=torch.channels_last)
                    wt = torch.randn(spec.oc, spec.cin, spec.r, spec.s, device="cuda", dtype=torch.float16) \
                        .to(memory_format=torch.channels_last)
                    row["t_cudnn"] = profiler.graph_time_us(
                        lambda: torch.nn.functional.conv2d(x, wt, stride=(spec.stride_h, spec.stride_w),
                                                           padding=(spec.pad_h, spec.pad_w)), it)
                    del x, wt
                rows.append(row)
                del r
                torch.cuda.empty_cache()
            # one batched verification launch for the whole network, shared by its global layers
            r0 = LayerRunner(specs[-1])
            t_ver = profiler.graph_time_us(r0.verify, args.iters)
            del r0
            L = len(rows)
            meas = {}
            for row in rows:
                i = row["i"]
                meas[(i, S.UNPROTECTED)] = row["t_un"] * 1e-6
                meas[(i, S.GLOBAL_ABFT)] = (row["t_gl"] + t_ver / L) * 1e-6     # activation checksum fused
                meas[(i, S.THREAD_ONE_SIDED)] = row["t_one"] * 1e-6
            layers = [(row["i"], P.GemmShape(row["m"], row["n"], row["k"])) for row in rows]
            plan = P.select(layers, P.BINARY16, dev, measured=P.MeasuredTimings(entries=meas))
            chosen = [lp.chosen for lp in plan.layers]
            t_o = sum(meas[(i, S.UNPROTECTED)] for i, _ in layers)
            t_g = sum(meas[(i, S.GLOBAL_ABFT)] for i, _ in layers)
            t_t = sum(meas[(i, S.THREAD_ONE_SIDED)] for i, _ in layers)
            t_ig = sum(meas[(i, c)] for (i, _), c in zip(layers, chosen))
            flops = sum(2 * row["m"] * row["n"] * row["k"] for row in rows)
            res = dict(net=net, config=cfg, batch=b, h=h, w=w, layers=L, gflop=flops / 1e9,
                       t_unprotected_us=t_o * 1e6, t_global_us=t_g * 1e6, t_thread_us=t_t * 1e6, t_ig_us=t_ig * 1e6,
                       overhead_pct=dict(global_=100 * (t_g / t_o - 1), thread=100 * (t_t / t_o - 1),
                                         ig=100 * (t_ig / t_o - 1)),
                       unprotected_tflops=flops / t_o / 1e12, protected_ig_tflops=flops / t_ig / 1e12,
                       plan=[c.value for c in chosen], verify_us=t_ver, per_layer=rows,
                       wall_s=round(time.time() - t0, 1))
            if args.cudnn:
                res["t_cudnn_us"] = sum(row["t_cudnn"] for row in rows)
            results.append(res)
            brief = {k: v for k, v in res.items() if k != "per_layer"}
            print(json.dumps(brief), flush=True)
            with open(args.out, "a") as fh:
                fh.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
