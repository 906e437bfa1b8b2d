"""profiles/<name>.md table from a tools/netbench.py JSONL: python tools/netbench_md.py IN.jsonl OUT.md"""
import json
import statistics
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
out = ["# Network-level ABFT overhead on one B200 (tools/netbench.py --configs hd1,b64,b256 --cudnn)",
       "",
       "Per network: the sum of its linear layers' times (PAPER.md:836). Each layer is CUDA-graph timed on its real",
       "input extent under unprotected / global / thread-one-sided; global takes the fastest of its three lhs",
       "variants per layer (checksum N-slice of the augmented weights, checksum-warp dot with rowck(B), standalone",
       "activation checksum pass) plus its share of the network's one verification launch. The intensity-guided",
       "plan is the reference selector (cost.select) fed with these measurements. cuDNN = torch conv2d,",
       "channels_last fp16, dense (reported for scale; not an ABFT baseline).",
       "",
       "| network | config | layers | GFLOP | unprotected us | cuDNN us | global % | thread % | IG % | IG TFLOP/s | global variants (slice/dot/standalone) |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    var = {}
    for r in d["per_layer"]:
        var[r["global_variant"]] = var.get(r["global_variant"], 0) + 1
    vs = "/".join(str(var.get(k, 0)) for k in ("fused", "dot", "standalone"))
    out.append("| %s | %s | %d | %.1f | %.0f | %.0f | %.1f | %.1f | %.1f | %.0f | %s |" % (
        d["net"], d["config"], d["layers"], d["gflop"], d["t_unprotected_us"], d.get("t_cudnn_us", 0),
        d["overhead_pct"]["global_"], d["overhead_pct"]["thread"], d["overhead_pct"]["ig"], d["protected_ig_tflops"], vs))
ig = [d["overhead_pct"]["ig"] for d in rows]
best = sum(1 for d in rows if d["overhead_pct"]["ig"] <= min(d["overhead_pct"]["global_"], d["overhead_pct"]["thread"]) + 1e-9)
out += ["", "Median IG overhead over the %d (network, config) pairs: %.1f %% (max %.1f %%). IG is at or below the better of"
        " always-global and always-thread-level on %d of %d." % (len(ig), statistics.median(ig), max(ig), best, len(rows))]
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out[9:]))
