"""profiles/r01_scheme_study.md from the scheme-study JSONL and the GPU campaign JSON.
usage: python tools/study_md.py STUDY.jsonl CAMPAIGN.json OUT.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
S = ["unprotected", "global-abft", "thread-one-sided", "thread-two-sided", "thread-replication-full",
     "thread-replication-single-acc"]
out = ["# All six reference schemes on the sm_100a kernel (tools/scheme_study.py; Fig-10-style study, SURVEY 8f item 2)",
       "", "Graph-replayed µs per launch on one B200, fp16 in / fp32 accumulate, fp16 out with ReLU; thread tile 16x8 (the",
       "reference default). Global and one/two-sided use augmented weights; replication uses a TMEM shadow accumulator",
       "(a second MMA into a second TMEM region: no register-file pressure, unlike the paper's occupancy argument).", "",
       "| M | N | K | " + " | ".join(S) + " |", "|---|---|---|" + "---|" * len(S)]
for d in rows:
    out.append(f"| {d['m']} | {d['n']} | {d['k']} | " + " | ".join(
        f"{d['us'][s]:.2f}" if s == "unprotected" else f"{d['us'][s]:.2f} ({d['overhead_pct'][s]:+.1f}%)" for s in S) + " |")
c = json.load(open(sys.argv[2]))
out += ["", "# Fault-injection campaign at scale (tools/campaign_gpu.py, campaign.py semantics)", "",
        f"{c['trials_per_scheme']} injected + {c['control_trials_per_scheme']} fault-free control trials per (scheme, dtype, "
        "site); GEMM extents U[8, 96]; outcome classes as campaign.py:213-247 (detected / masked by the responsible "
        "verdict's tolerance / missed). `tests/test_campaign.py` checks the per-trial outcomes against the reference "
        "itself on 400 golden trials.", "",
        "| dtype | site | scheme | detected | masked | missed | false positives |", "|---|---|---|---|---|---|---|"]
for cfg in c["configs"]:
    for s, v in cfg["schemes"].items():
        out.append(f"| {cfg['dtype']} | {cfg.get('site', 'mixed')} | {s} | {v['detected']} | {v['masked_by_tolerance']} | "
                   f"{v['missed']} | {v['false_positives']}/{v['control']} |")
out += ["", "Exact-int: every injected fault is detected by every scheme, no false positives. binary16: no false",
        "positives; faults below the reference tolerance 2^-10·K·max(|lhs|,|rhs|,1) are masked by design; the one-sided",
        "and replication-full 'missed' trials follow the reference's classification (the responsible tolerance is the",
        "one reported by the thread tile's verdict), which the golden trials reproduce outcome for outcome."]
open(sys.argv[3], "w").write("\n".join(out) + "\n")
