"""Stall-reason breakdown of the SASS lines executed exactly `ex` times (one code region) in an ncu report.
usage: python tools/ncu_stalls.py REP [ex ...]   (no ex: list the most-sampled execution counts)"""
import csv, os, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(hdr) and "Instructions Executed" not in r]
iex, ist, isrc = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
if len(sys.argv) == 2:
    agg = defaultdict(lambda: [0, 0])
    for r in body:
        agg[int(r[iex] or 0)][0] += int(r[ist] or 0)
        agg[int(r[iex] or 0)][1] += 1
    top = sorted(agg.items(), key=lambda x: -x[1][0])[:12]
    for ex, (st, n) in top:
        print(f"ex={ex:9d} samples={st:6d} instructions={n}")
    exs = [ex for ex, _ in top[:4]]
else:
    exs = list(map(int, sys.argv[2:]))
for ex in exs:
    tot = defaultdict(int)
    top = []
    for r in body:
        if int(r[iex] or 0) != ex:
            continue
        for i in stall_cols:
            tot[hdr[i]] += int(r[i] or 0)
        top.append((int(r[ist] or 0), r[isrc][:80]))
    print(f"ex={ex}: " + ", ".join(f"{k[6:]}={v}" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
    # (STALL_ORDER=1: every sampled line of the region in program order, with its top stall reason)
    if os.environ.get("STALL_ORDER"):
        for r in body:
            if int(r[iex] or 0) == ex and int(r[ist] or 0) > 0:
                why = max(stall_cols, key=lambda i: int(r[i] or 0))
                print(f"   {int(r[ist]):5d} {hdr[why][6:18]:12s} {r[isrc][:90]}")
        continue
    for st, src in sorted(top, reverse=True)[:int(os.environ.get("STALL_TOP", "12"))]:
        print(f"   {st:5d}  {src}")
