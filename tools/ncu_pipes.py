"""Per-kernel pipe / unit utilisation and stall breakdown from an ncu report's raw page.
usage: python tools/ncu_pipes.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:60], r[hdr.index("gpu__time_duration.sum")], units[hdr.index("gpu__time_duration.sum")])
    items = []
    for i, h in enumerate(hdr):
        v = r[i].replace(",", "")
        try:
            f = float(v)
        except ValueError:
            continue
        if ("pct_of_peak_sustained_active" in h and ("pipe" in h or "throughput" in h)) or \
                h.startswith("smsp__average_warp_latency_issue_stalled") or \
                h.startswith("smsp__average_warps_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled"):
            items.append((f, h))
    for f, h in sorted(items, reverse=True)[:40]:
        print(f"   {f:12.3f}  {h}")
