"""Summary of a one-kernel ncu --set full report (the profiles/ text format), optionally writing
profiles/dominant.json for bench.py's roofline traffic:
  python tools/ncu_layer_summary.py REP "description" [net layer batch scheme [flags variant] -> dominant.json]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep, desc = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (vals[i].replace(",", ""), units[i]) for i, h in enumerate(hdr)}
print(f"# ncu --set full --clock-control none: {desc}")
print(f"# kernel: {m.get('Kernel Name', ('?',))[0]}")
for k in KEYS:
    if k in m:
        print(f"{k} = {m[k][0]} {m[k][1]}")
stalls = []
for h, (v, u) in m.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in stalls) or 1.0
print("# warp-state samples (all warps, incl. idle role warps waiting on barriers): " +
      ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(stalls, reverse=True)[:6]))
if len(sys.argv) > 6:
    net, layer, batch, scheme = sys.argv[3:7]

    def byt(k):
        v, u = m[k]
        return float(v) * SCALE.get(u, 1)
    cfg = {"net": net, "layer": layer, "batch": int(batch), "scheme": scheme}
    if len(sys.argv) > 8:      # the launch's plan: plan_flags and global variant (bench.py matches both)
        cfg.update(flags=int(sys.argv[7]), variant=sys.argv[8])
    dj = {"tag": "r02", "config": cfg,
          "dram_bytes_read": byt("dram__bytes_read.sum"), "dram_bytes_write": byt("dram__bytes_write.sum"),
          "source": f"profiles/r02_ncu_{layer}_{scheme}.txt"}
    with open(os.path.join(ROOT, "gpurun_out", "dominant.json"), "w") as fh:
        json.dump(dj, fh, indent=1)
