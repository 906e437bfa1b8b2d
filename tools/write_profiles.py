"""Summarise a round's ncu captures (gpurun_out/) into profiles/ (tracked):
  profiles/<TAG>_launches.txt            per-kernel launch list of the bench's timed IG steps
  profiles/<TAG>_ncu_<name>.txt          key counters of each --set full capture
  profiles/dominant.json                 dram bytes / duration of the dominant kernel (read by bench.py)
usage: python tools/write_profiles.py TAG"""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1]
OUT = os.path.join(ROOT, "profiles")
os.makedirs(OUT, exist_ok=True)
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3,
         "msecond": 1e3, "ms": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


dominant = None
for name, desc in (("dominant", "global-abft 2048x512x512 (DLRM top b2048 layer 0, the bench's dominant kernel)"),
                   ("unprot", "unprotected 2048x512x512"), ("onesided", "thread-one-sided 2048x512x512")):
    rep = os.path.join(ROOT, "gpurun_out", f"{name}_{TAG}.ncu-rep")
    if not os.path.exists(rep):
        continue
    m = raw(rep)
    lines = [f"# ncu --set full --clock-control none, {desc}", f"# kernel: {m.get('Kernel Name', ('?',))[0]}"]
    for k in KEYS:
        if k in m:
            lines.append(f"{k} = {m[k][0]} {m[k][1]}")
    with open(os.path.join(OUT, f"{TAG}_ncu_{name}.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if name == "dominant":
        def num(k):
            v, u = m[k]
            return float(v.replace(",", "")) * SCALE.get(u, 1)
        dominant = dict(tag=TAG, config=dict(m=2048, n=512, k=512, scheme="global-abft"),
                        dram_bytes_read=num("dram__bytes_read.sum"), dram_bytes_write=num("dram__bytes_write.sum"),
                        gpu_time_us_cold=num("gpu__time_duration.sum"), source=f"profiles/{TAG}_ncu_dominant.txt")
if dominant:
    with open(os.path.join(OUT, "dominant.json"), "w") as fh:
        json.dump(dominant, fh, indent=1)
lp = os.path.join(ROOT, "gpurun_out", f"launches_{TAG}.csv")
if os.path.exists(lp):
    s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), lp], capture_output=True,
                       text=True).stdout
    with open(os.path.join(OUT, f"{TAG}_launches.txt"), "w") as fh:
        fh.write("# ncu --nvtx --nvtx-include timed_ig/ --metrics gpu__time_duration.sum (cold, serialised):\n"
                 "# python bench.py --steps 2 --warmup 3 --plan-json <plans of the timed run>\n" + s)
print("profiles written for", TAG)
