"""Summarise an ncu report: key counters (+ optional grep pattern) for each profiled kernel."""
import csv, subprocess, sys
rep = sys.argv[1]
pat = sys.argv[2:] or []
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__average_warp_latency_issue_stalled"]
for r in rows[2:]:
    for i, h in enumerate(hdr):
        if h in KEYS or any(p in h for p in pat):
            print(f"{h} = {r[i]} {units[i]}")
    print("--")
