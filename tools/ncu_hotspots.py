"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source=sass`."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[ist] or 0) for r in body)
print("total samples", tot)
for idx, r in sorted(enumerate(body), key=lambda x: -int(x[1][ist] or 0))[:top]:
    print(f"{idx:5d} {int(r[ist]):6d} {100*int(r[ist])/tot:5.1f}% ex={r[iex]:>8}  {r[isrc].strip()[:90]}")
