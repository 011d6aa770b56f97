"""Hot SASS lines of an ncu report (needs --import-source / -lineinfo).

usage: python scripts/ncu_source_hot.py report.ncu-rep [top=40]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
tot_i = sum(int(d["Instructions Executed"] or 0) for d in data)
print(f"instructions executed (warp-level): {tot_i}, stall samples: {tot_s}, sass lines: {len(data)}")
for i, d in enumerate(data):
    d["idx"] = i
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    print(f"{d['idx']:5d} {d['Warp Stall Sampling (All Samples)']:>6s} {d['Instructions Executed']:>10s}  {d['Source'][:90]}")
