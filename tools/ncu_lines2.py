"""Per-source-line instruction counts and stall samples from an ncu report
(`--page source --print-source cuda,sass`): python tools/ncu_lines2.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
import os
kf = os.environ.get("NCU_KERNEL")
out = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + kf] if kf else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, res = None, None, []
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr and len(row) == len(hdr) and row[0]:
        try:
            ie, s = int(row[7] or 0), int(row[4] or 0)
        except ValueError:
            continue
        res.append((ie, s, fname, row[0], row[1].strip()[:100]))
tot = sum(r[0] for r in res) or 1
ts = sum(r[1] for r in res) or 1
print(f"total warp instructions {tot}  stall samples {ts}")
for r in sorted(res, key=lambda r: -r[0])[:top]:
    print(f"{r[0] / 1e6:8.2f}M {100 * r[0] / tot:5.1f}%  samp {100 * r[1] / ts:5.1f}%  {r[2]}:{r[3]}  {r[4]}")
