"""Summarise an ncu report: key SOL / occupancy / pipe / stall metrics per kernel."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
want = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for r in rows[1:]:
    if len(r) <= vi: continue
    if want is None or any(w.lower() in r[mi].lower() for w in want):
        print(r[ki].split("(")[0][-28:], "|", r[si][:22], "|", r[mi], "=", r[vi], r[ui])
