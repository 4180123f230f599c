"""Per-source-line stall samples and executed instructions from an ncu report
(`--page source --print-source cuda,sass`).  Usage: ncu_lines.py rep [kernel-regex] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["--kernel-name", "regex:" + sys.argv[2]]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
path = None
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    # cuda rows carry a line number in col 0; sass rows have an empty col 0
    if r[0]:
        line = (path, int(r[0]), r[1][:80])
        continue
    try:
        s = float(r[4] or 0)
        e = float(r[7] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(line, [0.0, 0.0])
    a[0] += s
    a[1] += e
tot_s = sum(v[0] for v in agg.values()) or 1
tot_e = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot_s:.0f}  warp-instr {tot_e:.0f}")
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot_s:5.1f}% {100 * e / tot_e:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
