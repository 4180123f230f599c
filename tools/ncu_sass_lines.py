"""SASS-level instruction counts of an ncu report, attributed to CUDA source
lines: python tools/ncu_sass_lines.py rep.ncu-rep  (prints (file, line, sass, count))."""
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, cur, rows = None, None, None, []
    for row in csv.reader(io.StringIO(out)):
        if len(row) >= 2 and row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row and row[0] == "Line No":
            hdr = row
            continue
        if not hdr or len(row) != len(hdr):
            continue
        if row[0]:
            cur = (fname, int(row[0]))
            continue
        if not row[2].startswith("0x"):
            continue
        rows.append({"src": cur, "addr": int(row[2], 16), "sass": row[3].strip(), "inst": int(row[7] or 0),
                     "samples": int(row[4] or 0), "threads": float(row[10] or 0) if len(row) > 10 else 0.0})
    return rows


if __name__ == "__main__":
    for r in sorted(load(sys.argv[1]), key=lambda r: r["addr"]):
        print(f"{r['addr'] & 0xfffff:6x} {r['inst']:10d} {r['samples']:6d} {r['src'][0]}:{r['src'][1]:<5d} {r['sass']}")
