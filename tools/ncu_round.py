"""Summaries of the round's ncu captures -> profiles/<round>/ (text) and the
per-kernel DRAM traffic / utilisation tables bench.py attaches to its roofline
objects (profiles/ncu_traffic.json, profiles/ncu_util.json).
Usage: python tools/ncu_round.py <dir with .ncu-rep files> <profiles/rNN>"""
import csv
import json
import os
import subprocess
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_slots_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "shared_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
}


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        if "<" in name.split("(")[0]:
            short += "<" + name.split("(")[0].split("<", 1)[1]
        vals = {}
        for k, m in METRICS.items():
            if m in h:
                try:
                    j = h.index(m)
                    vals[k] = float(r[j].replace(",", "")) * scale.get(units[j], 1.0)
                except ValueError:
                    pass
        stalls = {c.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[h.index(c)] or 0)
                  for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        vals["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        res.append((short, vals))
    return res


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tpath, upath = (os.path.join(root, "profiles", f) for f in ("ncu_traffic.json", "ncu_util.json"))
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    util = json.load(open(upath)) if os.path.exists(upath) else {}
    lines = []
    for f in sorted(os.listdir(src)):
        if not f.endswith(".ncu-rep"):
            continue
        for short, v in kernels(os.path.join(src, f)):
            key = short.split("<")[0] if "steady" not in f else short.split("<")[0]
            lines.append(f"## {f}: {short}")
            for k, x in v.items():
                lines.append(f"  {k} = {x}")
            by = v.get("dram_read_bytes", 0) + v.get("dram_write_bytes", 0)
            tag = key + ("<true>" if "<1>" in short and "raster" in short else "")
            traffic[tag] = int(by)
            util[tag] = {k: v[k] for k in ("issue_slots_busy_pct", "fma_pipe_pct", "alu_pipe_pct", "xu_pipe_pct",
                                          "lsu_pipe_pct", "shared_wavefronts_pct", "warps_active_pct", "dram_pct",
                                          "duration_us", "inst_executed") if k in v}
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full capture per "
                        "kernel (profiles/r02/ncu_summary.txt); the upscalers are captured in steady state with "
                        "--cache-control none (20th launch of a 4-buffer rotation), the others with ncu's default "
                        "cache flush before the replayed launch")
    open(os.path.join(dst, "ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    json.dump(util, open(upath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
