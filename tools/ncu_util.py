"""Pipe / issue / shared-memory utilisation of one kernel from an ncu --set full
report -> profiles/ncu_util.json (bench.py attaches it to the roofline object).
Usage: ncu_util.py <rep> <key>"""
import csv, json, os, subprocess, sys

NAMES = {
    "issue_slots_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "shared_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "duration_us": "gpu__time_duration.sum",
}
rep, key = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, r = rows[0], rows[2]
vals = {k: float(r[h.index(m)].replace(",", "")) for k, m in NAMES.items() if m in h}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_util.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[key] = vals
json.dump(d, open(path, "w"), indent=1)
print(key, vals)
