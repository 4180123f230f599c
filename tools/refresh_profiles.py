"""Copy a profile_round.sh result (gpurun_out/prof) into profiles/<round>/: bench
lines, CUPTI kernel tables, launch-list summary, per-kernel ncu summaries, and
refresh profiles/ncu_traffic.json (dram bytes per launch) and ncu_util.json.
Usage: refresh_profiles.py [src=gpurun_out/prof] [round=r01]"""
import csv, glob, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof")
dst = os.path.join(ROOT, "profiles", sys.argv[2] if len(sys.argv) > 2 else "r01")
os.makedirs(dst, exist_ok=True)
names = {"bench_c3.json": "bench_c3_n1.json", "bench_c2.json": "bench_c2_n1.json",
         "bench_c4.json": "bench_c4_n1.json", "bench_c5_train.json": "bench_c5_train_n1.json",
         "bench_ref.json": "bench_ref_n1.json", "kprof_c3.txt": "kprof_c3.txt", "kprof_c5.txt": "kprof_c5_train.txt"}
for a, b in names.items():
    p = os.path.join(src, a)
    if os.path.exists(p):
        lines = [l for l in open(p).read().splitlines() if l.strip() and "Warn" not in l and "_warn_once" not in l]
        open(os.path.join(dst, b), "w").write("\n".join(lines[-1:] if a.endswith(".json") else lines) + "\n")
if os.path.exists(os.path.join(src, "launches.csv")):
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches_bench16.csv"))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                          os.path.join(src, "launches.csv"), "30"], capture_output=True, text=True).stdout
    open(os.path.join(dst, "launch_list_summary.txt"), "w").write(out)

traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for rep in sorted(glob.glob(os.path.join(src, "ncu_*.ncu-rep"))):
    tag = os.path.basename(rep)[4:-8]
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                          capture_output=True, text=True).stdout
    open(os.path.join(dst, f"ncu_{tag}.txt"), "w").write(summ)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
        tot = 0.0
        try:
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = h.index(m)
                tot += float(r[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                        "Gbyte": 1e9}.get(rows[1][i], 1)
        except (ValueError, IndexError):
            continue
        traffic[name] = int(tot)
    if tag == "raster_fwd_kernel":
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_util.py"), rep, "raster_fwd_kernel"])
json.dump(traffic, open(traffic_path, "w"), indent=1)
print("traffic", traffic)
