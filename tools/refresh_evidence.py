"""Copy a round's GPU evidence from gpurun_out/ into profiles/: bench lines, the launch-list summary
of the default bench command, ncu --set full summaries, and the DRAM bytes per launch of the dominant
kernels (profiles/traffic.json, read by bench.py for roofline.traffic).

    python tools/refresh_evidence.py r02
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
R = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

for f in sorted(os.listdir(G)):
    if f.startswith("bench_") and f.endswith(".json") and os.path.getsize(os.path.join(G, f)) > 0:
        shutil.copy(os.path.join(G, f), os.path.join(P, f"{R}_{f}"))

if os.path.exists(os.path.join(G, "launches_c4.csv")):
    shutil.copy(os.path.join(G, "launches_c4.csv"), os.path.join(P, f"{R}_launches_c4.csv"))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"),
                          os.path.join(G, "launches_c4.csv")], capture_output=True, text=True).stdout
    with open(os.path.join(P, f"{R}_launches_c4_summary.txt"), "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 2 --warmup 1 "
                 "--no-cpu-baseline   (default bench workload c4)\n")
        fh.write("cold-cache, serialised launches (warm-up + timed + profiled + e2e passes): compare SHARES of the "
                 "MVM step, not absolute times\n")
        fh.write(out)

TITLES = {
    "c4": "c4 (BASELINE.json configs[3], bench.py default): ncu --set full --clock-control none, "
          "tools/prof_run.py --config c4 --calls 2",
    "c3": "c3 (BASELINE.json configs[2]): 2-D strip kernels and DMMA DFT passes, ncu --set full --clock-control "
          "none, tools/prof_run.py --config c3 --calls 2",
    "c2": "c2 (BASELINE.json configs[1]): ncu --set full --clock-control none, tools/prof_run.py --config c2 "
          "--calls 3",
}
traffic = {}
for c, title in TITLES.items():
    rep = os.path.join(G, f"prof_{c}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, title],
                         capture_output=True, text=True).stdout
    with open(os.path.join(P, f"{R}_ncu_full_{c}_summary.txt"), "w") as fh:
        fh.write(out)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    per = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        kind = "spread" if "spread" in name else ("interp" if "interp" in name else None)
        if kind is None:
            continue
        b = float(r[h.index("dram__bytes_read.sum")]) * (1e6 if rows[1][h.index("dram__bytes_read.sum")] == "Mbyte" else 1)
        b += float(r[h.index("dram__bytes_write.sum")]) * (1e6 if rows[1][h.index("dram__bytes_write.sum")] == "Mbyte" else 1)
        per.setdefault(kind, []).append(b)
    traffic[c] = {k: sum(v) / len(v) for k, v in per.items()}
if traffic:
    old = json.load(open(os.path.join(P, "traffic.json")))
    old["bytes_per_launch"].update(traffic)
    old["round"] = R
    old["source"] = ("ncu --set full captures (dram__bytes_read.sum + dram__bytes_write.sum, mean per launch of the "
                     "captured launches): profiles/" + R + "_ncu_full_{c4,c3,c2}_summary.txt")
    json.dump(old, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print("ok", sorted(traffic))
