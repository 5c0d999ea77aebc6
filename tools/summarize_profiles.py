"""Write the round's profile summaries under profiles/ from gpurun_out/ (ncu reports, launch list,
bench lines).  Usage: python tools/summarize_profiles.py r01"""
import csv
import collections
import json
import os
import shutil
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
G, P = "gpurun_out", "profiles"
os.makedirs(P, exist_ok=True)

# bench lines
for f in sorted(os.listdir(G)):
    if f.startswith("bench_") and f.endswith(".json"):
        shutil.copy(os.path.join(G, f), os.path.join(P, f"{R}_{f}"))

# launch list of the default bench command
rows = [r for r in csv.reader(open(os.path.join(G, "launches_c2.csv"))) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = collections.defaultdict(list)
order = []
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("void ", "")
    if k not in d:
        order.append(k)
    d[k].append(float(r[vi].replace(",", "")))
shutil.copy(os.path.join(G, "launches_c2.csv"), os.path.join(P, f"{R}_launches_c2.csv"))
with open(os.path.join(P, f"{R}_launches_c2_summary.txt"), "w") as out:
    out.write("ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 3 --warmup 3 "
              "--no-cpu-baseline   (default bench workload c2)\n")
    out.write("cold-cache, serialised launches: compare SHARES of the MVM step, not absolute times\n\n")
    out.write(f"{'kernel':45s} {'launches':>8s} {'mean us':>9s}\n")
    for k in order:
        v = d[k]
        out.write(f"{k:45s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f}\n")
    mvm = [k for k in order if any(s in k for s in ("k_spread", "k_dft", "k_plane", "k_pencil", "k_interp", "k_epilogue"))]
    tot = sum(sum(d[k]) / len(d[k]) for k in mvm)
    out.write("\nper-MVM-step share (mean launch time of each kernel, one launch each per step):\n")
    for k in mvm:
        m = sum(d[k]) / len(d[k])
        out.write(f"  {k:45s} {m / 1e3:8.2f} us  {100 * m / tot:5.1f}%\n")
    out.write(f"  total {tot / 1e3:.1f} us per step (serialised, cold)\n")

# ncu full captures
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__ops_path_tensor_src_fp64.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
CMD = {"c2": "ncu --set full --clock-control none --import-source on "
             "-k regex:'k_spread|k_plane|k_pencil|k_dft|k_interp|k_epilogue' -s 6 -c 6 "
             "python tools/prof_run.py --config c2 --calls 3",
       "c4": "ncu --set full --clock-control none --import-source on -k regex:'k_spread|k_interp' -s 2 -c 2 "
             "python tools/prof_run.py --config c4 --calls 2"}
traffic = {}
for cfg in ("c2", "c4"):
    rep = os.path.join(G, f"prof_{cfg}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(os.path.join(P, f"{R}_ncu_full_{cfg}_summary.txt"), "w") as out:
        out.write(CMD[cfg] + "\n")
        for r in rows[2:]:
            out.write("\n== " + r[hdr.index("Kernel Name")][:100] + "\n")
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    out.write(f"  {k:82s} {r[i]} {units[i]}\n")
            name = r[hdr.index("Kernel Name")]
            stage = "spread" if "k_spread" in name else "interp" if "k_interp" in name else None
            if stage:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                b = sum(float(r[hdr.index(k)].replace(",", "")) * scale.get(units[hdr.index(k)], 1)
                        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                traffic.setdefault(cfg, {})[stage] = b
    if cfg == "c4":
        shutil.copy(rep, os.path.join(P, f"{R}_prof_{cfg}.ncu-rep"))
json.dump({"round": R, "source": "ncu --set full captures (dram__bytes_read.sum + dram__bytes_write.sum per launch)",
           "bytes_per_launch": traffic}, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print("ok")
