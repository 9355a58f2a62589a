"""Turn a gpurun_out/prof/ evidence run (scripts/box_profiles.sh) into the
committed summaries under profiles/ (dev aid).

  profiles/<R>_bench_<cfg>.json         bench lines
  profiles/<R>_launches_c2_summary.csv  per-kernel totals of the ncu launch list
  profiles/<R>_ncu_enum_details.txt     ncu --page details of the enum capture
  profiles/<R>_ncu_selected_metrics.json  (enum_kernel entry replaced)
  profiles/traffic.json                 (enum_kernel entry replaced)
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = os.path.join("gpurun_out", "prof")
DST = "profiles"
NCU = "/usr/local/cuda/bin/ncu"

for cfg in ("c2", "c3", "c4", "c5", "reference", "reference_c5"):
    p = os.path.join(SRC, f"{R}_bench_{cfg}.json")
    if os.path.exists(p) and os.path.getsize(p) > 0:
        line = open(p).read().strip().splitlines()[-1]
        json.loads(line)
        with open(os.path.join(DST, f"{R}_bench_{cfg}.json"), "w") as f:
            f.write(line + "\n")

# launch list -> per-kernel summary
p = os.path.join(SRC, f"{R}_launches_c2.csv")
if os.path.exists(p):
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] == "ns" else (v * 1000.0 if r[ui] == "ms" else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    with open(os.path.join(DST, f"{R}_launches_c2_summary.csv"), "w") as f:
        f.write("# ncu launch list of `python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e` (C2)\n")
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): compare SHARES\n")
        f.write("# enum_kernel<1> is the untimed work-counting instantiation bench.py runs after the timed region\n")
        f.write("kernel,launches,total_us,share\n")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{n},{us:.1f},{us / tot:.4f}\n")

# full capture of enum_kernel
rep = os.path.join(SRC, f"{R}_enum_c2.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    out = []
    for r in csv.reader(det.splitlines()):
        if len(r) >= 15 and r[0] != "ID":
            out.append(f"{r[0]} | {r[-5]} | {r[-4]} | {r[-2]} {r[-3]}".rstrip())
    with open(os.path.join(DST, f"{R}_ncu_enum_details.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none -k regex:enum_kernel --launch-skip 15 -c 1 "
                "python scripts/prof_c2.py  (C2 PMS solve, level k = 16)\n")
        f.write("\n".join(out) + "\n")
    raw = list(csv.reader(subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    h, u, v = raw[0], raw[1], raw[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
            "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "sm__cycles_elapsed.avg.per_second", "launch__grid_size"]
    m = {w: [v[h.index(w)], u[h.index(w)]] for w in want if w in h}
    sel_p = os.path.join(DST, f"{R}_ncu_selected_metrics.json")
    sel = json.load(open(sel_p)) if os.path.exists(sel_p) else {}
    sel["enum_kernel"] = [m]
    sel["_enum_kernel_source"] = ("ncu --set full --clock-control none, scripts/prof_c2.py "
                                  "(C2 PMS solve), enum_kernel launch 16 (level k = 16)")
    json.dump(sel, open(sel_p, "w"), indent=1)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = sum(float(m[k][0]) * scale.get(m[k][1], 1) for k in
                  ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
    tp = os.path.join(DST, "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t["enum_kernel"] = int(traffic)
    json.dump(t, open(tp, "w"), indent=1)
    print("enum_kernel traffic", traffic, "bytes")
print("done")
