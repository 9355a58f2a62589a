"""Turn an evidence run of scripts/box_evidence.sh (gpurun_out/<R>/) into the
committed summaries under profiles/ (dev aid).

  profiles/<R>_bench.json, <R>_bench_reference.json   the bench lines
  profiles/<R>_gpu_tests_tail.txt                     tail of pytest -m gpu
  profiles/<R>_launches_c2_summary.csv                per-kernel totals of the ncu launch list
  profiles/<R>_ncu_<name>_details.txt                 ncu --page details of each capture
  profiles/<R>_ncu_<name>_lines.txt                   per-source-line stall summary (scripts/ncu_lines.py)
  profiles/<R>_ncu_summary.json                       selected counters (scripts/ncu_summary.py)
  profiles/<R>_onegpu_n2/                             bench.py N = 2 on one GPU (functional)

    python scripts/summarize_profiles.py r02
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_lines  # noqa: E402
import ncu_summary  # noqa: E402

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
SRC = os.path.join("gpurun_out", R)
DST = "profiles"
NCU = ncu_summary.NCU


def last_json_line(p):
    for line in reversed(open(p).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            json.loads(line)
            return line
    raise ValueError(f"no JSON line in {p}")


for name in ("bench", "bench_reference"):
    p = os.path.join(SRC, f"{name}.json")
    if os.path.exists(p) and os.path.getsize(p) > 0:
        with open(os.path.join(DST, f"{R}_{name}.json"), "w") as f:
            f.write(last_json_line(p) + "\n")
        print("bench line", name)

p = os.path.join(SRC, "tests.log")
if os.path.exists(p):
    tail = open(p).read().strip().splitlines()[-6:]
    with open(os.path.join(DST, f"{R}_gpu_tests_tail.txt"), "w") as f:
        f.write("# python -m pytest tests -m gpu -q  (one B200)\n" + "\n".join(tail) + "\n")

# launch list -> per-kernel summary
p = os.path.join(SRC, "launches_c2.csv")
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
        f.write("# ncu launch list of `python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e`\n")
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): compare SHARES\n")
        f.write("# queue_kernel<1,...> launches are the untimed work-counting instantiation bench.py runs after the timed region\n")
        f.write("kernel,launches,total_us,share\n")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{n},{us:.1f},{us / tot:.4f}\n")
    print("launch list", len(rows) - 1, "launches")

CAPTURES = {  # capture file -> (summary key, what)
    "q_c2": ("queue_kernel_c2", "queue_kernel, C2 fused PMS + MHS walk (scripts/prof_c2.py c2)"),
    "q_c3": ("queue_kernel_c3", "queue_kernel, C3 fused exhaustive walk (scripts/prof_c2.py c3)"),
    "q_c4": ("queue_kernel_c4", "queue_kernel, C4 WPMS + MHS (scripts/prof_c2.py c4)"),
    "count_c5": ("count_kernel_c5", "count_kernel, C5 recount pass on the 8 GiB matrix (scripts/prof_c5.py --full)"),
    "lscatter_c5": ("lscatter_kernel_c5", "lscatter_kernel, C5 list build (scripts/time_lists.py)"),
    "lgreedy_c5": ("lgreedy_kernel_c5", "lgreedy_kernel, C5 pick loop (scripts/time_lists.py)"),
}
sp = os.path.join(DST, f"{R}_ncu_summary.json")
summ = json.load(open(sp)) if os.path.exists(sp) else {}
for cap, (key, what) in CAPTURES.items():
    rep = os.path.join(SRC, f"{cap}.ncu-rep")
    if not os.path.exists(rep):
        continue
    det = subprocess.run([NCU, "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(DST, f"{R}_ncu_{cap}_details.txt"), "w") as f:
        f.write(f"# ncu --set full --import-source on --clock-control none: {what}\n")
        f.write(det)
    src = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(SRC, f"{cap}_source.csv")
    open(tmp, "w").write(src)
    buf = io.StringIO()
    old = sys.stdout
    sys.stdout = buf
    try:
        ncu_lines.main(tmp, 40)
    finally:
        sys.stdout = old
    with open(os.path.join(DST, f"{R}_ncu_{cap}_lines.txt"), "w") as f:
        f.write(f"# per source line: % of warp-stall samples, % of instructions, top stalls -- {what}\n")
        f.write(buf.getvalue())
    s = ncu_summary.summary(rep)
    s["what"] = what
    summ[key] = s
    print("capture", cap, "->", key, round(s.get("duration_us", 0), 1), "us")
json.dump(summ, open(sp, "w"), indent=1)

src_dir = os.path.join(SRC, "onegpu")
if os.path.isdir(src_dir):
    dst_dir = os.path.join(DST, f"{R}_onegpu_n2")
    os.makedirs(dst_dir, exist_ok=True)
    for fn in os.listdir(src_dir):
        shutil.copy(os.path.join(src_dir, fn), os.path.join(dst_dir, fn))
    print("onegpu", sorted(os.listdir(dst_dir)))
print("done")
