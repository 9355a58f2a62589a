"""Selected counters of ncu --set full captures -> profiles/<R>_ncu_summary.json
(the hardware view bench.py quotes beside each roofline).

    python scripts/ncu_summary.py <R> name=path.ncu-rep [name=path.ncu-rep ...]

Per capture (first profiled launch): duration, SM clock, issue-slot and pipe
utilisation, warp cycles per issued instruction, the main stall reasons per
issue, achieved occupancy, executed instructions, DRAM bytes.
"""
import csv
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
PICK = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "sm_mhz": ("sm__cycles_elapsed.avg.per_second", 1e-6),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "warp_cycles_per_issue": ("smsp__average_warp_latency_per_inst_issued.ratio", 1),
    "active_threads_per_warp_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
}
STALLS = ["barrier", "long_scoreboard", "wait", "short_scoreboard", "membar", "branch_resolving",
          "math_pipe_throttle", "no_instruction", "not_selected", "selected", "sleeping", "lg_throttle",
          "mio_throttle", "dispatch_stall"]


def summary(rep):
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    out = {"kernel": d.get("Kernel Name", "")[:120], "source": os.path.basename(rep)}
    for name, (k, scale) in PICK.items():
        v = num(k)
        if v is not None:
            if k == "gpu__time_duration.sum" and u.get(k) == "us":
                scale = 1.0
            if k == "gpu__time_duration.sum" and u.get(k) == "ms":
                scale = 1e3
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                         "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u.get(k), 1.0)
            if k == "sm__cycles_elapsed.avg.per_second":
                scale = {"Ghz": 1e3, "GHz": 1e3, "Mhz": 1.0, "MHz": 1.0}.get(u.get(k), 1e-6)
            out[name] = v * scale
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    st = {}
    for s in STALLS:
        v = num(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
        if v is not None and v >= 0.05:
            st[s] = round(v, 3)
    out["stalls_per_issue"] = st
    return out


def main():
    R = sys.argv[1]
    path = os.path.join("profiles", f"{R}_ncu_summary.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        res[name] = summary(rep)
        print(name, json.dumps(res[name])[:300])
    with open(path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
