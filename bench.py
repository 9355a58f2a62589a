#!/usr/bin/env python
"""bench.py -- the Solve step of GPURepair (arXiv 2011.08373) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5]
                    [--impl ours|reference] [--no-cpu-baseline]

A *step* is one pass of the whole hot path over
one batch: device clause packing, exact PMS (a), exact MHS (b) and greedy mhs
(c) of every instance.  The default workload is BASELINE.json configs[1]
("c2": 748 suite-shaped instances, m <= 32, <= 64 clauses).  Under torchrun
every rank solves its own seeded 748-instance batch (weak scaling, no
data-path collective); the timed region is bracketed by a barrier and a
synchronize, and the time is the max over ranks.

One JSON line on rank 0.  value = candidate assignments decided per second
(exact PMS + MHS) over all ranks; instances_per_s alongside.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate assignments checked/sec and instances solved/sec at 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-kernels", action="store_true",
                    help="record per-kernel CUDA-event durations inside the library")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for i, n in enumerate(names):
                    if r[5 + i].lower().startswith("active"):
                        reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- workloads
def make_workload(cfg: str, rank: int):
    from paper_2011_08373_b200 import synth

    if cfg == "c1":
        return synth.c1_instances(), "C1: paper example in m=8 (2 instances)"
    if cfg == "c2":
        return (synth.c2_batch(seed=synth.seed_for(2, rank)),
                "C2: 748 suite-shaped instances, m<=32, <=64 clauses (PAPER.md:194, 593-602)")
    if cfg == "c3":
        cb, _, _ = synth.c3_instance()
        return cb, "C3: m=48, 200 clauses, k*=16, exhaustive levels"
    if cfg == "c4":
        return (synth.c4_batch(seed=synth.seed_for(4, rank)),
                "C4: 10000 WPMS instances, m=40, w~U{50..100}, planted SAT")
    raise ValueError(cfg)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)
    import torch
    import torch.distributed as dist

    import paper_2011_08373_b200 as gr

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    if a.config == "c5":
        return run_c5(a, rank, world, dev)
    cb, desc = make_workload(a.config, rank)
    flags = gr.GR_FLAG_EXHAUSTIVE if a.config == "c3" else 0
    db = gr.DeviceBatch.from_host(cb, device=dev, flags=flags)
    outs = [gr.DeviceResult.empty(cb.B, cb.W, dev) for _ in range(3)]
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        gr.solve_pms(db, outs[0])
        gr.mhs_exact(db, outs[1])
        gr.mhs_greedy(db, outs[2])

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gr_prof = gr.profiler() if a.profile_kernels else None
    total_ms = 0.0
    with ClockSampler(local) as clk:
        if gr_prof:
            gr_prof.start()
        for _ in range(a.steps):
            flush.fill_(1)  # L2 flush between timed iterations (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
        if gr_prof:
            kern = gr_prof.stop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    res = [o.to_host() for o in outs]
    cands = int(res[0]["decided"].astype(np.float64).sum() + res[1]["decided"].astype(np.float64).sum())
    t = torch.tensor([total_ms, float(cands), float(cb.B)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms, cands_all, inst_all = float(tmax[0]), float(tsum[1]), float(tsum[2])
    else:
        cands_all, inst_all = float(cands), float(cb.B)
    sec = total_ms / 1e3
    value = cands_all * a.steps / sec
    line = {
        "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded, SURVEY.md §8(d) recipe; DESIGN.md §6)",
        "config": {"workload": desc, "instances_per_gpu": cb.B, "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"batch-sharded x{world}" if world > 1 else "single GPU"},
        "instances_per_s": inst_all * a.steps / sec,
        "candidates_per_step": cands_all,
        "status_counts": {int(k): int(v) for k, v in zip(*np.unique(res[0]["status"], return_counts=True))},
        "clocks": clk.summary(),
        "gpu_launches": None,
    }
    if gr_prof:
        line["kernels"] = kern
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_c5(a, rank, world, dev):
    raise SystemExit("c5 bench: not yet wired")


def run_reference(a, rank, world):
    """The oracle (the CPU reference of this tier) on a bounded sample."""
    if rank != 0:
        return
    import oracle
    from paper_2011_08373_b200 import synth

    cb, desc = make_workload(a.config, 0)
    idx = [b for b in range(cb.B) if cb.m[b] <= 24]
    sub = cb.subset(idx)
    ts, cands = [], 0
    for s in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        p = oracle.batch("pms", sub)
        h = oracle.batch("mhs", sub)
        g = oracle.batch("greedy", sub)
        dt = time.perf_counter() - t0
        if s >= a.warmup:
            ts.append(dt)
            cands = float(p.decided.astype(np.float64).sum() + h.decided.astype(np.float64).sum())
    sec = float(np.sum(ts))
    v = cands * a.steps / sec
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "candidates/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": desc},
        "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": oracle.num_threads(),
                         "kind": "oracle", "sample": f"{len(idx)} of {cb.B} instances (m <= 24)"},
        "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
