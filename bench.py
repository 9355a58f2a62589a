#!/usr/bin/env python
"""bench.py -- the Solve step of GPURepair (arXiv 2011.08373) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config all|c1|c2|c3|c4|c5]
                    [--impl ours|reference] [--no-cpu-baseline] [--no-e2e]

A *step* is one pass of the whole hot path over
one batch of synthetic input: device clause packing, exact PMS (a), exact MHS
(b) and greedy mhs (c) of every instance.  The headline workload is
BASELINE.json configs[1] ("c2": 748 suite-shaped instances, m <= 32, <= 64
clauses), the configuration the metric is quoted on (DESIGN.md §5 says why
C2 and not the larger C4).  With the default ``--config all`` the same JSON
line also carries one sub-record per other config (``configs``: C1, C3, C4,
C5), each with its own timing, clocks, e2e, roofline and cpu_baseline.

Timed region: device-resident inputs -> device results, CUDA events on the
launching stream, L2 flushed (256 MiB write) between steps, barrier +
synchronize on both sides, max over ranks.  `e2e` repeats the step through
the public API from pinned host buffers with the H2D / D2H copies inside.

Multi-GPU (torchrun, one rank per GPU): C2/C4 -- every rank solves its own
seeded batch (independent problems: no data-path collective, weak scaling);
at N > 1 a `strong` sub-record also splits ONE batch by cost over the ranks
with one NCCL all-gather of the results.  C3 -- each level's colex rank range
split over the ranks, one NCCL all-reduce MIN per level (strong scaling, on
the exhaustive no-refutation workload).  C5 -- clause columns split, one
all-reduce SUM of the counts per pick (strong).  C1 -- replicas.

value = candidate assignments decided per second over all ranks (exact PMS +
MHS; DESIGN.md §5 defines the count); instances_per_s alongside.
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

# ---- the exact solvers' roofline ----------------------------
# bound "alu": INT32 ALU-pipe lane-ops.  Peak = the LOP3/IADD3 micro-benchmark
# (scripts/int_peak.cu) measured on a B200 of this pool: 64 lanes/clk/SM
# (profiles/r02_int_peak.json); B300_MICROARCH.md "IADD3/LOP3 ... on alu-pipe,
# rt_SMSP = 2" gives the same 16 lanes/clk per SMSP.
INT_PEAK_FILE = os.path.join(ROOT, "profiles", "r02_int_peak.json")
ALU_LANES_PER_CLK_SM = 64
# Algorithmic INT ALU ops per unit of work the queue kernel performs (units
# counted by the kernel's counting instantiation, gr_profile(2)); the minimum
# ALU instructions of each step as written (DESIGN.md §5 derives each):
#   positive clause test  U & P == 0 ? (1) ; F &= H_j(P) on two words (2)
#   negative clause test  rest = N & ~U (1) ; rest outside the region ? (1) ;
#                         |rest| <= j ? (POPC + compare: 2)
#   refutation-scan clause  P & U (1), P & [0,e) (1), & used (1), used |= (1)
#   sub-block             window masks (3), base/pos advance (2), iterator
#                         step (sibling / child / pop: 3), witness ctz (1)
#   lane window           colex unrank: one compare + decrement per scanned
#                         row of the binomial table (about m_eff rows)
OPS_U32 = {"pos": 3, "neg": 4, "scan": 4, "blocks": 9, "windows": 64}
WIDE_EXTRA = 1  # one more op per clause test / scan clause on 64-bit masks


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="all", choices=["all", "c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        p.update(hbm_gbs=float(d.get("hbm_gbs", p["hbm_gbs"])),
                 sm_max_mhz=float(d.get("sm_max_mhz", p["sm_max_mhz"])),
                 source="MEASURED_PEAKS.json")
    return p


def int_peak(sms: int):
    """INT32 ALU lane-ops/s: the committed micro-benchmark measurement
    (LOP3.LUT, 1184 CTAs x 256 threads x 8 chains), else 64 lanes/clk/SM x
    148 x the max SM clock."""
    if os.path.exists(INT_PEAK_FILE):
        with open(INT_PEAK_FILE) as f:
            d = json.load(f)
        return (float(d["lop3"]["lane_ops_per_s"]),
                f"measured: scripts/int_peak.cu LOP3 on a B200 ({d['lop3']['lane_ops_per_clk_per_sm']} "
                f"lanes/clk/SM at {d['lop3']['sm_mhz_in_kernel']} MHz; {os.path.relpath(INT_PEAK_FILE, ROOT)})")
    pk = peaks()
    return (sms * ALU_LANES_PER_CLK_SM * pk["sm_max_mhz"] * 1e6,
            f"{sms} SMs x {ALU_LANES_PER_CLK_SM} lanes/clk x {pk['sm_max_mhz']:.0f} MHz")


def ncu_summary(name: str):
    """Selected counters of a committed ncu --set full capture (profiles/)."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f).get(name)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + clock-event (throttle) reasons DURING the timed region.

    The fields of the recipe's `nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,
    clocks_event_reasons.*` line, read through NVML (the library nvidia-smi
    queries) every 2 ms so that short timed regions still get samples; only
    the samples between start() and stop() count.  Falls back to nvidia-smi
    -lms 100 when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.nvml = index, [], None, None
        self.t0 = self.t1 = None
        self.stop_evt = threading.Event()
        self.max_mhz = None

    def _handle(self):
        import pynvml as nv
        import torch

        nv.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = "%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return nv, nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv, nv.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.nvml = (nv, h)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            t_end = time.perf_counter() + 2.0  # the poller is live before the timed region
            while not self.rows and time.perf_counter() < t_end:
                time.sleep(0.001)
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll(self):
        nv, h = self.nvml
        getr = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_evt.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                bits = int(getr(h))
            except Exception:
                break
            self.rows.append((time.perf_counter(), mhz, bits))
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) > 8:
                try:
                    mhz, mx = float(r[1]), float(r[2])
                except ValueError:
                    continue
                self.max_mhz = mx
                bits = sum(1 << i for i in range(4) if r[5 + i].lower().startswith("active"))
                self.rows.append((time.perf_counter(), mhz, -1 - bits))

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *a):
        self.stop_evt.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.nvml:
            self.t.join(timeout=1)

    def summary(self):
        t0 = self.t0 if self.t0 is not None else -1e30
        t1 = self.t1 if self.t1 is not None else 1e30
        rows = [r for r in list(self.rows) if t0 <= r[0] <= t1]
        reasons = set()
        for _, _, bits in rows:
            if bits >= 0 and self.nvml:
                nv = self.nvml[0]
                for name, const in self.REASONS:
                    if bits & int(getattr(nv, const, 0)):
                        reasons.add(name)
            elif bits < 0:
                b = -1 - bits
                for i, name in enumerate(("hw_slowdown", "hw_thermal_slowdown",
                                          "sw_thermal_slowdown", "sw_power_cap")):
                    if b >> i & 1:
                        reasons.add(name)
        sm = [r[1] for r in rows]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "samples_all": len(self.rows),
                "window_s": (t1 - t0) if self.t0 is not None and self.t1 is not None else None,
                "source": "NVML every 2 ms in the timed region" if self.nvml
                else "nvidia-smi -lms 100 in the timed region"}


# ---------------------------------------------------------------- workloads
DESC = {
    "c1": "C1: the paper's worked example (PAPER.md:26) in m=8, instances A+B; PMS + MHS + greedy",
    "c2": "C2: 748 suite-shaped instances, m<=32, <=64 clauses (PAPER.md:194, 593-602); PMS + MHS + greedy",
    "c3": "C3: one instance m=48, 200 mixed clauses, k*=16; PMS + MHS, levels 0..16 exhaustive",
    "c4": "C4: 10000 WPMS instances, m=40, w~U{50..100}, planted SAT; WPMS + MHS + greedy",
}


def make_workload(cfg: str, rank: int):
    from paper_2011_08373_b200 import synth

    if cfg == "c1":
        return synth.c1_instances()
    if cfg == "c2":
        return synth.c2_batch(seed=synth.seed_for(2, rank))
    if cfg == "c3":
        return synth.c3_instance()[0]
    if cfg == "c4":
        return synth.c4_batch(seed=synth.seed_for(4, rank))
    raise ValueError(cfg)


def host_tensors(cb, pinned: bool):
    import torch

    def t(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a).view(dt))
        return x.pin_memory() if pinned else x

    masks = cb.masks if cb.masks.shape[0] else np.zeros((1, cb.W), np.uint64)
    h = {"m": t(cb.m.astype(np.int32), np.int32), "off": t(cb.off.astype(np.int64), np.int64),
         "n_pos": t(cb.n_pos.astype(np.int32), np.int32),
         "masks": t(masks.astype(np.uint64).view(np.int64), np.int64)}
    if cb.w is not None:
        h["w"] = t(cb.w.astype(np.uint32).view(np.int32), np.int32)
    return h


def device_batch(h, cb, dev, flags):
    import paper_2011_08373_b200 as gr

    n = np.diff(cb.off)
    d = {k: v.to(dev, non_blocking=True) for k, v in h.items()}
    return gr.DeviceBatch(m=d["m"], off=d["off"], n_pos=d["n_pos"], masks=d["masks"],
                          w=d.get("w"), B=cb.B, W=cb.W, total_clauses=int(cb.off[-1]),
                          max_clauses=int(n.max()) if n.size else 0,
                          wstride=int(cb.w.shape[1]) if cb.w is not None else 0, flags=flags)


class Ctx:
    """rank / world / device / collectives of this process"""

    def __init__(self, rank, world, local, dev):
        self.rank, self.world, self.local, self.dev = rank, world, local, dev

    def max_(self, vals):
        """elementwise max over ranks (device time: max over ranks)"""
        import torch

        t = torch.tensor(vals, dtype=torch.float64, device=self.dev)
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def sum_(self, vals):
        import torch

        t = torch.tensor(vals, dtype=torch.float64, device=self.dev)
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.tolist()

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier()


def time_steps(step, steps, ctx, flush, clocks=True):
    """K timed steps (CUDA events on the current stream, L2 flushed between
    steps, synchronised, barrier before); returns (total ms, clocks)."""
    import torch

    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    ctx.barrier()
    total = 0.0
    with ClockSampler(ctx.local) as clk:
        clk.start()
        for _ in range(steps):
            flush.fill_(1)  # L2 flush between timed iterations (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            total += e0.elapsed_time(e1)
        clk.stop()
    torch.cuda.synchronize()
    return total, (clk.summary() if clocks else None)


def exact_roofline(cb, step, flush, step_ms, sms, cfg="c2"):
    """The dominant kernel (queue_kernel, the device level loop) of one
    untimed step: its event-timed duration (gr_profile(1)) and its work units
    (gr_profile(2), the counting instantiation) -> algorithmic INT ALU ops
    per second against the measured INT32 ALU peak."""
    import paper_2011_08373_b200 as gr
    import torch

    flush.fill_(1)
    torch.cuda.synchronize()
    prof = gr.profiler(1).start()
    step()
    kern = prof.stop()
    wprof = gr.profiler(2).start()
    step()
    wk = wprof.stop()
    torch.cuda.synchronize()
    q = kern.get("queue_kernel")
    w = wk.get("queue_kernel", {}).get("work")
    if not q or not w:
        return None, kern
    units = dict(zip(["pos", "neg", "scan", "blocks", "cands", "windows", "wide", "_"], w))
    ops = sum(OPS_U32[k] * units[k] for k in OPS_U32) + WIDE_EXTRA * units["wide"]
    sec = q["ms"] / 1e3
    peak, src = int_peak(sms)
    ach = ops / sec
    roof = {"bound": "alu", "achieved": ach / 1e12, "peak": peak / 1e12, "unit": "Tops/s",
            "frac": ach / peak, "traffic": None, "kernel": "queue_kernel",
            "per_launch": {"launches": q["launches"], "ms": q["ms"] / q["launches"],
                           "alu_ops": ops / q["launches"],
                           "units": {k: v / q["launches"] for k, v in units.items() if k != "_"}},
            "per_unit": ("INT ALU ops: positive clause test 3, negative 4, refutation-scan clause "
                         "4 (+1 on 64-bit masks), sub-block 9, lane window 64 (DESIGN.md §5)"),
            "peak_source": src,
            "share_of_step": q["ms"] / step_ms if step_ms else None,
            "timing": "one untimed step, CUDA events around the launch (gr_profile(1))",
            "traffic_note": "on-chip work: clause records in shared memory, ~0 HBM bytes"}
    hw = ncu_summary(f"queue_kernel_{cfg}")
    if hw:
        roof["ncu"] = hw
        roof["traffic"] = hw.get("dram_bytes_per_launch")
        roof["ncu_note"] = ("ncu --set full of this config's queue_kernel launch (scripts/prof_c2.py "
                            f"{cfg}; profiles/r02_ncu_summary.json): the hardware view -- issue slots, "
                            "pipes, stall cycles per issue (barrier = CTAs idle waiting for work)")
    return roof, kern


def kernels_of(k):
    return {n: {"launches": v["launches"], "ms_per_step": v["ms"]} for n, v in k.items()}


def run_exact(a, cfg, ctx, flush, sub=False):
    """C1-C4: pack + PMS + MHS (one launch for both) + greedy of the batch."""
    import torch

    import paper_2011_08373_b200 as gr
    from paper_2011_08373_b200 import multigpu

    rank, world, dev = ctx.rank, ctx.world, ctx.dev
    sharded = cfg == "c3" and world > 1
    cb = make_workload(cfg, rank)
    flags = gr.GR_FLAG_EXHAUSTIVE if cfg == "c3" else 0
    hb = host_tensors(cb, pinned=True)
    db = device_batch(hb, cb, dev, flags)
    torch.cuda.synchronize()
    outs = [gr.DeviceResult.empty(cb.B, cb.W, dev) for _ in range(3)]

    def step_local(dbx, o):  # PMS + MHS (one launch) and the greedy beside it on a side stream
        gr.solve_step(dbx, o[0], o[1], o[2])

    def step_sharded(dbx, o):  # C3 at N > 1: level rank ranges over the ranks, NCCL MIN per level
        multigpu.solve_pair_sharded(dbx, rank, world, out_pms=o[0], out_mhs=o[1])
        gr.mhs_greedy(dbx, o[2])

    step = step_sharded if sharded else step_local
    steps = a.steps
    for _ in range(a.warmup):
        step(db, outs)
    l0 = gr.launch_count()
    total_ms, clocks = time_steps(lambda: step(db, outs), steps, ctx, flush)
    launches = gr.launch_count() - l0
    res = gr.to_host_many(outs)
    cands = float(res[0]["decided"].astype(np.float64).sum() + res[1]["decided"].astype(np.float64).sum())
    cands_rank = cands / world if sharded else cands
    inst_rank = cb.B / world if sharded else cb.B
    tmax = ctx.max_([total_ms])[0]
    cands_all, inst_all = ctx.sum_([cands_rank, inst_rank])
    sec = tmax / 1e3
    rec = {"workload": DESC[cfg], "value": cands_all * steps / sec, "unit": "candidates/s",
           "ms_per_step": tmax / steps, "steps": steps, "warmup": a.warmup,
           "instances_per_s": inst_all * steps / sec, "candidates_per_step": cands_all,
           "instances_per_step": inst_all,
           "scaling": "strong" if sharded else "weak",
           "parallelism": (f"level rank ranges x{world} (NCCL allreduce MIN per level)" if sharded
                           else (f"one seeded batch per rank x{world}" if world > 1 else "single GPU")),
           "gpu_launches": launches, "clocks": clocks,
           "status_counts": {str(int(k)): int(v) for k, v in
                             zip(*np.unique(res[0]["status"], return_counts=True))}}
    # ---- roofline of the dominant kernel + per-kernel breakdown (untimed)
    if not sharded:
        roof, kern = exact_roofline(cb, lambda: step(db, outs), flush, tmax / steps,
                                    torch.cuda.get_device_properties(dev).multi_processor_count, cfg)
        rec["roofline"] = roof
        rec["kernels"] = kernels_of(kern)
        rec["kernels_note"] = "one extra untimed step with CUDA events around every launch"
    # ---- C3: the deterministic no-refutation workload for scaling
    if cfg == "c3":
        dbn = device_batch(hb, cb, dev, flags | gr.GR_FLAG_NO_PRUNE)
        nsteps = 3
        stepn = (lambda: step(dbn, outs))
        stepn()
        ms_n, clk_n = time_steps(stepn, nsteps, ctx, flush)
        ms_n = ctx.max_([ms_n])[0]
        rn = gr.to_host_many(outs[:2])
        cn = float(rn[0]["decided"].astype(np.float64).sum() + rn[1]["decided"].astype(np.float64).sum())
        rec["exhaustive_no_refutation"] = {
            "ms_per_step": ms_n / nsteps, "steps": nsteps, "value": cn * nsteps / (ms_n / 1e3),
            "unit": "candidates/s", "clocks": clk_n,
            "note": ("the scaling workload (SURVEY §8(d) C3): levels 0..16 decided sub-block by "
                     "sub-block (GR_FLAG_NO_PRUNE, deterministic work), same results; the headline "
                     "C3 figure above is the pruned walk (latency)")}
        del dbn
    # ---- C2 / C4 at N > 1: one batch split over the ranks (strong scaling)
    if cfg in ("c2", "c4") and world > 1:
        rec["strong"] = strong_batch(a, cfg, ctx, flush)
    # ---- e2e through the public API from pinned host buffers
    if not a.no_e2e:
        h2d = sum(int(v.numel() * v.element_size()) for v in hb.values())
        e2e_ms, host = 0.0, None
        stream = torch.cuda.current_stream()
        for s in range(a.warmup + steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dbx = device_batch(hb, cb, dev, flags)
            step(dbx, outs)
            host = gr.to_host_many(outs)
            e1.record(stream)
            e1.synchronize()
            if s >= a.warmup:
                e2e_ms += e0.elapsed_time(e1)
        d2h = sum(int(x.nbytes) for r in host for x in r.values())
        e2e_ms = ctx.max_([e2e_ms])[0]
        rec["e2e"] = {"value": cands_all * steps / (e2e_ms / 1e3), "unit": "candidates/s",
                      "instances_per_s": inst_all * steps / (e2e_ms / 1e3),
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "ms_per_step": e2e_ms / steps}
    # ---- the oracle on the host, and the GPU on the same sample
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline(cfg, cb, ctx, flush)
    return rec


def strong_batch(a, cfg, ctx, flush):
    """One shared batch dealt over the ranks by measured per-instance work
    (multigpu.shard_instances on the decided counts of a first solve), each
    rank solving its slice, one NCCL all-gather of the results -- the whole
    job's wall time on the device, max over ranks."""
    import torch

    import paper_2011_08373_b200 as gr
    from paper_2011_08373_b200 import multigpu

    cb = make_workload(cfg, 0)
    costs = multigpu.measured_costs(cb, ctx.dev)
    parts = multigpu.shard_instances(costs, ctx.world)
    mine = cb.subset(parts[ctx.rank]) if parts[ctx.rank] else None
    db = gr.DeviceBatch.from_host(mine, device=ctx.dev) if mine is not None else None
    outs = [gr.DeviceResult.empty(mine.B, mine.W, ctx.dev) for _ in range(3)] if mine else None
    gather = multigpu.nccl_allgather(device=ctx.dev)

    def step():
        return multigpu.solve_batch_sharded_device(cb, parts, ctx.rank, db, outs, gather)

    for _ in range(max(1, a.warmup)):
        got = step()
    ms, _ = time_steps(step, a.steps, ctx, flush, clocks=False)
    ms = ctx.max_([ms])[0]
    cands = float(got["decided_pms"].astype(np.float64).sum() + got["decided_mhs"].astype(np.float64).sum())
    return {"ms_per_step": ms / a.steps, "value": cands * a.steps / (ms / 1e3), "unit": "candidates/s",
            "instances_per_s": cb.B * a.steps / (ms / 1e3), "scaling": "strong",
            "parallelism": f"one batch dealt by measured cost over {ctx.world} ranks + NCCL all_gather"}


# ---------------------------------------------------------------- C5
C5_SAMPLE_N = 1 << 21


def run_c5(a, ctx, flush):
    import torch

    import paper_2011_08373_b200 as gr
    from paper_2011_08373_b200 import multigpu, synth

    rank, world, dev = ctx.rank, ctx.world, ctx.dev
    sharded = world > 1
    csr, H = synth.c5_clauses(seed=synth.seed_for(5, 0 if sharded else rank))
    po, pv = csr.pos_off, csr.pos_var
    if sharded:
        c0, c1 = multigpu.column_range(csr.n_pos, rank, world)
        po, pv = (po[c0:c1 + 1] - po[c0]).astype(np.int64), pv[po[c0]:po[c1]]
    d = {"po": torch.from_numpy(po).to(dev), "pv": torch.from_numpy(pv).to(dev),
         "no": torch.from_numpy(csr.neg_off).to(dev), "nv": torch.from_numpy(csr.neg_var).to(dev)}
    stream = torch.cuda.current_stream()

    def solve(bm):
        if sharded:
            assign, status, picks, npk = multigpu.greedy_matrix_sharded(bm, rank, world)
            return gr.GreedyMatrixResult(assign, status, picks, npk)
        return gr.mhs_greedy_matrix(bm)

    nnz = int(po[-1])

    def step(keep_csr, dd=None):
        dd = dd or d
        if keep_csr and not sharded:  # f3: from the clause lists alone, no bit matrix
            return None, gr.mhs_greedy_lists(csr.m, dd["po"], dd["pv"], dd["no"], dd["nv"],
                                             device=dev, nnz=nnz)
        bm = gr.pack_bitmatrix(csr.m, dd["po"], dd["pv"], dd["no"], dd["nv"], device=dev,
                               check=False, keep_csr=keep_csr)
        return bm, solve(bm)

    steps = max(1, min(a.steps, 5))  # a recounting step streams ~257 x 8.6 GB
    warm = max(1, min(a.warmup, 2))

    def timed(keep_csr, nsteps):
        for _ in range(warm):
            bm, r = step(keep_csr)
            del bm
        torch.cuda.synchronize()
        ctx.barrier()
        l0 = gr.launch_count()
        ms = 0.0
        with ClockSampler(ctx.local) as clk:
            clk.start()
            for _ in range(nsteps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                bm, r = step(keep_csr)
                e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
                ld = bm.ld if bm is not None else 0
                del bm
            clk.stop()
        launches = gr.launch_count() - l0
        prof = gr.profiler(1).start()  # per-kernel breakdown of one step, untimed
        bm, r1 = step(keep_csr)
        del bm
        kern = prof.stop()
        return ms, r, ld, kern, launches, clk.summary()

    # primary: the north-star design -- recounting passes streaming the 8 GiB
    # bit matrix (count_kernel, HBM roofline); then the f3 incremental greedy
    total_ms, r, ld, kern, launches, clocks = timed(False, steps)
    inc_ms, r2, _, kern2, _, clocks2 = timed(True, a.steps)
    total_ms, inc_ms = ctx.max_([total_ms, inc_ms])
    same = (r2.picks.cpu() == r.picks.cpu()).all().item() and r2.n_picks == r.n_picks
    pk = peaks()
    ck = kern["count_kernel"]
    bytes_per_launch = csr.m * ld * 8 + 3 * ld * 8  # R + U_in + U_out + R[v*] row (mark)
    eff = r.n_picks + 1  # passes that did work in the profiled step
    ach = bytes_per_launch / (ck["ms"] / eff / 1e3) / 1e9
    a_ = r.assign.cpu().numpy().view(np.uint64)
    size = int(sum(bin(int(x)).count("1") for x in a_))
    n = csr.n_pos if sharded else csr.n_pos * world  # whole-job clauses per step
    rec = {"workload": ("C5: greedy mhs, m=4096, n=2^24 positive clauses (8 GiB bit matrix); "
                        "step = device pack + greedy + prune + phi- check"),
           "value": n * steps / (total_ms / 1e3), "unit": "clauses/s (greedy)",
           "ms_per_step": total_ms / steps, "steps": steps, "warmup": warm,
           "scaling": "strong" if sharded else "weak",
           "parallelism": (f"clause columns x{world} (NCCL allreduce SUM of the counts per pick)"
                           if sharded else "single GPU"),
           "l2": "inputs (8 GiB) larger than L2",
           "greedy": {"picks": r.n_picks, "size": size, "status": int(r.status.item()), "planted": 256,
                      "passes": ck["launches"]},
           "f3_incremental": {"what": ("the same greedy from the clause lists alone (gr_mhs_greedy_lists: "
                                       "device-built variable -> clause lists, exact incremental counts, "
                                       "no bit matrix), identical picks" if not sharded else
                                       "incremental counts over the column-sharded matrix (CSR kept)"),
                              "ms_per_step": inc_ms / a.steps, "steps": a.steps,
                              "value": n * a.steps / (inc_ms / 1e3), "unit": "clauses/s (greedy)",
                              "speedup": (total_ms / steps) / (inc_ms / a.steps),
                              "identical_picks": bool(same), "clocks": clocks2,
                              "kernels": kernels_of(kern2)},
           "gpu_launches": launches, "clocks": clocks,
           "roofline": {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": ach / pk["hbm_gbs"], "traffic": None, "kernel": "count_kernel",
                        "share_of_step": ck["ms"] / (total_ms / steps),
                        "per_launch": {"bytes": bytes_per_launch, "ms": ck["ms"] / eff},
                        "peak_source": pk["source"] + " (copy, read+write)"},
           "kernels": kernels_of(kern)}
    hw = ncu_summary("count_kernel_c5")
    if hw:
        rec["roofline"]["ncu"] = hw
        rec["roofline"]["traffic"] = hw.get("dram_bytes_per_launch")
    if not a.no_e2e:  # pinned host CSR -> device, pack + greedy, result -> host, every step
        hp = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
              for k, v in (("po", po), ("pv", pv), ("no", csr.neg_off), ("nv", csr.neg_var))}
        h2d = sum(int(t.numel() * t.element_size()) for t in hp.values())
        ems, host = 0.0, None
        for s_ in range(warm + steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dd = {k: v.to(dev, non_blocking=True) for k, v in hp.items()}
            bm, rr = step(False, dd)
            host = [rr.assign.cpu(), rr.picks.cpu(), rr.status.cpu()]
            e1.record(stream)
            e1.synchronize()
            del bm, dd
            if s_ >= warm:
                ems += e0.elapsed_time(e1)
        d2h = sum(int(x.numel() * x.element_size()) for x in host)
        ems = ctx.max_([ems])[0]
        rec["e2e"] = {"value": n * steps / (ems / 1e3), "unit": "clauses/s (greedy)",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ems / steps}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline_c5(ctx, flush)
    return rec


def c5_oracle_once(csr):
    import oracle

    t0 = time.perf_counter()
    g = oracle.greedy_csr(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
    return time.perf_counter() - t0, g


def cpu_baseline_c5(ctx, flush):
    """The oracle's textbook greedy (recount per pick) on a C5-recipe instance
    with 1/8 of the clauses, repeated for >= 10 s; the GPU (recounting path,
    same pack + greedy) timed on the same instance."""
    import oracle
    import paper_2011_08373_b200 as gr
    from paper_2011_08373_b200 import synth

    csr, _ = synth.c5_clauses(seed=synth.seed_for(5, 0), n=C5_SAMPLE_N)
    sec, reps = 0.0, 0
    while sec < 10.0 and reps < 20:
        dt, _ = c5_oracle_once(csr)
        sec += dt
        reps += 1

    def gstep():
        bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var,
                               device=ctx.dev, check=False, keep_csr=False)
        gr.mhs_greedy_matrix(bm)

    gstep()
    gms, _ = time_steps(gstep, 3, ctx, flush, clocks=False)
    return {"value": C5_SAMPLE_N * reps / sec, "unit": "clauses/s (greedy)",
            "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{reps} greedy solve(s) of a C5-recipe instance with n = 2^21 clauses "
                      f"(1/8 of C5), m = 4096", "seconds": sec,
            "same_set_gpu": {"value": C5_SAMPLE_N * 3 / (gms / 1e3), "unit": "clauses/s (greedy)",
                             "ms_per_step": gms / 3,
                             "note": "the GPU step (host CSR already on the device) on that same instance"}}


# ---------------------------------------------------------------- CPU oracle legs
def c3_oracle_batch(n):
    """n C3-recipe instances scaled to m = 33 (11 groups of 3, k* = 11; clause
    counts scaled by 33/48), one seed each: the oracle (one thread per
    instance) finishes each in ~2.5 s where C3 itself would take hours."""
    from paper_2011_08373_b200 import synth

    insts = []
    for i in range(n):
        cb, _, _ = synth.c3_instance(seed=synth.seed_for(3) + 1000 + i, m=33, groups=11,
                                     n_rand_pos=124 * 33 // 48, n_neg=60 * 33 // 48)
        m, npos, mk, _ = cb.instance(0)
        cl = [synth.mask_to_vars(mk[j]) for j in range(mk.shape[0])]
        insts.append((m, cl[:npos], cl[npos:]))
    return synth.batch_from_lists(insts, W=1)


def oracle_sample(cfg, cb):
    """Bounded sample of the workload for the CPU oracle (about 10-30 s)."""
    if cfg == "c3":
        import oracle

        n = oracle.num_threads()
        return (c3_oracle_batch(n),
                f"{n} C3-recipe instances at m = 33 (11 groups, k* = 11), PMS + MHS, first witness")
    if cfg == "c2":
        idx = [b for b in range(cb.B) if cb.m[b] <= 26]
        return cb.subset(idx), f"{len(idx)} of {cb.B} C2 instances (those with m <= 26), PMS+MHS+greedy"
    if cfg == "c4":
        idx = list(range(48))
        return cb.subset(idx), f"first 48 of {cb.B} C4 instances, WPMS+MHS+greedy"
    return cb, "whole workload, PMS+MHS+greedy"


def run_oracle_once(sub):
    import oracle

    t0 = time.perf_counter()
    p = oracle.batch("pms", sub)
    h = oracle.batch("mhs", sub)
    oracle.batch("greedy", sub)
    cands = float(p.decided.astype(np.float64).sum() + h.decided.astype(np.float64).sum())
    return time.perf_counter() - t0, cands


def cpu_baseline(cfg, cb, ctx, flush):
    """The oracle as it stands on this host's cores, on a bounded sample of
    the workload; and the GPU step timed on that same sample (like-for-like
    instances/s and candidates/s: the decided counts are the same by parity)."""
    import oracle
    import paper_2011_08373_b200 as gr

    sub, desc = oracle_sample(cfg, cb)
    sec, cands, reps = 0.0, 0.0, 0
    while sec < 10.0 and reps < 50 and (cfg != "c1" or reps < 100000):
        dt, c = run_oracle_once(sub)
        sec += dt
        cands += c
        reps += 1
        if cfg == "c1" and sec >= 2.0:
            break
    flags = gr.GR_FLAG_EXHAUSTIVE if cfg == "c3" else 0
    flags = 0 if cfg == "c3" else flags  # the oracle sample runs first-witness
    db = gr.DeviceBatch.from_host(sub, device=ctx.dev, flags=flags)
    outs = [gr.DeviceResult.empty(sub.B, sub.W, ctx.dev) for _ in range(3)]

    def gstep():
        gr.solve_step(db, outs[0], outs[1], outs[2])

    gstep()
    gms, _ = time_steps(gstep, 5, ctx, flush, clocks=False)
    g = gr.to_host_many(outs[:2])
    gc = float(g[0]["decided"].astype(np.float64).sum() + g[1]["decided"].astype(np.float64).sum())
    ov, oi = cands / sec, sub.B * reps / sec
    gv, gi = gc * 5 / (gms / 1e3), sub.B * 5 / (gms / 1e3)
    return {"value": ov, "unit": "candidates/s", "cores": oracle.num_threads(), "kind": "oracle",
            "instances_per_s": oi, "sample": f"{reps} pass(es) over {desc}", "seconds": sec,
            "same_set_gpu": {"value": gv, "unit": "candidates/s", "instances_per_s": gi,
                             "ms_per_step": gms / 5, "ratio_instances_per_s": gi / oi,
                             "note": "the GPU step on the oracle's sample (same instances, same "
                                     "decided counts by parity)"}}


# ---------------------------------------------------------------- main
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)
    import torch
    import torch.distributed as dist

    import paper_2011_08373_b200 as gr  # noqa: F401  (fails loudly without the CUDA library)

    # functional check of the multi-rank code on one GPU (never a measurement):
    # GR_BENCH_ONE_GPU=1 puts every rank on cuda:0 with the gloo backend --
    # the ranks' kernels never wait on each other, only host collectives do
    one_gpu = os.environ.get("GR_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = Ctx(rank, world, local, dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    head_cfg = "c2" if a.config == "all" else a.config
    head = run_c5(a, ctx, flush) if head_cfg == "c5" else run_exact(a, head_cfg, ctx, flush)
    line = {
        "metric": METRIC, "value": head["value"], "unit": head["unit"], "n_gpus": world,
        "steps": head["steps"], "warmup": head["warmup"], "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": head["scaling"], "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded, SURVEY.md §8(d) recipe; DESIGN.md §6)",
        "config": {"workload": head["workload"],
                   "l2": head.get("l2", "flushed between timed steps (256 MiB write)"),
                   "parallelism": head["parallelism"]},
    }
    for k, v in head.items():
        if k not in ("workload", "value", "unit", "steps", "warmup", "ms_per_step", "scaling",
                     "parallelism", "l2"):
            line[k] = v
    if a.config == "all":
        subs = {}
        for cfg in ("c1", "c3", "c4", "c5"):
            try:
                subs[cfg] = run_c5(a, ctx, flush) if cfg == "c5" else run_exact(a, cfg, ctx, flush, sub=True)
            except Exception as e:  # a failing sub-config must not hide the headline
                subs[cfg] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()
        line["configs"] = subs
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(a, rank, world):
    """--impl reference: the CPU oracle (this tier's reference) on the host,
    on the headline config (C2; --config c1..c5 for the others)."""
    if rank != 0:
        return
    import oracle

    cfg = "c2" if a.config == "all" else a.config
    if cfg == "c5":
        from paper_2011_08373_b200 import synth

        csr, _ = synth.c5_clauses(seed=synth.seed_for(5, 0), n=C5_SAMPLE_N)
        ts = []
        for s in range(a.warmup + a.steps):
            dt, _ = c5_oracle_once(csr)
            if s >= a.warmup:
                ts.append(dt)
        sec = float(np.sum(ts))
        v = C5_SAMPLE_N * a.steps / sec
        sdesc = "greedy over a C5-recipe instance with n = 2^21 clauses (1/8 of C5), m = 4096"
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "clauses/s (greedy)",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": "C5 sample: " + sdesc},
            "cpu_baseline": {"value": v, "unit": "clauses/s (greedy)", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": sdesc},
            "e2e": {"value": v, "unit": "clauses/s (greedy)", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    cb = make_workload(cfg, 0)
    sub, sdesc = oracle_sample(cfg, cb)
    ts, cands = [], 0.0
    for s in range(a.warmup + a.steps):
        dt, c = run_oracle_once(sub)
        if s >= a.warmup:
            ts.append(dt)
            cands += c
    sec = float(np.sum(ts))
    v = cands / sec
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "candidates/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": DESC[cfg]},
        "instances_per_s": sub.B * a.steps / sec,
        "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": oracle.num_threads(),
                         "kind": "oracle", "sample": sdesc},
        "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
