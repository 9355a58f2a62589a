#!/usr/bin/env python
"""bench.py -- the Solve step of GPURepair (arXiv 2011.08373) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5]
                    [--impl ours|reference] [--no-cpu-baseline]

A *step* is one pass of the whole hot path over
one batch of synthetic input: device clause packing, exact PMS (a), exact MHS
(b) and greedy mhs (c) of every instance.  The default workload is
BASELINE.json configs[1] ("c2": 748 suite-shaped instances, m <= 32, <= 64
clauses), the configuration the metric is quoted on.  Under torchrun every
rank solves its own seeded 748-instance batch (weak scaling, no data-path
collective; "c3" instead splits each level's colex rank range across the
ranks with an NCCL all-reduce MIN per level -- strong scaling).

The timed region is device-resident inputs -> device results, CUDA events on
the launching stream, L2 flushed (256 MiB write) between steps, barrier +
synchronize on both sides, max over ranks.  `e2e` repeats the step through the
public API from pinned host buffers with the H2D / D2H copies inside.

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
INT_LANES_PER_SM_CLK = 128  # INT32 issue: 4 SMSPs x 32 lanes x 1 warp-instruction/clk
# SURVEY.md §8(d) per-unit figure: a candidate-at-a-time enumerator spends one
# clause test (W + 1 ops) plus an amortised successor (~4 ops) per candidate.
OPS_PER_CANDIDATE = {32: 6, 64: 7}   # m_eff <= 32 (one 32-bit word) / <= 64
TEST_OPS = {32: 3, 64: 4}   # SASS per clause test: LOP3.P (U & P) + 2 predicated LOP3 (F &= H)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
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


def ncu_evidence(kernel: str):
    """Selected counters of the committed ncu --set full capture (profiles/)."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_selected_metrics.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f).get(kernel)
    if not d:
        return None
    m = d[0]
    pick = {"alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "active_lanes_per_warp_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
            "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"}
    out = {k: float(m[v][0]) for k, v in pick.items() if v in m}
    out["source"] = "profiles/r01_ncu_selected_metrics.json"
    return out


def traffic_of(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed ncu --set full capture (profiles/traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get(kernel)


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
def make_workload(cfg: str, rank: int):
    from paper_2011_08373_b200 import synth

    if cfg == "c1":
        return synth.c1_instances(), "C1: the paper's example (PAPER.md:26) in m=8, instances A+B"
    if cfg == "c2":
        return (synth.c2_batch(seed=synth.seed_for(2, rank)),
                "C2: 748 suite-shaped instances, m<=32, <=64 clauses (PAPER.md:194, 593-602)")
    if cfg == "c3":
        cb, _, _ = synth.c3_instance()
        return cb, "C3: one instance m=48, 200 clauses, k*=16, levels 0..16 exhaustive"
    if cfg == "c4":
        return (synth.c4_batch(seed=synth.seed_for(4, rank)),
                "C4: 10000 WPMS instances, m=40, w~U{50..100}, planted SAT")
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
    from paper_2011_08373_b200 import multigpu

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
    if a.config == "c5":
        return run_c5(a, rank, world, local, dev)
    cb, desc = make_workload(a.config, rank)
    flags = gr.GR_FLAG_EXHAUSTIVE if a.config == "c3" else 0
    hb = host_tensors(cb, pinned=True)
    db = device_batch(hb, cb, dev, flags)
    torch.cuda.synchronize()
    outs = [gr.DeviceResult.empty(cb.B, cb.W, dev) for _ in range(3)]
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    sharded = a.config == "c3" and world > 1

    def step(dbx, o):
        if sharded:  # rank-range sharding of each level, NCCL all-reduce MIN per level
            multigpu.solve_exact_sharded(dbx, gr.PMS, rank, world, out=o[0])
            multigpu.solve_exact_sharded(dbx, gr.MHS, rank, world, out=o[1])
        else:  # PMS and MHS level loops interleaved on two streams
            gr.solve_pms_mhs(dbx, o[0], o[1])
        gr.mhs_greedy(dbx, o[2])

    for _ in range(a.warmup):
        step(db, outs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---------------- timed region (device-resident inputs) ----------------
    # (no per-launch events in here: the kernel breakdown comes from one
    # extra, untimed step below)
    l0 = gr.launch_count()
    total_ms = 0.0
    with ClockSampler(local) as clk:
        clk.start()
        for _ in range(a.steps):
            flush.fill_(1)  # L2 flush between timed iterations (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(db, outs)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
        clk.stop()
    launches = gr.launch_count() - l0
    torch.cuda.synchronize()
    # per-kernel breakdown of one step, untimed, under gr_profile(1)
    flush.fill_(1)
    prof = gr.profiler(1).start()
    step(db, outs)
    kern = prof.stop()
    torch.cuda.synchronize()
    res = [o.to_host() for o in outs]
    cands = float(res[0]["decided"].astype(np.float64).sum() + res[1]["decided"].astype(np.float64).sum())
    if sharded:
        cands_rank = cands / world  # every rank holds the full result
    else:
        cands_rank = cands
    # ---------------- roofline pass (untimed): the solves serialised so launch
    # durations are not shared between streams, then the counting instantiation
    def serial_step(dbx, o):
        if sharded:
            step(dbx, o)
        else:
            gr.solve_pms(dbx, o[0])
            gr.mhs_exact(dbx, o[1])
            gr.mhs_greedy(dbx, o[2])

    flush.fill_(1)
    rprof = gr.profiler(1).start()
    serial_step(db, outs)
    kern_serial = rprof.stop()
    wprof = gr.profiler(2).start()
    serial_step(db, outs)
    wk = wprof.stop()
    # ---------------- the same step without subtree refutation (untimed for
    # the headline): every sub-block decided by its own clause tests
    nop_ms = None
    if not sharded:
        dbn = device_batch(hb, cb, dev, flags | gr.GR_FLAG_NO_PRUNE)
        step(dbn, outs)
        torch.cuda.synchronize()
        nop_ms = 0.0
        for _ in range(a.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(dbn, outs)
            e1.record(stream)
            e1.synchronize()
            nop_ms += e0.elapsed_time(e1)
        del dbn
    # ---------------- e2e through the public API from pinned host buffers --
    e2e_ms, h2d, d2h = None, 0, 0
    if not a.no_e2e:
        h2d = sum(int(v.numel() * v.element_size()) for v in hb.values())
        for s in range(a.warmup + a.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dbx = device_batch(hb, cb, dev, flags)
            step(dbx, outs)
            host = gr.to_host_many(outs)
            e1.record(stream)
            e1.synchronize()
            if s >= a.warmup:
                e2e_ms = (e2e_ms or 0.0) + e0.elapsed_time(e1)
        d2h = sum(int(x.nbytes) for r in host for x in r.values())
    # ---------------- reduce over ranks ---------------------------------------
    t = torch.tensor([total_ms, cands_rank, float(cb.B if not sharded else cb.B / world),
                      e2e_ms or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        tmax, tsum = t.clone(), t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        total_ms, cands_all, inst_all, e2e_ms = float(tmax[0]), float(tsum[1]), float(tsum[2]), float(tmax[3])
    else:
        cands_all, inst_all = cands_rank, float(cb.B)
    sec = total_ms / 1e3
    value = cands_all * a.steps / sec
    # ---------------- roofline of the dominant kernel (enum_kernel) ---------
    pk = peaks()
    ek = kern_serial.get("enum_kernel", {"launches": 0, "ms": 0.0})
    ew = wk.get("enum_kernel", {"launches": 0, "work": [0, 0, 0, 0]})
    tests, blocks, wcands, tests64 = ew["work"]
    wide = int((cb.m > 32).sum()) > cb.B // 2
    roof = None
    if ek["launches"] and ew["launches"]:
        per_launch_s = ek["ms"] / ek["launches"] / 1e3
        # units: candidates decided per launch (the metric's unit), averaged
        # over the serialised pass's enum_kernel launches
        cands_launch = cands_rank / ek["launches"]
        opc = OPS_PER_CANDIDATE[64 if wide else 32]
        achieved = cands_launch * opc / per_launch_s / 1e12
        peak_tops = 148 * INT_LANES_PER_SM_CLK * pk["sm_max_mhz"] * 1e6 / 1e12
        test_ops = TEST_OPS[32] * (tests - tests64) + TEST_OPS[64] * tests64
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_tops, "unit": "Tops/s",
                "frac": achieved / peak_tops, "traffic": traffic_of("enum_kernel"),
                "kernel": "enum_kernel",
                "per_unit": f"{opc} INT ops per candidate decided (SURVEY.md §8(d): 1 clause test "
                            f"+ amortised successor of a candidate-at-a-time enumerator)",
                "frac_note": ("> 1 is expected: the kernel decides up to 128 candidates per clause "
                              "test (bit-parallel sub-blocks) and refutes whole subtrees with one "
                              "clause; the hardware view is ncu's ALU-pipe / issue utilisation "
                              "(below) and clause_test_frac"),
                "per_launch": {"candidates": cands_launch, "ms": per_launch_s * 1e3,
                               "clause_tests": tests / ew["launches"],
                               "candidates_in_tested_blocks": wcands / ew["launches"],
                               "candidate_blocks": blocks / ew["launches"]},
                "peak_source": f"INT32 issue: 148 SMs x {INT_LANES_PER_SM_CLK} lanes/clk x "
                               f"{pk['sm_max_mhz']:.0f} MHz ({pk['source']})",
                "clause_test_frac": test_ops / ew["launches"] / per_launch_s / 1e12 / peak_tops,
                "ncu": ncu_evidence("enum_kernel"),
                "launch_timing": "untimed serialised pass (PMS and MHS solved one after the other)",
                "share_of_step": (kern.get("enum_kernel", {"ms": 0.0})["ms"] / (total_ms / a.steps)
                                  if total_ms else None),
                "share_note": "enum_kernel event time of one extra untimed step / timed step time"}
    line = {
        "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded, SURVEY.md §8(d) recipe; DESIGN.md §6)",
        "config": {"workload": desc, "instances_per_gpu": cb.B,
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": (f"level rank-range sharded x{world} (NCCL allreduce MIN per level)"
                                   if sharded else (f"batch x{world} (one seeded batch per rank)"
                                                    if world > 1 else "single GPU"))},
        "instances_per_s": inst_all * a.steps / sec,
        "candidates_per_step": cands_all,
        "e2e": ({"value": cands_all * a.steps / (e2e_ms / 1e3), "unit": "candidates/s",
                 "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                 "ms_per_step": e2e_ms / a.steps} if e2e_ms else None),
        "gpu_launches": launches,
        "roofline": roof,
        "without_subtree_refutation": ({"ms_per_step": nop_ms / a.steps,
                                        "value": cands_all * a.steps / (nop_ms / 1e3),
                                        "unit": "candidates/s",
                                        "note": "GR_FLAG_NO_PRUNE: every sub-block decided by its "
                                                "own clause tests; same results"}
                                       if nop_ms else None),
        "clocks": clk.summary(),
        "status_counts": {str(int(k)): int(v) for k, v in zip(*np.unique(res[0]["status"], return_counts=True))},
        "kernels": {k: {"launches": v["launches"], "ms_per_step": v["ms"]} for k, v in kern.items()},
        "kernels_note": "one extra untimed step with CUDA events around every launch",
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a.config, cb)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- C5
def run_c5(a, rank, world, local, dev):
    import torch

    import paper_2011_08373_b200 as gr
    from paper_2011_08373_b200 import synth

    from paper_2011_08373_b200 import multigpu

    # N > 1: one C5 phi+ split by clause columns across the ranks (SURVEY.md
    # §8(e) C5): each rank packs and streams its own column range, one NCCL
    # all-reduce (SUM) of the 4096 counts per pick -- strong scaling
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

    def step(keep_csr, dd=None):
        dd = dd or d
        bm = gr.pack_bitmatrix(csr.m, dd["po"], dd["pv"], dd["no"], dd["nv"], device=dev,
                               check=False, keep_csr=keep_csr)
        return bm, solve(bm)

    def timed(keep_csr, steps):
        for _ in range(max(1, min(a.warmup, 2))):
            bm, r = step(keep_csr)
            del bm
        torch.cuda.synchronize()
        l0 = gr.launch_count()
        ms = 0.0
        with ClockSampler(local) as clk:
            clk.start()
            for _ in range(steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                bm, r = step(keep_csr)
                e1.record(stream)
                e1.synchronize()
                ms += e0.elapsed_time(e1)
                ld = bm.ld
                del bm
            clk.stop()
        launches = gr.launch_count() - l0
        # per-kernel breakdown of one step, untimed, under gr_profile(1)
        prof = gr.profiler(1).start()
        bm, r1 = step(keep_csr)
        del bm
        kern = prof.stop()
        return ms, r, ld, kern, launches, clk.summary()

    # primary: the north-star design -- recounting passes streaming the 8 GiB
    # bit matrix (count_kernel, HBM roofline); then the f3 incremental greedy
    total_ms, r, ld, kern, launches, clocks = timed(False, a.steps)
    inc_ms, r2, _, kern2, _, _ = timed(True, a.steps)
    if world > 1:  # device time, max over ranks
        import torch.distributed as dist

        t = torch.tensor([total_ms, inc_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, inc_ms = t.tolist()
    same = (r2.picks.cpu() == r.picks.cpu()).all().item() and r2.n_picks == r.n_picks
    pk = peaks()
    ck = kern["count_kernel"]
    bytes_per_launch = csr.m * ld * 8 + 3 * ld * 8  # R + U_in + U_out + R[v*] row (mark)
    # passes that did work: n_picks + 1 per solve (up to 7 more are queued
    # no-ops after `done`; their few microseconds stay in the total)
    eff = r.n_picks + 1  # of the one profiled step
    ach = bytes_per_launch / (ck["ms"] / eff / 1e3) / 1e9
    a_ = r.assign.cpu().numpy().view(np.uint64)
    size = int(sum(bin(int(x)).count("1") for x in a_))
    # whole-job clauses per step: the one split phi+ (sharded) or one per rank
    n = csr.n_pos if sharded else csr.n_pos * world
    # e2e through the public API: pinned host CSR -> device, pack + greedy,
    # result (assignment, picks, status) -> host, every step
    e2e = None
    if not a.no_e2e:
        hp = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
              for k, v in (("po", po), ("pv", pv), ("no", csr.neg_off), ("nv", csr.neg_var))}
        h2d = sum(int(t.numel() * t.element_size()) for t in hp.values())
        ems, d2h = 0.0, 0
        for s_ in range(max(1, min(a.warmup, 2)) + a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dd = {k: v.to(dev, non_blocking=True) for k, v in hp.items()}
            bm, rr = step(False, dd)
            host = [rr.assign.cpu(), rr.picks.cpu(), rr.status.cpu()]
            e1.record(stream)
            e1.synchronize()
            del bm, dd
            if s_ >= max(1, min(a.warmup, 2)):
                ems += e0.elapsed_time(e1)
        d2h = sum(int(x.numel() * x.element_size()) for x in host)
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n * a.steps / (ems / 1e3), "unit": "clauses/s (greedy)",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ems / a.steps}
    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        cpu = cpu_baseline_c5(rank)
    line = {
        "metric": METRIC, "value": n * a.steps / (total_ms / 1e3), "unit": "clauses/s (greedy)",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic", "config": {"workload": "C5: greedy mhs, m=4096, n=2^24 positive clauses (8 GiB bit matrix); step = device pack + greedy + prune",
                                        "l2": "inputs (8 GiB) larger than L2",
                                        "parallelism": (f"clause columns sharded x{world} (NCCL allreduce SUM of the counts per pick)"
                                                        if sharded else "single GPU")},
        "greedy": {"picks": r.n_picks, "size": size, "status": int(r.status.item()), "planted": 256,
                   "passes": ck["launches"]},
        "f3_incremental": {"ms_per_step": inc_ms / a.steps, "speedup": total_ms / inc_ms,
                           "identical_picks": bool(same),
                           "kernels": {k: {"launches": v["launches"], "ms_per_step": v["ms"]}
                                       for k, v in kern2.items()}},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": ach / pk["hbm_gbs"], "traffic": traffic_of("count_kernel_c5"),
                     "traffic_source": "profiles/traffic.json (ncu --set full, scripts/prof_c5.py --full)",
                     "kernel": "count_kernel", "share_of_step": ck["ms"] / (total_ms / a.steps),
                     "per_launch": {"bytes": bytes_per_launch, "ms": ck["ms"] / eff},
                     "ncu": ncu_evidence("count_kernel")},
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "kernels": {k: {"launches": v["launches"], "ms_per_step": v["ms"]} for k, v in kern.items()},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


C5_SAMPLE_N = 1 << 21


def c5_oracle_once(csr):
    import oracle

    t0 = time.perf_counter()
    g = oracle.greedy_csr(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
    return time.perf_counter() - t0, g


def cpu_baseline_c5(rank):
    """The oracle's textbook greedy (recount per pick) on a C5-recipe instance
    with 1/8 of the clauses, repeated for >= 10 s."""
    import oracle
    from paper_2011_08373_b200 import synth

    csr, _ = synth.c5_clauses(seed=synth.seed_for(5, rank), n=C5_SAMPLE_N)
    sec, reps = 0.0, 0
    while sec < 10.0 and reps < 20:
        dt, _ = c5_oracle_once(csr)
        sec += dt
        reps += 1
    return {"value": C5_SAMPLE_N * reps / sec, "unit": "clauses/s (greedy)",
            "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{reps} greedy solve(s) of a C5-recipe instance with n = 2^21 clauses "
                      f"(1/8 of C5), m = 4096", "seconds": sec}


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
        return cb.subset(idx), f"first 48 of {cb.B} C4 instances, WPMS"
    return cb, "whole workload"


def run_oracle_once(cfg, sub):
    import oracle

    t0 = time.perf_counter()
    p = oracle.batch("pms", sub)
    cands = float(p.decided.astype(np.float64).sum())
    if cfg != "c4":
        h = oracle.batch("mhs", sub)
        oracle.batch("greedy", sub)
        cands += float(h.decided.astype(np.float64).sum())
    return time.perf_counter() - t0, cands


def cpu_baseline(cfg, cb):
    import oracle

    sub, desc = oracle_sample(cfg, cb)
    sec, cands, reps = 0.0, 0.0, 0
    while sec < 10.0 and reps < 50:
        dt, c = run_oracle_once(cfg, sub)
        sec += dt
        cands += c
        reps += 1
    return {"value": cands / sec, "unit": "candidates/s", "cores": oracle.num_threads(),
            "kind": "oracle", "sample": f"{reps} pass(es) over {desc}", "seconds": sec}


def run_reference(a, rank, world):
    """--impl reference: the CPU oracle (this tier's reference) on the host."""
    if rank != 0:
        return
    import oracle

    if a.config == "c5":
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
    cfg = a.config if a.config in ("c1", "c2", "c3", "c4") else "c2"
    cb, desc = make_workload(cfg, 0)
    sub, sdesc = oracle_sample(cfg, cb)
    ts, cands = [], 0.0
    for s in range(a.warmup + a.steps):
        dt, c = run_oracle_once(cfg, sub)
        if s >= a.warmup:
            ts.append(dt)
            cands += c
    sec = float(np.sum(ts))
    v = cands / sec
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "candidates/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": desc},
        "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": oracle.num_threads(),
                         "kind": "oracle", "sample": sdesc},
        "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
