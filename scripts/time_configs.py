"""Quick device timings of each config (development aid; not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402


def timed(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, r


which = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
if "c2" in which:
    cb = synth.c2_batch()
    db = gr.DeviceBatch.from_host(cb)
    for name, fn in (("pms", gr.solve_pms), ("mhs", gr.mhs_exact), ("greedy", gr.mhs_greedy)):
        fn(db)
        ms, r = timed(lambda: fn(db), 3)
        h = r.to_host()
        d = h["decided"].astype(np.float64).sum()
        print(f"c2 {name}: {ms:.2f} ms  decided={d:.3e}  cand/s={d / ms * 1e3:.3e}", flush=True)
if "c3" in which:
    cb, H, grp = synth.c3_instance()
    for flags in (0, gr.GR_FLAG_EXHAUSTIVE):
        db = gr.DeviceBatch.from_host(cb, flags=flags)
        ms, r = timed(lambda: gr.solve_pms(db))
        h = r.to_host()
        d = float(h["decided"][0])
        print(f"c3 flags={flags}: {ms:.1f} ms decided={d:.3e} cand/s={d / ms * 1e3:.3e} assign={h['assign'][0,0]}", flush=True)
if "c4" in which:
    cb = synth.c4_batch()
    db = gr.DeviceBatch.from_host(cb)
    gr.solve_pms(db)
    ms, r = timed(lambda: gr.solve_pms(db))
    h = r.to_host()
    d = h["decided"].astype(np.float64).sum()
    print(f"c4 pms: {ms:.1f} ms decided={d:.3e} cand/s={d / ms * 1e3:.3e} inst/s={cb.B / ms * 1e3:.1f}", flush=True)
if "c5" in which:
    t = time.time()
    csr, H = synth.c5_clauses()
    print(f"c5 gen {time.time() - t:.1f}s nnz={csr.pos_var.size}", flush=True)
    ms, bm = timed(lambda: gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var))
    print(f"c5 pack {ms:.1f} ms bad={bm.bad}", flush=True)
    ms, r = timed(lambda: gr.mhs_greedy_matrix(bm))
    a = r.assign.cpu().numpy().view(np.uint64)
    size = sum(bin(int(x)).count("1") for x in a)
    passes = r.n_picks + 1
    gbytes = csr.m * bm.ld * 8 / 1e9
    print(f"c5 greedy: {ms:.1f} ms picks={r.n_picks} |S|={size} status={int(r.status.item())} "
          f"per-pass={ms / passes:.3f} ms  ~{gbytes * passes / ms * 1e3:.0f} GB/s", flush=True)
