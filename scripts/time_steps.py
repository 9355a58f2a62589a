"""Device timings of the exact-solver steps the bench runs (development aid,
not the bench): C2 (PMS + MHS fused, + greedy), C3 (exhaustive, fused),
C4 (WPMS + MHS, + greedy).  CUDA events, L2 flushed, median of N.

    python scripts/time_steps.py [c2 c3 c4] [--reps N]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

reps = 7
args = [a for a in sys.argv[1:]]
if "--reps" in args:
    i = args.index("--reps")
    reps = int(args[i + 1])
    del args[i:i + 2]
which = args or ["c2", "c3", "c4"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))


for cfg in which:
    if cfg == "c2":
        cb, flags = synth.c2_batch(), 0
    elif cfg == "c3":
        cb, flags = synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE
    elif cfg == "c3p":
        cb, flags = synth.c3_instance()[0], 0
    elif cfg == "c4":
        cb, flags = synth.c4_batch(), 0
    else:
        continue
    db = gr.DeviceBatch.from_host(cb, flags=flags)
    outs = [gr.DeviceResult.empty(cb.B, cb.W, "cuda") for _ in range(3)]
    med, mn = timed(lambda: gr.solve_pms_mhs(db, outs[0], outs[1]))
    h = gr.to_host_many(outs[:2])
    d = float(h[0]["decided"].astype(np.float64).sum() + h[1]["decided"].astype(np.float64).sum())
    gm, _ = timed(lambda: gr.mhs_greedy(db, outs[2]))
    side = torch.cuda.Stream()

    def both_serial():
        gr.solve_pms_mhs(db, outs[0], outs[1])
        gr.mhs_greedy(db, outs[2])

    def both_overlap():  # the greedy on a side stream, launched first
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        gr.mhs_greedy(db, outs[2], stream=side)
        gr.solve_pms_mhs(db, outs[0], outs[1])
        cur.wait_stream(side)

    sm, _ = timed(both_serial)
    om, _ = timed(both_overlap)
    print(f"{cfg}: pms+mhs median {med:.3f} ms (min {mn:.3f})  greedy {gm:.3f} ms  "
          f"decided {d:.4e}  sat {int((h[0]['status'] == 0).sum())}/{cb.B}  "
          f"step serial {sm:.3f} overlapped {om:.3f} ms", flush=True)
