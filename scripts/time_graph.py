"""solve_step launched vs replayed from a CUDA graph (gr.StepGraph), and the
graph's results against the launched step's (dev aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=21):
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
    return float(np.median(ts))


for cfg in (sys.argv[1:] or ["c1", "c2", "c3", "c4"]):
    cb, flags = {"c1": (synth.c1_instances(), 0), "c2": (synth.c2_batch(), 0),
                 "c3": (synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE), "c4": (synth.c4_batch(), 0)}[cfg]
    db = gr.DeviceBatch.from_host(cb, flags=flags)
    ref = gr.to_host_many(list(gr.solve_step(db)))
    g = gr.StepGraph(db)
    got = gr.to_host_many(g.replay())
    same = all(np.array_equal(a[k], b[k]) for a, b in zip(got, ref) for k in ("status", "cost", "assign", "decided"))
    for _ in range(3):  # replays again: the ring is cleared each time
        got = gr.to_host_many(g.replay())
        same = same and all(np.array_equal(a[k], b[k]) for a, b in zip(got, ref) for k in ("status", "cost", "assign", "decided"))
    outs = [gr.DeviceResult.empty(cb.B, cb.W, "cuda") for _ in range(3)]
    tl = timed(lambda: gr.solve_step(db, *outs))
    tg = timed(g.replay)
    print(f"{cfg}: launched {tl:.4f} ms  graph {tg:.4f} ms  identical={same}", flush=True)
