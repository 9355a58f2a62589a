"""Per-rank C2 batches (seed_for(2, rank)): solve time of each on one GPU
(weak-scaling balance check; dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

for r in range(8):
    cb = synth.c2_batch(seed=synth.seed_for(2, r))
    db = gr.DeviceBatch.from_host(cb)
    o = [gr.DeviceResult.empty(cb.B, cb.W) for _ in range(2)]
    gr.solve_pms_mhs(db, o[0], o[1])
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.solve_pms_mhs(db, o[0], o[1])
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    d = float(o[0].decided.double().sum() + o[1].decided.double().sum())
    print(r, "ms %.3f" % sorted(ts)[2], "cands %.3g" % d, flush=True)
