"""Per-level device time of the C2 exact PMS solve (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
cb = synth.c2_batch() if cfg == "c2" else synth.c4_batch()
db = gr.DeviceBatch.from_host(cb)
for rep in range(2):
    s = gr.ExactSession(db, gr.PMS)
    torch.cuda.synchronize()
    n = s.prepare()
    tot = 0.0
    k = 1
    rows = []
    while n > 0 and k <= 64:
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        s.level(k)
        e1.record()
        n2 = s.finish(k)
        e2.record()
        e2.synchronize()
        rows.append((k, e0.elapsed_time(e1), e1.elapsed_time(e2), n, n2))
        tot += e0.elapsed_time(e2)
        n = n2
        k += 1
    if rep:
        for r in rows:
            print("k=%2d level %.3f ms finish %.3f ms active %d -> %d" % r)
        print("total %.2f ms" % tot)
