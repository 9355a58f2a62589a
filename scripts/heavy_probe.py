"""One C2 instance alone (default: the heavy b = 62) with a fixed lane window
(GR_LANE_CANDIDATES set by the caller): step time and the work units of the
counting instantiation (dev aid: per-window overhead vs window length).

    GR_LANE_CANDIDATES=4096 python scripts/heavy_probe.py [b]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 62
cb = synth.c2_batch().subset([b])
db = gr.DeviceBatch.from_host(cb)
p, h = gr.solve_pms_mhs(db)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.solve_pms_mhs(db, p, h)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
r = gr.to_host_many([p, h])
pr = gr.profiler(2).start()
gr.solve_pms_mhs(db, p, h)
k = pr.stop()
w = k["queue_kernel"]["work"]
names = ["pos", "neg", "scan", "blocks", "cands", "windows", "wide", "-"]
print(f"L={os.environ.get('GR_LANE_CANDIDATES', 'adaptive')} ms={np.median(ts):.3f} status={int(r[0]['status'][0])} "
      f"cost={int(r[0]['cost'][0])} decided={float(r[0]['decided'][0]):.3e}/{float(r[1]['decided'][0]):.3e}",
      {n: f"{v:.3e}" for n, v in zip(names, w)}, flush=True)
