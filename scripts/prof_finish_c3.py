"""One C3 PMS solve (a single instance): an ncu target for the finish
kernel's fixed per-level cost (dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cb, _, _ = synth.c3_instance()
db = gr.DeviceBatch.from_host(cb)
r = gr.solve_pms(db).to_host()
torch.cuda.synchronize()
print("ok", int(r["status"][0]), int(r["cost"][0]))
