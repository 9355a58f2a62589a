"""One WPMS solve of the C4 batch -- a short command for ncu on enum_kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cb = synth.c4_batch()
db = gr.DeviceBatch.from_host(cb)
r = gr.solve_pms(db).to_host()
torch.cuda.synchronize()
print("ok", int((r["status"] == 0).sum()), "SAT of", cb.B)
