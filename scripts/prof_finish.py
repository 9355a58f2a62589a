"""The C2 fused PMS + MHS solve (the bench's step minus greedy) -- a short
command for ncu --set full of finish_fused_kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cb = synth.c2_batch()
db = gr.DeviceBatch.from_host(cb)
for _ in range(2):
    rp, rm = gr.solve_pms_mhs(db)
torch.cuda.synchronize()
print("ok", int((rp.to_host()["status"] == 0).sum()), "SAT of", cb.B)
