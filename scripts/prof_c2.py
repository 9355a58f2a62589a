"""One C2 bench step's exact solve (gr_solve_pms_mhs: PMS + MHS in one fused
walk, the device level loop queue_kernel) -- a short command for ncu --set
full (-k regex:queue_kernel).  `c3` / `c4` as the first argument profile those
configs' steps instead."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c3":
    cb, flags = synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE
elif cfg == "c4":
    cb, flags = synth.c4_batch(), 0
else:
    cb, flags = synth.c2_batch(), 0
db = gr.DeviceBatch.from_host(cb, flags=flags)
p, h = gr.solve_pms_mhs(db)
r = p.to_host()
torch.cuda.synchronize()
print("ok", cfg, int((r["status"] == 0).sum()), "SAT of", cb.B)
