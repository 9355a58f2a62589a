"""Work units of the exact solvers' device level loop for one config
(gr_profile(2): the counting instantiation) -- development aid for the lane
window sizing and the roofline's per-unit model.

    python scripts/work_units.py [c2|c3|c4]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
cb, flags = {"c2": (synth.c2_batch(), 0), "c3": (synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE),
             "c4": (synth.c4_batch(), 0)}[cfg]
db = gr.DeviceBatch.from_host(cb, flags=flags)
gr.solve_pms_mhs(db)
torch.cuda.synchronize()
pr = gr.profiler(2).start()
gr.solve_pms_mhs(db)
k = pr.stop()
w = k["queue_kernel"]["work"]
names = ["pos_tests", "neg_tests", "scan_clauses", "sub_blocks", "cands_in_blocks", "windows", "wide_ops", "-"]
print(cfg, {n: f"{v:.3e}" for n, v in zip(names, w)})
