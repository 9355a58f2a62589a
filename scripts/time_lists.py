"""C5 through gr_mhs_greedy_lists: per-kernel times (dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

csr, H = synth.c5_clauses()
d = {k: torch.from_numpy(v).cuda() for k, v in (("po", csr.pos_off), ("pv", csr.pos_var),
                                                  ("no", csr.neg_off), ("nv", csr.neg_var))}
nnz = int(csr.pos_off[-1])
for _ in range(2):
    r = gr.mhs_greedy_lists(csr.m, d["po"], d["pv"], d["no"], d["nv"], nnz=nnz)
torch.cuda.synchronize()
pr = gr.profiler(1).start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = gr.mhs_greedy_lists(csr.m, d["po"], d["pv"], d["no"], d["nv"], nnz=nnz)
e1.record()
e1.synchronize()
k = pr.stop()
print(f"total {e0.elapsed_time(e1):.3f} ms picks {r.n_picks}", {n: round(v['ms'], 3) for n, v in k.items()})
