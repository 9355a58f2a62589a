"""Greedy over a C5 bit matrix -- a short command for ncu --set full on
count_kernel.  Default: reduced C5 (m = 4096, n = 2^22: 2 GiB, > L2);
--full: the C5 workload itself (n = 2^24, 8 GiB); --lists: the full C5
through gr_mhs_greedy_lists as well (no bit matrix)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

n = 1 << 24 if ("--full" in sys.argv or "--lists" in sys.argv) else 1 << 22
csr, H = synth.c5_clauses(n=n)
bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var, keep_csr=False)
r = gr.mhs_greedy_matrix(bm)
torch.cuda.synchronize()
print("ok n", n, "ld", bm.ld, "picks", r.n_picks, "status", int(r.status.item()))
if "--lists" in sys.argv:
    r2 = gr.mhs_greedy_lists(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
    torch.cuda.synchronize()
    print("lists picks", r2.n_picks, "status", int(r2.status.item()))
