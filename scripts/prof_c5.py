"""Greedy over a reduced C5 bit matrix (m = 4096, n = 2^22: 2 GiB, > L2) -- a
short command for ncu --set full on count_kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

csr, H = synth.c5_clauses(n=1 << 22)
bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
r = gr.mhs_greedy_matrix(bm)
torch.cuda.synchronize()
print("ok picks", r.n_picks, "status", int(r.status.item()))
