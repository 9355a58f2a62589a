"""A small run of every kernel (for compute-sanitizer)."""
import random, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
rng = random.Random(1)
insts, ws = [], []
for _ in range(60):
    m = rng.randint(0, 40)
    pos = [sorted(rng.sample(range(1, m + 1), rng.randint(1, min(m, 4)))) for _ in range(rng.randint(0, 12))] if m else []
    neg = [sorted(rng.sample(range(1, m + 1), rng.randint(1, min(m, 3)))) for _ in range(rng.randint(0, 4))] if m else []
    insts.append((m, [list(c) for c in {tuple(c) for c in pos}], [list(c) for c in {tuple(c) for c in neg}]))
    ws.append([rng.randint(5, 7) for _ in range(40)])
cb = synth.batch_from_lists(insts, weights=ws, W=1)
db = gr.DeviceBatch.from_host(cb, flags=gr.GR_FLAG_WEIGHTED_GREEDY)
for f in (gr.solve_pms, gr.mhs_exact, gr.mhs_greedy):
    f(db)
gr.solve(db, gr.GR_STRATEGY_MHS)
gr.solve_pms_mhs(db)
csr, H = synth.c5_clauses(m=300, n=5000, n_planted=20)
for keep in (True, False):
    bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var, keep_csr=keep)
    gr.mhs_greedy_matrix(bm)
torch.cuda.synchronize()
print("ok")
