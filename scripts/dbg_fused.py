import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2011_08373_b200 as gr
from test_parity import rand_batch, gpu_solve
cb = rand_batch(7, 300, 20, 24)
db = gr.DeviceBatch.from_host(cb, weighted=False)
p, h = gr.solve_pms_mhs(db); p, h = p.to_host(), h.to_host()
rp, rh = gpu_solve(cb, "pms"), gpu_solve(cb, "mhs")
bad = np.nonzero((h["status"] != rh["status"]) | (h["assign"][:,0] != rh["assign"][:,0]) | (h["decided"] != rh["decided"]))[0]
print("bad mhs", bad[:10], len(bad))
for b in bad[:5]:
    m, npos, mk, _ = cb.instance(int(b))
    print(b, "m", m, "npos", npos, "nneg", mk.shape[0]-npos, "fused", h["status"][b], h["assign"][b], h["decided"][b], "sep", rh["status"][b], rh["assign"][b], rh["decided"][b], "pms", rp["status"][b], rp["decided"][b])
    print("   pos", [bin(int(x)) for x in mk[:npos,0]][:8], "neg", [bin(int(x)) for x in mk[npos:,0]][:8])
