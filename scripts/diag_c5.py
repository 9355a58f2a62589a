import sys, time
import torch
sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 24)
csr, H = synth.c5_clauses(n=n)
bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
r = gr.mhs_greedy_matrix(bm); torch.cuda.synchronize()
pr = gr.profiler(1).start()
t = time.time(); r = gr.mhs_greedy_matrix(bm); torch.cuda.synchronize(); dt = time.time() - t
k = pr.stop()
print(f"wall {dt*1e3:.1f} ms picks {r.n_picks}")
for name, v in sorted(k.items(), key=lambda x: -x[1]["ms"]):
    print(f"  {name:24s} launches {v['launches']:6d}  ms {v['ms']:9.3f}  avg_us {1e3*v['ms']/max(v['launches'],1):8.2f}")
