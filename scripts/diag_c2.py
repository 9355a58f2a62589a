"""C2 diagnostics: per-solver work counters and per-instance-class split."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

cb = synth.c2_batch()
db = gr.DeviceBatch.from_host(cb)
gr.solve_pms(db)
torch.cuda.synchronize()
for mode in (1, 2):
    pr = gr.profiler(mode).start()
    r = gr.solve_pms(db).to_host()
    k = pr.stop()
    e = k["enum_kernel"]
    print(f"mode {mode}: enum launches {e['launches']} ms {e['ms']:.2f} work {e['work']}")
    if mode == 2:
        t, b, c, t64 = e["work"]
        print(f"  tests/block {t / b:.2f}  cands/block {c / b:.2f}  tests/cand {t / c:.3f}")
st = r["status"]
dec = r["decided"].astype(np.float64)
for name, mask in (("SAT", st == 0), ("UNSAT", st == 1)):
    print(name, int(mask.sum()), f"decided {dec[mask].sum():.3e}")
big = np.argsort(-dec)[:10]
for b in big:
    m, npos, mk, _ = cb.instance(int(b))
    print(f"  inst {b}: m={m} npos={npos} nneg={mk.shape[0]-npos} status={st[b]} decided={dec[b]:.3e}")
# time the UNSAT-heavy subset alone
idx = [int(b) for b in np.nonzero(st == 1)[0]]
sub = gr.DeviceBatch.from_host(cb.subset(idx))
gr.solve_pms(sub)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); gr.solve_pms(sub); e1.record(); e1.synchronize()
print("UNSAT subset ms", e0.elapsed_time(e1))
idx = [int(b) for b in np.nonzero(st == 0)[0]]
sub = gr.DeviceBatch.from_host(cb.subset(idx))
gr.solve_pms(sub)
torch.cuda.synchronize()
e0.record(); gr.solve_pms(sub); e1.record(); e1.synchronize()
print("SAT subset ms", e0.elapsed_time(e1))
