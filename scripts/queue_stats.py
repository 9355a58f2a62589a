"""Queue counters of the last device level loop (dev aid): task records,
ring entries and tickets of each solve's workspace after gr_solve_pms_mhs.

    python scripts/queue_stats.py [c2|c3|c3p|c4]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr  # noqa: E402
from paper_2011_08373_b200 import _native as N, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
cb, flags = {"c2": (synth.c2_batch(), 0), "c3": (synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE),
             "c3p": (synth.c3_instance()[0], 0), "c4": (synth.c4_batch(), 0)}[cfg]
db = gr.DeviceBatch.from_host(cb, flags=flags)
gr.solve_pms_mhs(db)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.solve_pms_mhs(db)
e1.record()
e1.synchronize()
ws = N._ws_cache[(str(db.m.device), "pair")]
b = db.struct(True)
half = (N.lib().gr_workspace_bytes(__import__("ctypes").byref(b), 0) + 255) // 256 * 256
for h in (0, 1):
    ctrl = ws[h * half: h * half + 128].cpu().numpy().view(np.uint64)
    # Ctrl: next_chunk, total_chunks, (n_active,n_remaining), lane_cands, (fin_ticket,pad0),
    #       q_tickets, q_entries, q_budget, q_tasks, (q_remaining,pad2), q_work
    print(f"{cfg} ms={e0.elapsed_time(e1):.3f} half{h}: tickets={ctrl[5]} entries={ctrl[6]} "
          f"budget={int(ctrl[7].view(np.int64))} tasks={ctrl[8]} work_left={ctrl[10]}")

# task records of the PMS workspace (the fused walk's only queue): the level timeline
import ctypes
L = N.lib()
L.gr_debug_tasks_offset.restype = ctypes.c_size_t
L.gr_debug_tasks_offset.argtypes = [ctypes.c_void_p]
toff = L.gr_debug_tasks_offset(ctypes.byref(b))
ctl = ws[0:128].cpu().numpy().view(np.uint64)
cnt, nchild = int(ctl[8]), int(ctl[11])
r = ws[toff: toff + 128 * cnt].cpu().numpy().view(np.uint64).reshape(-1, 16)
print(f"  root tasks {cnt}, child tasks (donated remainders) {nchild}")
if cnt > 40:  # batches: the level chain of the instance that commits last (the critical path)
    bcol = (r[:, 6] & np.uint64(0xffffffff)).astype(np.int64)
    last = int(bcol[np.argmax(r[:, 10].astype(np.int64))])
    print(f"  critical instance b={last} (m={int(cb.m[last])}, clauses={int(cb.off[last + 1] - cb.off[last])})")
    r = r[bcol == last]
    r = r[np.argsort(r[:, 8].astype(np.int64))]
t0 = int(r[:, 8].min())
for row in r:
    k = int(row[6] >> np.uint64(32))
    f = lambda x: (int(x) - t0) / 1e3 if x else -1.0
    print(f"  k={k:2d} nch={int(row[2]):7d} L={int(row[3]):8d} make={f(row[8]):8.1f} exhaust={f(row[9]):8.1f} "
          f"commit={f(row[10]):8.1f} last={f(row[11]):8.1f} us  succ={int(row[7] & np.uint64(0xffffffff))} "
          f"depth={int((row[7] >> np.uint64(48)) & np.uint64(255))} cancelled={int(row[7] >> np.uint64(56))}")
