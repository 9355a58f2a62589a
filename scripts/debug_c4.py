"""Parity of chosen C4 instances under different lane-window knobs (dev aid).

    python scripts/debug_c4.py <instance> [<instance> ...]
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
idx = [int(x) for x in sys.argv[1:]] or [2649]
code = """
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
idx = %r
e = np.load('tests/golden/expected_c4.npz')
cb = synth.c4_batch()
sub = cb.subset(idx) if len(idx) < 5 else cb
import os
db = gr.DeviceBatch.from_host(sub, flags=int(os.environ.get('DBG_FLAGS', '0')))
r = gr.solve_pms(db).to_host()
for j, b in enumerate(idx):
    jj = j if len(idx) < 5 else b
    ok = (r['assign'][jj] == e['pms_assign'][b]).all() and r['cost'][jj] == e['pms_cost'][b]
    print(b, 'ok' if ok else 'BAD', 'got', int(r['assign'][jj, 0]), int(r['cost'][jj]), int(r['decided'][jj]),
          'want', int(e['pms_assign'][b, 0]), int(e['pms_cost'][b]), int(e['pms_decided'][b]))
"""
envs = [{"GR_LANE_CANDIDATES": "65536"}, {"GR_LANE_CANDIDATES": "65536", "GR_HOST_LOOP": "1"},
        {"GR_LANE_CANDIDATES": "65536", "DBG_FLAGS": "4"}, {"GR_LANE_CANDIDATES": "1024"},
        {"GR_LANE_CANDIDATES": "2048"}, {"GR_LANE_CANDIDATES": "512"},
        {"GR_LANE_CANDIDATES": "2048", "GR_HOST_LOOP": "1"}]
for env in envs:
    for full in (False,):
        ids = idx if not full else idx + list(range(5))
        out = subprocess.run([sys.executable, "-c", code % (ids,)], env={**os.environ, **env},
                             capture_output=True, text=True)
        print(env, "full" if full else "subset", (out.stdout + out.stderr[-500:]).strip().replace("\n", " | "))
