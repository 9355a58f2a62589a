import os, random, sys
import numpy as np
sys.path.insert(0, ".")
import oracle, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
rng = random.Random(5)
insts = []
for _ in range(40):
    m = rng.randint(8, 18)
    pos = [sorted(rng.sample(range(1, m + 1), rng.randint(1, 4))) for _ in range(rng.randint(4, 20))]
    neg = [sorted(rng.sample(range(1, m + 1), rng.randint(1, 3))) for _ in range(rng.randint(0, 6))]
    insts.append((m, [list(c) for c in {tuple(c) for c in pos}], [list(c) for c in {tuple(c) for c in neg}]))
ws = [[rng.randint(5, 9) for _ in range(40)] for _ in insts]
for weighted in (False, True):
    cb = synth.batch_from_lists(insts, weights=ws if weighted else None, W=1)
    db = gr.DeviceBatch.from_host(cb)
    for which, fn in (("pms", gr.solve_pms), ("mhs", gr.mhs_exact)):
        g = fn(db).to_host(); o = oracle.batch(which, cb)
        bad = np.nonzero((g["status"] != o.status) | (g["assign"][:, 0] != o.assign[:, 0]) | (g["cost"] != o.cost))[0]
        print(os.environ.get("GR_LANE_CANDIDATES"), "weighted" if weighted else "unit", which, "bad", bad.tolist())
        for b in bad[:3]:
            m, npos, mk, w = cb.instance(int(b))
            print("   inst", b, "m", m, "npos", npos, "nneg", mk.shape[0]-npos, "gpu", g["status"][b], synth.mask_to_vars(g["assign"][b]), g["cost"][b], "oracle", o.status[b], synth.mask_to_vars(o.assign[b]), o.cost[b])
