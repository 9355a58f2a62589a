"""Write tests/golden/expected_*.npz -- stored oracle results for the seeded
workloads.  Calls only oracle/ (and the shared input generator synth.py); no
value here comes from the CUDA path.

    python scripts/make_expected.py [c1 c2 c3 c4 c5]
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2011_08373_b200 import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def digest(cb) -> str:
    h = hashlib.sha256()
    for a in (cb.m, cb.off, cb.n_pos, cb.masks) + ((cb.w,) if cb.w is not None else ()):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def save(name, cb, **res):
    path = os.path.join(OUT, f"expected_{name}.npz")
    np.savez_compressed(path, digest=np.array(digest(cb)), **res)
    print("wrote", path)


def run_batch(cb, which, weighted=True):
    t = time.time()
    r = oracle.batch(which, cb, reduce=1, weighted=weighted)
    print(f"  oracle {which}: {time.time() - t:.1f}s")
    return r


def main(which):
    if "c1" in which:
        cb = synth.c1_instances()
        p, h, g = run_batch(cb, "pms"), run_batch(cb, "mhs"), run_batch(cb, "greedy")
        save("c1", cb, pms_status=p.status, pms_assign=p.assign, pms_cost=p.cost,
             pms_decided=p.decided, mhs_status=h.status, mhs_assign=h.assign, mhs_cost=h.cost,
             greedy_status=g.status, greedy_assign=g.assign, greedy_cost=g.cost)
    if "c2" in which:
        cb = synth.c2_batch()
        p, h, g = run_batch(cb, "pms"), run_batch(cb, "mhs"), run_batch(cb, "greedy")
        save("c2", cb, pms_status=p.status, pms_assign=p.assign, pms_cost=p.cost,
             pms_decided=p.decided, mhs_status=h.status, mhs_assign=h.assign, mhs_cost=h.cost,
             mhs_decided=h.decided, greedy_status=g.status, greedy_assign=g.assign,
             greedy_cost=g.cost)
    if "c3" in which:
        cb, H, grp = synth.c3_instance()
        m, npos, mk, _ = cb.instance(0)
        nfeas, best = oracle.min_feasible_product(grp, npos, mk)
        save("c3", cb, n_feasible_product=np.array(nfeas), assign=np.array(best, np.uint64),
             planted=np.array(sum(1 << v for v in H), np.uint64))
    if "c4" in which:  # all 10 000 WPMS instances, their MHS and greedy
        cb = synth.c4_batch()
        p, h, g = run_batch(cb, "pms"), run_batch(cb, "mhs"), run_batch(cb, "greedy")
        save("c4", cb, pms_status=p.status, pms_assign=p.assign, pms_cost=p.cost,
             pms_decided=p.decided, mhs_status=h.status, mhs_assign=h.assign, mhs_cost=h.cost,
             mhs_decided=h.decided, greedy_status=g.status, greedy_assign=g.assign,
             greedy_cost=g.cost)
    if "c5" in which:  # the full 2^24-clause greedy
        t = time.time()
        csr, H = synth.c5_clauses()
        print(f"  c5 generated in {time.time() - t:.1f}s")
        t = time.time()
        g = oracle.greedy_csr(csr.m, csr.pos_off, csr.pos_var.astype(np.int32), csr.neg_off,
                              csr.neg_var)
        print(f"  oracle greedy: {time.time() - t:.1f}s, {len(g.picks)} picks, |S| = {g.n_final}")
        h = hashlib.sha256()
        for a in (csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var):
            h.update(np.ascontiguousarray(a).tobytes())
        path = os.path.join(OUT, "expected_c5.npz")
        np.savez_compressed(path, digest=np.array(h.hexdigest()), picks=g.picks.astype(np.int32),
                            in_S=np.flatnonzero(g.in_S).astype(np.int32), status=np.array(g.status),
                            n_final=np.array(g.n_final))
        print("wrote", path)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
