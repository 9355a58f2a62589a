"""The seeded input recipes: shapes,
distinctness, planted structure and determinism.  CPU only."""
import numpy as np

import oracle
from paper_2011_08373_b200 import synth


def test_c2_recipe():
    cb = synth.c2_batch()
    assert cb.B == 748 and cb.W == 1
    assert (cb.m >= 0).all() and (cb.m <= 32).all()
    n = np.diff(cb.off)
    assert (n <= 64).all() and (n[cb.m == 0] == 0).all()
    for b in range(cb.B):
        m, npos, mk, _ = cb.instance(b)
        allowed = np.uint64((1 << m) - 1) if m < 64 else np.uint64(~0 & ((1 << 64) - 1))
        assert ((mk[:, 0] & ~allowed) == 0).all()
        assert len(set(mk[:npos, 0].tolist())) == npos  # distinct positives
        assert len(set(mk[npos:, 0].tolist())) == mk.shape[0] - npos
    # the m histogram follows PAPER.md:593-602 roughly (203/734 kernels have m = 0)
    assert 0.2 < (cb.m == 0).mean() < 0.35
    neg_frac = 1 - cb.n_pos.sum() / max(int(cb.off[-1]), 1)
    assert 0.15 < neg_frac < 0.35


def test_c2_deterministic():
    a, b = synth.c2_batch(), synth.c2_batch()
    assert (a.masks == b.masks).all() and (a.off == b.off).all()
    c = synth.c2_batch(seed=synth.seed_for(2, rank=1))
    assert not (c.masks.shape == a.masks.shape and (c.masks == a.masks).all())


def test_c4_recipe_planted_sat():
    cb = synth.c4_batch(B=40)
    assert (cb.m == 40).all() and cb.w is not None
    assert (cb.w[:, :40] >= 50).all() and (cb.w[:, :40] <= 100).all()
    n = np.diff(cb.off)
    assert (n >= 16).all() and (n <= 64).all()
    for b in range(cb.B):
        m, npos, mk, w = cb.instance(b)
        assert all(bin(int(x)).count("1") >= 2 for x in mk[:npos, 0])  # positive size >= 2
        assert oracle.pms(m, npos, mk, w=w).status == oracle.SAT  # SAT by construction


def test_c5_recipe_small():
    csr, H = synth.c5_clauses(m=512, n=20000, n_planted=32)
    assert csr.n_pos == 20000 and csr.n_neg == 64
    Hs = set(H.tolist())
    rows = [tuple(csr.pos_var[csr.pos_off[c]:csr.pos_off[c + 1]].tolist()) for c in range(csr.n_pos)]
    assert len(set(rows)) == len(rows)  # distinct clauses
    for r in rows:
        assert 3 <= len(r) <= 16 and len(set(r)) == len(r) and set(r) & Hs
    # the planted set hits every clause: the greedy set is no larger than H(Delta+) x |H|
    g = oracle.greedy_csr(csr.m, csr.pos_off, csr.pos_var.astype(np.int32), csr.neg_off, csr.neg_var)
    assert g.n_final <= len(H) * sum(1.0 / i for i in range(1, csr.n_pos + 1))


def test_paper_weights_formula():
    rng = np.random.default_rng(3)
    w = synth.paper_weights(rng, 5000)
    assert set(np.unique(w).tolist()) <= {1, 10, 100, 13, 22, 112}
