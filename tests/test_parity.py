"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
element by element (status, assignment mask, cost; greedy pick order) on the
same seeded inputs.  Everything here is integer: the bar is bit-exact."""
import os
import random

import numpy as np
import pytest

import oracle
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
from gr_testutil import load_golden

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

try:
    import torch

    HAVE_GPU = torch.cuda.is_available()
except Exception:  # pragma: no cover
    HAVE_GPU = False

if not HAVE_GPU:
    pytest.skip("needs a CUDA device", allow_module_level=True)


def gpu_solve(cb, which, flags=0):
    db = gr.DeviceBatch.from_host(cb, flags=flags)
    fn = {"pms": gr.solve_pms, "mhs": gr.mhs_exact, "greedy": gr.mhs_greedy}[which]
    r = fn(db).to_host()
    torch.cuda.synchronize()
    return r


def assert_same(g, o, which, idx=None, decided=False):
    st = (o.status if idx is None else o.status[idx]).copy()
    # oracle -1: |support(phi+)| > 64, beyond the exact solvers (GR_UNSUPPORTED)
    assert (g["status"][st == -1] == gr.GR_UNSUPPORTED).all()
    keep = st != -1
    g = {k: v[keep] for k, v in g.items()}
    o = type(o)(o.status[keep], o.assign[keep], o.cost[keep], o.decided[keep])
    st = st[keep]
    bad = np.nonzero(g["status"] != st)[0]
    assert bad.size == 0, f"{which}: status differs at {bad[:10]} gpu={g['status'][bad[:10]]} oracle={st[bad[:10]]}"
    a = o.assign if idx is None else o.assign[idx]
    bad = np.nonzero((g["assign"] != a).any(axis=1))[0]
    assert bad.size == 0, f"{which}: assignment differs at {bad[:10]}"
    c = o.cost if idx is None else o.cost[idx]
    bad = np.nonzero(g["cost"] != c)[0]
    assert bad.size == 0, f"{which}: cost differs at {bad[:10]}"
    if decided:
        d = o.decided if idx is None else o.decided[idx]
        sat = (g["status"] == 0) | (g["status"] == 2)
        bad = np.nonzero(sat & (g["decided"] != d))[0]
        assert bad.size == 0, f"{which}: decided differs at {bad[:10]}"


def oracle_all(cb, weighted=True):
    return (oracle.batch("pms", cb, weighted=weighted), oracle.batch("mhs", cb),
            oracle.batch("greedy", cb))


def check_batch(cb, decided=True):
    p, h, g = oracle_all(cb)
    assert_same(gpu_solve(cb, "pms"), p, "pms", decided=decided and cb.w is None)
    assert_same(gpu_solve(cb, "mhs"), h, "mhs", decided=decided)
    assert_same(gpu_solve(cb, "greedy"), g, "greedy")


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("name", ["paper_example.txt", "unrepairable.txt", "write_write_race.txt"])
def test_golden(name):
    gd = load_golden(name)
    cb = synth.batch_from_lists([(gd["m"], gd["pos"], gd["neg"])], W=1)
    check_batch(cb)
    if name == "paper_example.txt":
        r = gpu_solve(cb, "pms")
        assert synth.mask_to_vars(r["assign"][0]) == [2, 3, 4]
        assert synth.mask_to_vars(gpu_solve(cb, "greedy")["assign"][0]) == [1, 2]


def test_c1():
    cb = synth.c1_instances()
    e = np.load(os.path.join(GOLDEN, "expected_c1.npz"))
    r = gpu_solve(cb, "pms")
    assert (r["status"] == e["pms_status"]).all() and (r["assign"] == e["pms_assign"]).all()
    assert (r["cost"] == e["pms_cost"]).all() and (r["decided"] == e["pms_decided"]).all()
    assert r["assign"][:, 0].tolist() == [14, 49]
    h = gpu_solve(cb, "mhs")
    assert (h["status"] == e["mhs_status"]).all() and (h["assign"] == e["mhs_assign"]).all()
    g = gpu_solve(cb, "greedy")
    assert (g["status"] == e["greedy_status"]).all() and (g["assign"] == e["greedy_assign"]).all()


# ------------------------------------------------------------------ fuzz
def rand_batch(seed, B, mmax, nmax, W=1, weighted=False, p_neg=0.3, edge=True):
    rng = random.Random(seed)
    insts, ws = [], []
    for i in range(B):
        m = rng.randint(0, mmax)
        pos, neg, seen = [], [], set()
        n = rng.randint(0, nmax) if m else rng.randint(0, 1)
        for _ in range(n):
            if m == 0:
                break
            s = rng.randint(1, min(m, rng.choice([2, 3, 4, 8])))
            c = tuple(sorted(rng.sample(range(1, m + 1), s)))
            isneg = rng.random() < p_neg
            if (isneg, c) in seen:
                continue
            seen.add((isneg, c))
            (neg if isneg else pos).append(list(c))
        if edge and rng.random() < 0.03:
            (pos if rng.random() < 0.5 else neg).append([])  # empty clause (R6)
        if edge and rng.random() < 0.03 and pos:
            pos.append(list(pos[0]))  # duplicate clause (R9)
        insts.append((m, pos, neg))
        ws.append([rng.randint(1, 100) for _ in range(max(m, 1))])
    return synth.batch_from_lists(insts, weights=ws if weighted else None, W=W)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_small_unit(seed):
    check_batch(rand_batch(seed, 300, 14, 16))


@pytest.mark.parametrize("seed", range(3))
def test_fuzz_small_weighted(seed):
    check_batch(rand_batch(100 + seed, 300, 14, 16, weighted=True))


@pytest.mark.parametrize("seed", range(3))
def test_fuzz_wide_masks(seed):
    # 33..64 variables (u64 lane path) with sparse clauses, and W = 2 inputs
    check_batch(rand_batch(200 + seed, 60, 40, 10, weighted=(seed == 1)))
    check_batch(rand_batch(300 + seed, 40, 100, 6, W=2))


def test_bad_inputs_and_unsupported():
    insts = [(4, [[1, 5]], []), (3, [[1]], [[2]]), (0, [], []), (2, [], [[1]]), (2, [[1, 2]], [[]])]
    cb = synth.batch_from_lists(insts, weights=[[1, 0], [1, 1, 1], [1], [5, 5], [1, 1]], W=1)
    cb.m[0] = 4  # b5 with m = 4 -> BADINPUT
    check_batch(cb)
    # > 64 support variables: exact solvers report UNSUPPORTED, greedy still works
    wide = synth.batch_from_lists([(100, [[i] for i in range(1, 80)], [])], W=2)
    r = gpu_solve(wide, "pms")
    assert r["status"][0] == gr.GR_UNSUPPORTED
    g = gpu_solve(wide, "greedy")
    st, a, _ = oracle.greedy(100, 79, wide.masks, W=2)
    assert g["status"][0] == st and (g["assign"][0] == a).all()


# ------------------------------------------------------------------ configs
def check_expected(cb, e, which, prefix, decided=False):
    r = gpu_solve(cb, which)
    for f in ("status", "assign", "cost"):
        exp = e[f"{prefix}_{f}"]
        got = r[f]
        bad = np.nonzero((got != exp).reshape(got.shape[0], -1).any(axis=1))[0]
        assert bad.size == 0, f"{prefix}.{f} differs at {bad[:10]}"
    if decided:
        sat = (r["status"] == 0) | (r["status"] == 2)
        bad = np.nonzero(sat & (r["decided"] != e[f"{prefix}_decided"]))[0]
        assert bad.size == 0, f"{prefix}.decided differs at {bad[:10]}"
    return r


def test_c2_full_batch():
    cb = synth.c2_batch()
    e = np.load(os.path.join(GOLDEN, "expected_c2.npz"))
    assert str(e["digest"]) == batch_digest(cb), "generator drift: re-run scripts/make_expected.py"
    check_expected(cb, e, "pms", "pms", decided=True)
    check_expected(cb, e, "mhs", "mhs", decided=True)
    check_expected(cb, e, "greedy", "greedy")
    # live oracle on a random sample of small instances
    idx = [b for b in range(cb.B) if cb.m[b] <= 16][:200]
    sub = cb.subset(idx)
    check_batch(sub)


def test_c2_level_loop_accounting():
    """The finish kernel's instance count drives the host level loop: after
    level k it is at most B, never grows, covers every instance whose optimum
    lies above k, and reaches 0 right after the last witness level (an
    uninitialised counter once let the loop run empty levels)."""
    cb = synth.c2_batch()
    e = np.load(os.path.join(GOLDEN, "expected_c2.npz"))
    sat = e["pms_status"] == gr.GR_SAT
    db = gr.DeviceBatch.from_host(cb)
    s = gr.ExactSession(db, gr.PMS)
    n = s.prepare()
    assert 0 <= n <= cb.B
    k, prev = 0, n
    while n:
        k += 1
        assert k <= 64
        s.level(k)
        n = s.finish(k)
        assert 0 <= n <= prev
        assert n >= int((sat & (e["pms_cost"] > k)).sum())
        prev = n
    assert k >= int(e["pms_cost"][sat].max())
    got = s.out.to_host()
    for f in ("status", "assign", "cost"):
        assert (got[f] == e[f"pms_{f}"]).all()


def test_c3_first_witness_exhaustive_and_shards():
    cb, H, grp = synth.c3_instance()
    e = np.load(os.path.join(GOLDEN, "expected_c3.npz"))
    for flags in (0, gr.GR_FLAG_EXHAUSTIVE):
        r = gpu_solve(cb, "pms", flags=flags)
        assert r["status"][0] == gr.GR_SAT
        assert int(r["assign"][0, 0]) == int(e["assign"])
        assert int(r["cost"][0]) == 16
    m, npos, mk, _ = cb.instance(0)
    assert oracle.feasible(int(r["assign"][0, 0]), npos, mk)
    # shard emulation: G sequential shards + host min == one GPU
    db = gr.DeviceBatch.from_host(cb)
    for G in (2, 3):
        s = gr.ExactSession(db, gr.PMS)
        s.prepare()
        n, k = 1, 0
        while n:
            k += 1
            keys = []
            for shard in range(G):
                s.level_keys().fill_(2**63 - 1)
                s.level(k, shard, G)
                keys.append(s.level_keys().clone())
            s.level_keys().copy_(torch.stack(keys).min(0).values)
            n = s.finish(k)
        got = s.out.to_host()
        assert int(got["assign"][0, 0]) == int(e["assign"]) and got["status"][0] == 0


def batch_digest(cb):
    import hashlib

    h = hashlib.sha256()
    for a in (cb.m, cb.off, cb.n_pos, cb.masks) + ((cb.w,) if cb.w is not None else ()):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_c4_full_batch():
    """All 10 000 C4 WPMS instances against the stored oracle
    results (scripts/make_expected.py, oracle only): status, assignment,
    weight and the decided count of the weighted level loop (every level up
    to the S_k stop), the MHS of every instance with its decided
    count, and the greedy; through the separate solves and through the one
    launch that serves WPMS + MHS together (gr_solve_pms_mhs)."""
    e = np.load(os.path.join(GOLDEN, "expected_c4.npz"))
    full = synth.c4_batch()
    assert str(e["digest"]) == batch_digest(full), "generator drift: re-run scripts/make_expected.py"
    r = check_expected(full, e, "pms", "pms")
    bad = np.nonzero(r["decided"] != e["pms_decided"])[0]
    assert bad.size == 0, f"pms.decided differs at {bad[:10]}"
    assert (r["status"] == 0).all()  # SAT by construction (planted H)
    check_expected(full, e, "mhs", "mhs", decided=True)
    check_expected(full, e, "greedy", "greedy")
    db = gr.DeviceBatch.from_host(full)
    p, h = gr.solve_pms_mhs(db)
    hp, hh = gr.to_host_many([p, h])
    for f in ("status", "assign", "cost", "decided"):
        assert np.array_equal(hp[f].reshape(full.B, -1), e[f"pms_{f}"].reshape(full.B, -1)), f
        assert np.array_equal(hh[f].reshape(full.B, -1), e[f"mhs_{f}"].reshape(full.B, -1)), f


# ------------------------------------------------------------------ greedy at scale
def csr_from_lists(cls):
    off = np.cumsum([0] + [len(c) for c in cls]).astype(np.int64)
    var = np.array([v for c in cls for v in c], np.int32)
    return off, var


def check_matrix(m, pos, neg, keep_csr=True, w=None):
    po, pv = csr_from_lists(pos)
    no, nv = csr_from_lists(neg)
    o = oracle.greedy_csr(m, po, pv, no, nv, w=w)
    bm = gr.pack_bitmatrix(m, po, pv, no, nv, keep_csr=keep_csr)
    if w is not None:
        bm.w = torch.from_numpy(np.asarray(w, np.uint32).view(np.int32)).cuda()
    assert bm.bad == 0
    r = gr.mhs_greedy_matrix(bm)
    torch.cuda.synchronize()
    assert r.n_picks == len(o.picks)
    assert r.picks.cpu().numpy()[: r.n_picks].tolist() == o.picks.tolist()
    a = r.assign.cpu().numpy().view(np.uint64)
    got = [i for i in range(m) if (int(a[i // 64]) >> (i % 64)) & 1]
    assert got == np.nonzero(o.in_S)[0].tolist()
    assert int(r.status.item()) == o.status


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("keep_csr", [True, False])  # incremental (f3) / recounting passes
def test_greedy_matrix_random(seed, keep_csr):
    rng = random.Random(seed)
    m = [7, 64, 300, 5000][seed]  # 5000 > 4096: the atomic (untiled) pack
    n = [1, 5000, 40000, 20000][seed]
    pos = [sorted(rng.sample(range(m), rng.randint(1, min(m, 6)))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), min(m, 2))) for _ in range(5)]
    check_matrix(m, pos, neg, keep_csr)


@pytest.mark.parametrize("keep_csr", [True, False])
def test_weighted_greedy_matrix(keep_csr):
    """f4 on the bit-matrix path (both the incremental and the recounting greedy)."""
    rng = random.Random(17)
    m, n = 300, 20000
    pos = [sorted(rng.sample(range(m), rng.randint(1, 6))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), 2)) for _ in range(5)]
    w = [rng.randint(1, 40) for _ in range(m)]
    check_matrix(m, pos, neg, keep_csr, w=w)


def test_pack_flags():
    """d_bad: 1 = id out of range, 2 = empty clause, 4 = repeated id."""
    for m in (100, 5000):
        for cls, want in (([[0, 1], [m]], 1), ([[0, 1], []], 2), ([[3, 3]], 4)):
            po, pv = csr_from_lists(cls)
            bm = gr.pack_bitmatrix(m, po, pv, np.zeros(1, np.int64), np.zeros(0, np.int32))
            assert bm.bad == want, (m, cls, bm.bad)


@pytest.mark.parametrize("keep_csr", [True, False])
def test_greedy_matrix_c5_shape_reduced(keep_csr):
    csr, H = synth.c5_clauses(m=4096, n=1 << 18)
    o = oracle.greedy_csr(csr.m, csr.pos_off, csr.pos_var.astype(np.int32), csr.neg_off, csr.neg_var)
    bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var,
                           keep_csr=keep_csr)
    r = gr.mhs_greedy_matrix(bm)
    torch.cuda.synchronize()
    assert r.picks.cpu().numpy()[: r.n_picks].tolist() == o.picks.tolist()
    a = r.assign.cpu().numpy().view(np.uint64)
    got = [i for i in range(csr.m) if (int(a[i // 64]) >> (i % 64)) & 1]
    assert got == np.nonzero(o.in_S)[0].tolist()
    assert int(r.status.item()) == o.status


_C5 = {}


def c5_full():
    if not _C5:
        import hashlib

        csr, H = synth.c5_clauses()
        h = hashlib.sha256()
        for a in (csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var):
            h.update(np.ascontiguousarray(a).tobytes())
        _C5.update(csr=csr, digest=h.hexdigest())
    return _C5["csr"], _C5["digest"]


@pytest.mark.parametrize("keep_csr", [False, True])  # recounting passes (north star) / f3
def test_c5_full_greedy_vs_oracle(keep_csr):
    """The full C5 greedy (m = 4096, n = 2^24 clauses, 8 GiB bit matrix) against
    the oracle's textbook recount greedy stored by scripts/make_expected.py:
    pick order, pruned set and phi- status (readings R11/R12)."""
    e = np.load(os.path.join(GOLDEN, "expected_c5.npz"))
    csr, digest = c5_full()
    assert str(e["digest"]) == digest, "generator drift: re-run scripts/make_expected.py c5"
    bm = gr.pack_bitmatrix(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var,
                           keep_csr=keep_csr)
    assert bm.bad == 0
    r = gr.mhs_greedy_matrix(bm)
    torch.cuda.synchronize()
    assert r.n_picks == e["picks"].size
    assert np.array_equal(r.picks.cpu().numpy()[: r.n_picks], e["picks"])
    a = r.assign.cpu().numpy().view(np.uint64)
    got = np.array([i for i in range(csr.m) if (int(a[i // 64]) >> (i % 64)) & 1], np.int32)
    assert np.array_equal(got, e["in_S"])
    assert int(r.status.item()) == int(e["status"])
    del bm, r
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ more paths
def _subprocess_solve(env, code):
    """Run a solve in a fresh process (the lane window is read once per process)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_small_lane_windows_split_sub_blocks():
    """L = 1 and 7 cut chunks and lane windows inside sub-blocks everywhere."""
    code = """
import numpy as np, oracle, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
import random
rng = random.Random(5)
insts = []
for _ in range(40):
    m = rng.randint(8, 18)
    pos = [sorted(rng.sample(range(1, m + 1), rng.randint(1, 4))) for _ in range(rng.randint(4, 20))]
    neg = [sorted(rng.sample(range(1, m + 1), rng.randint(1, 3))) for _ in range(rng.randint(0, 6))]
    insts.append((m, [list(c) for c in {tuple(c) for c in pos}], [list(c) for c in {tuple(c) for c in neg}]))
cb = synth.batch_from_lists(insts, weights=[[rng.randint(5, 9) for _ in range(40)] for _ in insts], W=1)
db = gr.DeviceBatch.from_host(cb)
for which, fn in (("pms", gr.solve_pms), ("mhs", gr.mhs_exact)):
    g = fn(db).to_host(); o = oracle.batch(which, cb)
    assert (g["status"] == o.status).all() and (g["assign"] == o.assign).all() and (g["cost"] == o.cost).all(), which
print("ok")
"""
    for L in ("1", "7", "300"):
        assert "ok" in _subprocess_solve({"GR_LANE_CANDIDATES": L}, code)


def test_c2_exhaustive_flag_same_results():
    cb = synth.c2_batch()
    e = np.load(os.path.join(GOLDEN, "expected_c2.npz"))
    for which, prefix in (("pms", "pms"), ("mhs", "mhs")):
        r = gpu_solve(cb, which, flags=gr.GR_FLAG_EXHAUSTIVE)
        for f in ("status", "assign", "cost"):
            assert (r[f].reshape(cb.B, -1) == e[f"{prefix}_{f}"].reshape(cb.B, -1)).all(), (which, f)


@pytest.mark.parametrize("extra", [0, gr.GR_FLAG_EXHAUSTIVE])
def test_no_prune_flag_same_results(extra):
    """GR_FLAG_NO_PRUNE (every sub-block decided by its own clause tests, no
    subtree refutation) gives the same statuses, assignments, costs and decided
    counts on C2, C4-shaped weighted instances and C3."""
    cases = [synth.c2_batch(), synth.c4_batch(B=300), synth.c3_instance()[0]]
    for cb in cases:
        for which in ("pms", "mhs"):
            a = gpu_solve(cb, which, flags=extra)
            b = gpu_solve(cb, which, flags=extra | gr.GR_FLAG_NO_PRUNE)
            for f in ("status", "assign", "cost", "decided"):
                assert (a[f] == b[f]).all(), (which, f)


def test_batch_shard_emulation():
    """Rank-range sharding of every level of a whole batch (G = 3 sequential
    shards, host MIN of the level keys) equals the single-GPU solve."""
    cb = rand_batch(77, 120, 24, 14, weighted=True)
    db = gr.DeviceBatch.from_host(cb)
    for which in (gr.PMS, gr.MHS):
        ref = (gr.solve_pms(db) if which == gr.PMS else gr.mhs_exact(db)).to_host()
        s = gr.ExactSession(db, which)
        n, k = s.prepare(), 0
        while n:
            k += 1
            keys = []
            for shard in range(3):
                s.level_keys().fill_(2**63 - 1)
                s.level(k, shard, 3)
                keys.append(s.level_keys().clone())
            s.level_keys().copy_(torch.stack(keys).min(0).values)
            n = s.finish(k)
        got = s.out.to_host()
        for f in ("status", "assign", "cost", "decided"):
            assert (got[f] == ref[f]).all(), (which, f)


def planted_instance(rng, m, n_pos, n_neg, h, smin=2, smax=5):
    """Every positive clause meets a planted set H (|H| = h), so k* <= h and the
    oracle finishes; negatives each keep a variable outside H."""
    H = set(rng.sample(range(1, m + 1), h))
    pos = set()
    while len(pos) < n_pos:
        c = tuple(sorted(rng.sample(range(1, m + 1), rng.randint(smin, smax))))
        if set(c) & H:
            pos.add(c)
    neg = set()
    while len(neg) < n_neg:
        c = tuple(sorted(rng.sample(range(1, m + 1), rng.randint(2, 3))))
        if not set(c) <= H:
            neg.add(c)
    return (m, [list(c) for c in pos], [list(c) for c in neg])


def test_many_clauses_global_memory_path():
    """> 512 packed clauses: records are read through L1 instead of shared memory."""
    rng = random.Random(3)
    insts = [planted_instance(rng, m, 600, 12, h) for m, h in ((20, 3), (30, 4), (44, 4), (60, 3))]
    check_batch(synth.batch_from_lists(insts, W=1))
    # weights in a narrow band keep the S_k >= W* stop within k* + 1 levels
    ws = [[rng.randint(10, 12) for _ in range(64)] for _ in insts]
    check_batch(synth.batch_from_lists(insts, weights=ws, W=1))


def test_wide_instances_many_clauses():
    """33..64 support variables with dense clause sets (u64 lanes, staged)."""
    rng = random.Random(11)
    insts = [planted_instance(rng, rng.randint(33, 64), rng.randint(40, 120), rng.randint(0, 20),
                              rng.randint(2, 6)) for _ in range(16)]
    ws = [[rng.randint(10, 12) for _ in range(64)] for _ in insts]
    check_batch(synth.batch_from_lists(insts, W=1))
    check_batch(synth.batch_from_lists(insts, weights=ws, W=1))


def test_greedy_count_shard_hook():
    """counts[v] over a column shard equals the plain count over its clauses."""
    rng = np.random.default_rng(2)
    m, n = 200, 3000
    cls = [sorted(rng.choice(m, size=int(rng.integers(1, 6)), replace=False).tolist()) for _ in range(n)]
    po, pv = csr_from_lists(cls)
    bm = gr.pack_bitmatrix(m, po, pv, np.zeros(1, np.int64), np.zeros(0, np.int32))
    U = torch.zeros(bm.ld, dtype=torch.int64, device="cuda")
    live = rng.random(n) < 0.6
    Uh = np.zeros(bm.ld, np.uint64)
    for c in np.nonzero(live)[0]:
        Uh[c // 64] |= np.uint64(1) << np.uint64(c % 64)
    U.copy_(torch.from_numpy(Uh.view(np.int64)))
    counts = torch.zeros(m, dtype=torch.int32, device="cuda")
    gr.greedy_count_shard(bm, U, counts)
    torch.cuda.synchronize()
    want = np.zeros(m, np.int64)
    for c in np.nonzero(live)[0]:
        for v in cls[c]:
            want[v] += 1
    assert (counts.cpu().numpy() == want).all()


@pytest.mark.parametrize("weighted", [False, True])
def test_composite_solve(weighted):
    """gr_solve (mhs strategy with MaxSAT fallback) == oracle."""
    cb = rand_batch(400 + weighted, 300, 14, 16, weighted=weighted)
    db = gr.DeviceBatch.from_host(cb)
    fb = torch.zeros(cb.B, dtype=torch.int32, device="cuda")
    g = gr.solve(db, gr.GR_STRATEGY_MHS, fell_back=fb).to_host()
    o = oracle.batch("solve", cb)
    assert (g["status"] == o.status).all()
    assert (g["assign"] == o.assign).all()
    assert (g["cost"] == o.cost).all()
    assert (fb.cpu().numpy() == o.decided.astype(np.int32)).all()
    assert fb.sum().item() > 0  # the fallback path ran
    m = gr.solve(db, gr.GR_STRATEGY_MAXSAT).to_host()
    p = oracle.batch("pms", cb)
    assert (m["status"] == p.status).all() and (m["assign"] == p.assign).all()


def test_incremental_kstart():
    """f2: start levels from the previous solve of a sub-formula give the full
    answer; decided equals the oracle's with the same start level."""
    rng = random.Random(8)
    base, grown = [], []
    for _ in range(150):
        m = rng.randint(10, 24)
        inst = planted_instance(rng, m, rng.randint(3, 20), rng.randint(0, 6), rng.randint(1, 5))
        base.append(inst)
        c = sorted(rng.sample(range(1, m + 1), rng.randint(1, 3)))
        grown.append((m, inst[1] + [c], inst[2]) if rng.random() < 0.6 else (m, inst[1], inst[2] + [c]))
    cb0 = synth.batch_from_lists(base, W=1)
    cb1 = synth.batch_from_lists(grown, W=1)
    r0 = gpu_solve(cb0, "pms")
    ks = np.where(r0["status"] == 0, r0["cost"].astype(np.int64), 1).astype(np.int32)
    db = gr.DeviceBatch.from_host(cb1)
    db.k_start = torch.from_numpy(ks).cuda()
    got = gr.solve_pms(db).to_host()
    full = oracle.batch("pms", cb1)
    assert (got["status"] == full.status).all() and (got["assign"] == full.assign).all()
    for b in range(cb1.B):
        m, npos, mk, _ = cb1.instance(b)
        o = oracle.pms_kstart(m, npos, mk, int(ks[b]))
        if o.status == 0:
            assert int(got["decided"][b]) == o.decided, b


@pytest.mark.parametrize("seed", range(3))
def test_weighted_greedy_and_solve(seed):
    """f4: the weighted mhs (ratio greedy) and the composite Solve built on it."""
    cb = rand_batch(500 + seed, 300, 30 if seed < 2 else 100, 16, weighted=True,
                    W=1 if seed < 2 else 2)
    db = gr.DeviceBatch.from_host(cb, flags=gr.GR_FLAG_WEIGHTED_GREEDY)
    g = gr.mhs_greedy(db).to_host()
    o = oracle.batch("greedy_w", cb)
    assert (g["status"] == o.status).all()
    assert (g["assign"] == o.assign).all()
    assert (g["cost"] == o.cost).all()
    if seed < 2:  # the exact fallback needs support <= 64
        fb = torch.zeros(cb.B, dtype=torch.int32, device="cuda")
        s = gr.solve(db, gr.GR_STRATEGY_MHS, fell_back=fb).to_host()
        so = oracle.batch("solve_w", cb)
        keep = so.status != -1
        assert (s["status"][keep] == so.status[keep]).all()
        assert (s["assign"][keep] == so.assign[keep]).all()
        assert (s["cost"][keep] == so.cost[keep]).all()


def test_pms_mhs_pair_on_two_streams():
    cb = synth.c2_batch()
    db = gr.DeviceBatch.from_host(cb)
    p, h = gr.solve_pms_mhs(db)
    p, h = p.to_host(), h.to_host()
    e = np.load(os.path.join(GOLDEN, "expected_c2.npz"))
    for f in ("status", "assign", "cost"):
        assert (p[f].reshape(cb.B, -1) == e[f"pms_{f}"].reshape(cb.B, -1)).all()
        assert (h[f].reshape(cb.B, -1) == e[f"mhs_{f}"].reshape(cb.B, -1)).all()
    rp, rh = gr.solve_pms(db).to_host(), gr.mhs_exact(db).to_host()
    assert (p["decided"] == rp["decided"]).all() and (h["decided"] == rh["decided"]).all()


# ------------------------------------------------------------------ column-sharded greedy
class _ThreadGroup:
    """In-process stand-in for the NCCL all-reduces of G ranks: one host
    thread per shard, all on this GPU; the exchange happens on the host between
    kernel launches (no kernel waits on another shard)."""

    def __init__(self, n):
        import threading

        self.n, self.bar, self.buf, self.res = n, threading.Barrier(n), [None] * n, None

    def allreduce(self, rank, op):
        def f(t):
            self.buf[rank] = t
            self.bar.wait()
            if rank == 0:
                acc = self.buf[0].clone()
                for x in self.buf[1:]:
                    acc = acc + x if op == "sum" else torch.maximum(acc, x)
                self.res = acc
            self.bar.wait()
            t.copy_(self.res)
            self.bar.wait()

        return f


def _shard_csr(po, pv, c0, c1):
    off = po[c0:c1 + 1] - po[c0]
    return off.astype(np.int64), pv[po[c0]:po[c1]]


@pytest.mark.parametrize("keep_csr", [True, False])  # incremental / recounting steps
@pytest.mark.parametrize("world", [1, 3])
def test_greedy_column_sharded(world, keep_csr):
    """gr_greedy_shard_* over G clause-column shards (G host threads on one
    GPU standing in for the ranks) = the oracle's greedy of the whole phi+."""
    import threading

    from paper_2011_08373_b200.multigpu import column_range, run_greedy_sharded

    rng = random.Random(5 + world)
    m, n = 300, 30000
    pos = [sorted(rng.sample(range(m), rng.randint(1, 6))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), 2)) for _ in range(6)]
    po, pv = csr_from_lists(pos)
    no, nv = csr_from_lists(neg)
    o = oracle.greedy_csr(m, po, pv, no, nv)
    grp = _ThreadGroup(world)
    out = [None] * world

    def run(r):
        c0, c1 = column_range(n, r, world)
        so, sv = _shard_csr(po, pv, c0, c1)
        bm = gr.pack_bitmatrix(m, so, sv, no, nv, keep_csr=keep_csr)
        sh = gr.GreedyShard(bm)
        out[r] = run_greedy_sharded(sh, grp.allreduce(r, "sum"), grp.allreduce(r, "max"),
                                    steps_per_check=8)
        torch.cuda.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for assign, status, picks, npk in out:
        assert picks.cpu().numpy()[:npk].tolist() == o.picks.tolist()
        a = assign.cpu().numpy().view(np.uint64)
        got = [i for i in range(m) if (int(a[i // 64]) >> (i % 64)) & 1]
        assert got == np.nonzero(o.in_S)[0].tolist()
        assert int(status.item()) == o.status


# ------------------------------------------------------------------ subtree refutation
def refutation_batch(seed, B, mlo, mhi, weighted=False):
    """Shapes that exercise the subtree refutation: many 1-3 variable positive
    clauses (empty restrictions, disjoint packings) and negative clauses that
    make dense levels UNSAT (negatives inside U); weights in a narrow band so
    the weight bound prunes (C4-like) or a wide one (it rarely does)."""
    rng = random.Random(seed)
    insts, ws = [], []
    for _ in range(B):
        m = rng.randint(mlo, mhi)
        pos, neg = set(), set()
        for _ in range(rng.randint(4, 30)):
            s = rng.choice([1, 2, 2, 3, 3, rng.randint(2, max(2, m // 3))])
            pos.add(tuple(sorted(rng.sample(range(1, m + 1), min(s, m)))))
        for _ in range(rng.randint(0, 14)):
            neg.add(tuple(sorted(rng.sample(range(1, m + 1), rng.choice([1, 2, 2, 3])))))
        insts.append((m, [list(c) for c in sorted(pos)], [list(c) for c in sorted(neg)]))
        lo = rng.choice([1, 50, 90])
        ws.append([rng.randint(lo, 100) for _ in range(m)])
    return synth.batch_from_lists(insts, weights=ws if weighted else None, W=1)


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("weighted", [False, True])
def test_refutation_shapes_vs_oracle(seed, weighted):
    cb = refutation_batch(100 + seed, 160, 10, 26, weighted)
    check_batch(cb)
    for which in ("pms", "mhs"):  # and the unpruned walk agrees
        a = gpu_solve(cb, which)
        b = gpu_solve(cb, which, flags=gr.GR_FLAG_NO_PRUNE)
        for f in ("status", "assign", "cost", "decided"):
            assert (a[f] == b[f]).all(), (which, f)


def test_batch_sharded_solve_threads():
    """solve_batch_sharded with G = 3 shards (host threads on this GPU, a host
    all-gather between them) = the single-GPU PMS of the whole batch."""
    import threading

    from paper_2011_08373_b200.multigpu import solve_batch_sharded

    cb = synth.c2_batch()
    ref = gpu_solve(cb, "pms")
    G = 3
    bar, buf, out = threading.Barrier(G), [None] * G, [None] * G
    lock = threading.Lock()  # one process per GPU has its own workspace; threads share one

    def run(r):
        def gather(t):
            buf[r] = t.clone()
            bar.wait()
            res = [x.clone() for x in buf]
            bar.wait()
            return res

        def solve(sub):
            with lock:
                return gr.solve_pms(gr.DeviceBatch.from_host(sub)).to_host()

        out[r] = solve_batch_sharded(cb, r, G, solve, gather)

    th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for o in out:
        for f in ("status", "cost", "decided"):
            assert (o[f] == ref[f]).all(), f
        assert (o["assign"].reshape(cb.B, -1) == ref["assign"].reshape(cb.B, -1)).all()


@pytest.mark.parametrize("case", ["fuzz", "refutation", "wide", "c3", "edge"])
def test_pms_mhs_fused_matches_separate(case):
    """gr_solve_pms_mhs (one walk deciding PMS and MHS, unit weights) gives
    the separate solvers' statuses, assignments, costs and decided counts."""
    if case == "fuzz":
        cb = rand_batch(7, 300, 20, 24)
    elif case == "refutation":
        cb = refutation_batch(31, 200, 10, 28)
    elif case == "wide":
        cb = rand_batch(8, 60, 44, 14)
    elif case == "c3":
        cb = synth.c3_instance()[0]
    else:  # empty negative clauses, empty phi+, duplicates (edge=True), m = 0
        cb = rand_batch(9, 400, 10, 12, edge=True, p_neg=0.5)
    db = gr.DeviceBatch.from_host(cb, weighted=False)
    p, h = gr.solve_pms_mhs(db)
    p, h = p.to_host(), h.to_host()
    rp, rh = gpu_solve(cb, "pms"), gpu_solve(cb, "mhs")
    for f in ("status", "assign", "cost", "decided"):
        assert (p[f] == rp[f]).all(), ("pms", f)
        assert (h[f] == rh[f]).all(), ("mhs", f)
    if case in ("fuzz", "edge"):
        o = oracle.batch("pms", cb)
        keep = o.status != -1
        assert (p["status"][keep] == o.status[keep]).all()


@pytest.mark.parametrize("which_cb", ["c2", "c3", "fuzz"])
def test_pms_mhs_fused_exhaustive(which_cb):
    """The fused walk with GR_FLAG_EXHAUSTIVE (witness level walked in full)
    = the separate exhaustive solvers, decided counts included."""
    cb = {"c2": lambda: synth.c2_batch(), "c3": lambda: synth.c3_instance()[0],
          "fuzz": lambda: rand_batch(11, 300, 20, 24)}[which_cb]()
    db = gr.DeviceBatch.from_host(cb, weighted=False, flags=gr.GR_FLAG_EXHAUSTIVE)
    p, h = gr.solve_pms_mhs(db)
    p, h = p.to_host(), h.to_host()
    rp = gpu_solve(cb, "pms", flags=gr.GR_FLAG_EXHAUSTIVE)
    rh = gpu_solve(cb, "mhs", flags=gr.GR_FLAG_EXHAUSTIVE)
    for f in ("status", "assign", "cost", "decided"):
        assert (p[f] == rp[f]).all(), ("pms", f)
        assert (h[f] == rh[f]).all(), ("mhs", f)


# ------------------------------------------------------------------ weighted prune order
@pytest.mark.parametrize("path", ["batched", "matrix_csr", "matrix_recount", "sharded3"])
def test_weighted_prune_order_golden_gpu(path):
    """tests/golden/weighted_prune_order.txt on every greedy path: the
    weighted mhs prunes in descending-weight order (reading R12)
    -> picks b1, b2, b3 and keeps {b2, b3} (weight 101)."""
    g = load_golden("weighted_prune_order.txt")
    m, pos, w, e = g["m"], g["pos"], g["w"], g["expect"]
    want = [int(x) for x in e["greedy"]]
    if path == "batched":
        cb = synth.batch_from_lists([(m, pos, [])], weights=[w], W=1)
        db = gr.DeviceBatch.from_host(cb, flags=gr.GR_FLAG_WEIGHTED_GREEDY)
        r = gr.mhs_greedy(db).to_host()
        assert synth.mask_to_vars(r["assign"][0]) == want
        assert int(r["cost"][0]) == int(e["greedy_cost"][0]) and r["status"][0] == 0
        return
    cls = [[v - 1 for v in c] for c in pos]
    po, pv = csr_from_lists(cls)
    no, nv = np.zeros(1, np.int64), np.zeros(0, np.int32)
    wt = torch.from_numpy(np.asarray(w, np.uint32).view(np.int32)).cuda()
    if path.startswith("matrix"):
        bm = gr.pack_bitmatrix(m, po, pv, no, nv, keep_csr=(path == "matrix_csr"))
        bm.w = wt
        r = gr.mhs_greedy_matrix(bm)
        assign, picks, npk = r.assign, r.picks, r.n_picks
    else:
        import threading

        from paper_2011_08373_b200.multigpu import column_range, run_greedy_sharded

        world = 3
        grp = _ThreadGroup(world)
        out = [None] * world

        def run(rk):
            c0, c1 = column_range(len(cls), rk, world)
            so, sv = _shard_csr(po, pv, c0, c1)
            bm = gr.pack_bitmatrix(m, so, sv, no, nv)
            bm.w = wt
            out[rk] = run_greedy_sharded(gr.GreedyShard(bm), grp.allreduce(rk, "sum"),
                                         grp.allreduce(rk, "max"), steps_per_check=4,
                                         w=np.asarray(w, np.uint32))
            torch.cuda.synchronize()

        th = [threading.Thread(target=run, args=(rk,)) for rk in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assign, _, picks, npk = out[0]
    torch.cuda.synchronize()
    assert [int(p) + 1 for p in picks.cpu().numpy()[:npk]] == [int(x) for x in e["picks"]]
    a = assign.cpu().numpy().view(np.uint64)
    assert [i + 1 for i in range(m) if (int(a[i // 64]) >> (i % 64)) & 1] == want


# ------------------------------------------------------------------ device level loop
def test_device_level_loop_matches_host_loop(tmp_path):
    """queue_kernel (the whole level loop in one persistent launch) and the
    level-synchronous host loop (GR_HOST_LOOP=1: one enumeration and one
    finish launch per level) give identical statuses, assignments, costs and
    decided counts: C2 and C3 fused PMS + MHS, C4-shaped WPMS + MHS in one
    launch, and the single solves."""
    code = """
import numpy as np, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
out = {}
cases = (("c2", synth.c2_batch(), 0), ("c4", synth.c4_batch(B=600), 0),
         ("c3", synth.c3_instance()[0], gr.GR_FLAG_EXHAUSTIVE), ("c3p", synth.c3_instance()[0], 0))
for name, cb, flags in cases:
    db = gr.DeviceBatch.from_host(cb, flags=flags)
    p, h = gr.solve_pms_mhs(db)
    a, b2 = gr.solve_pms(db), gr.mhs_exact(db)
    for tag, r in (("pair_pms", p), ("pair_mhs", h), ("pms", a), ("mhs", b2)):
        x = r.to_host()
        for f in ("status", "assign", "cost", "decided"):
            out[name + "_" + tag + "_" + f] = x[f]
np.savez(%r, **out)
print("ok")
"""
    res = {}
    # speculation 4 levels deep on every level size, no speculation, small windows
    modes = (("queue", {}), ("host", {"GR_HOST_LOOP": "1"}),
             ("queue_spec4", {"GR_QSPEC": "4", "GR_QSPEC_MAX": "18446744073709551615"}),
             ("queue_nospec", {"GR_QSPEC": "0"}),
             ("queue_small", {"GR_QLANE_MIN": "256", "GR_QLANE_MAX": "4096"}))
    for mode, env in modes:
        path = str(tmp_path / f"{mode}.npz")
        assert "ok" in _subprocess_solve(env, code % path)
        res[mode] = np.load(path)
    for mode, _ in modes[1:]:
        for k in res["queue"].files:
            assert np.array_equal(res["queue"][k], res[mode][k]), (mode, k)


@pytest.mark.parametrize("case", ["c2", "c3", "c3x"])
def test_pair_session_shard_emulation(case):
    """The fused PMS + MHS pair session (gr_pair_*) with every level's rank
    range split into G = 3 shards run one after the other on this GPU (host
    MIN of both key arrays, as the NCCL all-reduce does) equals
    gr_solve_pms_mhs: statuses, assignments, costs, decided counts."""
    if case == "c2":
        cb, flags = synth.c2_batch(), 0
    else:
        cb, flags = synth.c3_instance()[0], (gr.GR_FLAG_EXHAUSTIVE if case == "c3x" else 0)
    db = gr.DeviceBatch.from_host(cb, weighted=False, flags=flags)
    p, h = gr.solve_pms_mhs(db)
    ref = gr.to_host_many([p, h])
    s = gr.PairSession(db)
    n, k = s.prepare(), 0
    while n:
        k += 1
        got = [[], []]
        for shard in range(3):
            kp, km = s.level_keys()
            saved = (kp.clone(), km.clone())
            s.level(k, shard, 3)
            for i, t in enumerate(s.level_keys()):
                got[i].append(t.clone())
                t.copy_(saved[i])
        for i, t in enumerate(s.level_keys()):
            t.copy_(torch.stack(got[i]).min(0).values)
        n = s.finish(k)
    out = gr.to_host_many([s.out_pms, s.out_mhs])
    for i in (0, 1):
        for f in ("status", "assign", "cost", "decided"):
            assert np.array_equal(out[i][f], ref[i][f]), (case, i, f)


def test_long_windows_at_32_support_variables():
    """Regression (round 2): with m_eff = 32 exactly the iterator's 5-bit
    ancestor stack could not hold e_top = 32; a long lane window that popped
    back to depth 1 lost the rest of the level.  Instances with exactly 32
    support variables, unit and weighted, under long fixed lane windows
    (2^11 .. 2^20 candidates), against the oracle -- including C4 instance
    2649 where the optimum was missed."""
    code = """
import random, numpy as np, oracle, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
rng = random.Random(32)
insts, ws = [], []
for _ in range(60):
    m = rng.randint(32, 40)
    sup = sorted(rng.sample(range(1, m + 1), 32))
    pos = {tuple(sorted(rng.sample(sup, rng.randint(2, 5)))) for _ in range(rng.randint(6, 12))}
    pos |= {tuple(sup[i:i + 3]) for i in range(0, 30, 10)}
    neg = {tuple(sorted(rng.sample(sup, rng.randint(1, 3)))) for _ in range(rng.randint(0, 6))}
    insts.append((m, [list(c) for c in pos], [list(c) for c in neg]))
    ws.append([rng.randint(50, 100) for _ in range(40)])
c4 = synth.c4_batch().subset([2649])
for cb in (synth.batch_from_lists(insts, weights=ws, W=1), c4):
    for weighted in (True, False):
        db = gr.DeviceBatch.from_host(cb, weighted=weighted)
        p, h = gr.solve_pms_mhs(db)
        a, b = gr.to_host_many([p, h])
        op = oracle.batch("pms", cb, weighted=weighted)
        oh = oracle.batch("mhs", cb)
        for g, o in ((a, op), (b, oh)):
            assert (g["status"] == o.status).all() and (g["assign"] == o.assign).all()
            assert (g["cost"] == o.cost).all()
print("ok")
"""
    for L in ("2048", "65536", "1048576"):
        assert "ok" in _subprocess_solve({"GR_LANE_CANDIDATES": L}, code)


@pytest.mark.parametrize("weighted", [False, True])
def test_final_maxsat_query(weighted):
    """GR_STRATEGY_MHS_FINAL, the mhs strategy's final 'single query to a
    MaxSAT solver ... to ensure that the number of b_i's being set to true is
    the minimum': every instance gets the oracle's (weighted)
    PMS optimum; fell_back flags exactly the instances whose greedy answer
    broke phi- or was not minimum."""
    cb = rand_batch(600 + weighted, 300, 14, 16, weighted=weighted)
    db = gr.DeviceBatch.from_host(cb)
    fb = torch.zeros(cb.B, dtype=torch.int32, device="cuda")
    r = gr.solve(db, gr.GR_STRATEGY_MHS_FINAL, fell_back=fb).to_host()
    p = oracle.batch("pms", cb)
    g = oracle.batch("greedy", cb)
    keep = p.status != -1
    for f, o in (("status", p.status), ("assign", p.assign), ("cost", p.cost)):
        assert (r[f][keep] == o[keep]).all(), f
    want = np.zeros(cb.B, np.int32)
    for b in range(cb.B):
        if g.status[b] != 0:
            want[b] = 1
            continue
        chosen = [v - 1 for v in synth.mask_to_vars(g.assign[b])]  # 0-based
        gcost = sum(int(cb.w[b, v]) for v in chosen) if weighted else len(chosen)
        want[b] = int(p.status[b] == 0 and int(p.cost[b]) < gcost)
    got = fb.cpu().numpy()
    assert (got[keep] == want[keep]).all()
    assert want.sum() > 0 and (want == 0).sum() > 0


def test_weighted_key_overflow_unsupported():
    """A weighted key (W << rb | rank) that would not fit 63 bits gives
    GR_UNSUPPORTED for that instance, on the device level loop
    and on the host loop; the other instances of the batch are unaffected.
    Ten disjoint 4-variable clauses put the optimum at level 10 of m = 40;
    with weights near 2^31 the level-9 key needs bitlen(40 * 2^31) +
    bitlen(C(40, 9) - 1) = 37 + 28 > 63 bits."""
    pos = [list(range(4 * i + 1, 4 * i + 5)) for i in range(10)]
    insts = [(40, pos, []), (40, [[1, 2], [3, 4]], [[1]])]
    ws = [[(1 << 31) + i for i in range(40)], [(1 << 31) + i for i in range(40)]]
    cb = synth.batch_from_lists(insts, weights=ws, W=1)
    code = """
import numpy as np, oracle, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
pos = [list(range(4 * i + 1, 4 * i + 5)) for i in range(10)]
insts = [(40, pos, []), (40, [[1, 2], [3, 4]], [[1]])]
ws = [[(1 << 31) + i for i in range(40)], [(1 << 31) + i for i in range(40)]]
cb = synth.batch_from_lists(insts, weights=ws, W=1)
r = gr.solve_pms(gr.DeviceBatch.from_host(cb)).to_host()
o = oracle.batch("pms", cb)
assert r["status"][0] == gr.GR_UNSUPPORTED, r["status"]
assert r["status"][1] == o.status[1] == 0 and (r["assign"][1] == o.assign[1]).all() and r["cost"][1] == o.cost[1]
print("ok")
"""
    for env in ({}, {"GR_HOST_LOOP": "1"}):
        assert "ok" in _subprocess_solve(env, code)


# ------------------------------------------------------------------ greedy from lists (f3)
def check_lists(m, pos, neg, w=None):
    po, pv = csr_from_lists(pos)
    no, nv = csr_from_lists(neg)
    o = oracle.greedy_csr(m, po, pv, no, nv, w=w)
    wt = None if w is None else torch.from_numpy(np.asarray(w, np.uint32).view(np.int32)).cuda()
    r = gr.mhs_greedy_lists(m, po, pv.astype(np.int32), no, nv.astype(np.int32), w=wt)
    torch.cuda.synchronize()
    assert r.n_picks == len(o.picks)
    assert r.picks.cpu().numpy()[: r.n_picks].tolist() == o.picks.tolist()
    a = r.assign.cpu().numpy().view(np.uint64)
    got = [i for i in range(m) if (int(a[i // 64]) >> (i % 64)) & 1]
    assert got == np.nonzero(o.in_S)[0].tolist()
    assert int(r.status.item()) == o.status


@pytest.mark.parametrize("seed", range(4))
def test_greedy_lists_random(seed):
    """gr_mhs_greedy_lists (no bit matrix: device-built variable -> clause
    lists) = the oracle's textbook greedy: picks, pruned set, phi- status."""
    rng = random.Random(900 + seed)
    m = [7, 64, 300, 5000][seed]
    n = [1, 5000, 40000, 20000][seed]
    pos = [sorted(rng.sample(range(m), rng.randint(1, min(m, 6)))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), min(m, 2))) for _ in range(5)]
    check_lists(m, pos, neg)


def test_greedy_lists_weighted_and_golden():
    """The weighted mhs (R20) from lists, and the prune-order golden
    instance (descending weight, R12)."""
    rng = random.Random(19)
    m, n = 300, 20000
    pos = [sorted(rng.sample(range(m), rng.randint(1, 6))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), 2)) for _ in range(5)]
    check_lists(m, pos, neg, w=[rng.randint(1, 40) for _ in range(m)])
    g = load_golden("weighted_prune_order.txt")
    check_lists(g["m"], [[v - 1 for v in c] for c in g["pos"]], [], w=g["w"])


def test_greedy_lists_long_clauses_int16_unaligned():
    """Tiles whose literals exceed the scatter's shared literal map (clauses of
    20-60 variables: the thread-per-clause fallback), and int16 ids handed
    over as a slice that is not 16-byte aligned (the binding copies it)."""
    rng = random.Random(77)
    m, n = 3000, 3000
    pos = [sorted(rng.sample(range(m), rng.randint(20, 60))) for _ in range(n)]
    neg = [sorted(rng.sample(range(m), 2)) for _ in range(4)]
    check_lists(m, pos, neg)
    po, pv = csr_from_lists(pos)
    no, nv = csr_from_lists(neg)
    o = oracle.greedy_csr(m, po, pv, no, nv)
    buf = torch.zeros(pv.size + 1, dtype=torch.int16, device="cuda")
    buf[1:] = torch.from_numpy(pv.astype(np.int16)).cuda()
    pv16 = buf[1:]  # data_ptr % 16 == 2
    assert pv16.data_ptr() % 16 != 0
    r = gr.mhs_greedy_lists(m, po, pv16, no, nv.astype(np.int16))
    torch.cuda.synchronize()
    assert r.picks.cpu().numpy()[: r.n_picks].tolist() == o.picks.tolist()
    assert int(r.status.item()) == o.status


def test_greedy_lists_bad_and_empty():
    po, pv = csr_from_lists([[0, 1], [5]])
    r = gr.mhs_greedy_lists(4, po, pv, np.zeros(1, np.int64), np.zeros(0, np.int32))
    assert int(r.status.item()) == gr.GR_BADINPUT
    po, pv = csr_from_lists([[0, 1], []])
    r = gr.mhs_greedy_lists(4, po, pv, np.zeros(1, np.int64), np.zeros(0, np.int32))
    assert int(r.status.item()) == gr.GR_UNSAT


def test_c5_full_greedy_lists_vs_oracle():
    """The full C5 (2^24 clauses) through the list greedy, against the
    oracle's stored result."""
    e = np.load(os.path.join(GOLDEN, "expected_c5.npz"))
    csr, digest = c5_full()
    assert str(e["digest"]) == digest
    r = gr.mhs_greedy_lists(csr.m, csr.pos_off, csr.pos_var, csr.neg_off, csr.neg_var)
    torch.cuda.synchronize()
    assert r.n_picks == e["picks"].size
    assert np.array_equal(r.picks.cpu().numpy()[: r.n_picks], e["picks"])
    a = r.assign.cpu().numpy().view(np.uint64)
    got = np.array([i for i in range(csr.m) if (int(a[i // 64]) >> (i % 64)) & 1], np.int32)
    assert np.array_equal(got, e["in_S"])
    assert int(r.status.item()) == int(e["status"])


@pytest.mark.gpu
def test_solve_step_side_stream_matches_serial():
    """gr.solve_step (greedy on a side stream beside the PMS + MHS launch)
    gives the serial calls' results, on C2 (the bench's step)."""
    cb = synth.c2_batch()
    db = gr.DeviceBatch.from_host(cb)
    p, h = gr.solve_pms_mhs(db)
    g = gr.mhs_greedy(db)
    ref = gr.to_host_many([p, h, g])
    for _ in range(3):
        outs = gr.solve_step(db)
        got = gr.to_host_many(list(outs))
        for a, b in zip(got, ref):
            for k in ("status", "cost", "assign", "decided"):
                assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
def test_step_graph_replays_match():
    """gr.StepGraph (solve_step captured as a CUDA graph) gives the launched
    step's results on every replay (the ticket ring is cleared per launch)."""
    cb = synth.c2_batch()
    db = gr.DeviceBatch.from_host(cb)
    ref = gr.to_host_many(list(gr.solve_step(db)))
    g = gr.StepGraph(db)
    for _ in range(3):
        got = gr.to_host_many(g.replay())
        for a, b in zip(got, ref):
            for k in ("status", "cost", "assign", "decided"):
                assert np.array_equal(a[k], b[k]), k


def test_fused_time_slices_split_windows():
    """Tiny time slices (2000 clocks, shares down to 1 candidate) make the
    fused walk hand window remainders to idle lanes all the time: the
    results and decided counts of C2 stay the oracle's."""
    code = """
import os, numpy as np, paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
cb = synth.c2_batch()
e = np.load(os.path.join("tests", "golden", "expected_c2.npz"))
db = gr.DeviceBatch.from_host(cb)
for _ in range(2):
    p, h = gr.solve_pms_mhs(db)
    a, b = gr.to_host_many([p, h])
    for r, pre in ((a, "pms"), (b, "mhs")):
        assert (r["status"] == e[pre + "_status"]).all(), pre
        assert (r["cost"] == e[pre + "_cost"]).all(), pre
        assert (r["assign"].reshape(-1) == e[pre + "_assign"].reshape(-1)).all(), pre
        sat = e[pre + "_status"] == gr.GR_SAT
        assert (r["decided"][sat] == e[pre + "_decided"][sat]).all(), pre
print("ok")
"""
    assert "ok" in _subprocess_solve({"GR_QSLICE": "2000", "GR_QSPLIT_MIN": "1"}, code)
