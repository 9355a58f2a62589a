"""Pins for the CPU oracle: the oracle is checked against
what the paper and the mathematics fix, never against itself.

* the paper's worked example and case studies (tests/golden/*.txt, cited);
* closed forms (disjoint clauses, paths, complete graphs, stars);
* an independent brute force written here over Python *sets* (not masks);
* Koenig's theorem (min vertex cover = max matching in bipartite graphs);
* the colex-rank closed form of the level-enumeration candidate count;
* the defining invariants of a (minimal) hitting set and Johnson's bound.
"""
import itertools
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2011_08373_b200 import synth
from gr_testutil import load_golden

SAT, UNSAT, NEGV, BAD = oracle.SAT, oracle.UNSAT, oracle.SAT_NEG_VIOLATED, oracle.BADINPUT
STATUS = {"SAT": SAT, "UNSAT": UNSAT, "SAT_NEG_VIOLATED": NEGV, "BADINPUT": BAD}


def masks_of(pos, neg, W=1):
    cb = synth.batch_from_lists([(64 * W, pos, neg)], W=W)
    return cb.masks


def vars_of(mask):
    """joined assignment mask (any width) -> sorted 1-based b_i"""
    mask = int(mask)
    return [i + 1 for i in range(mask.bit_length()) if mask >> i & 1]


# ---------------------------------------------------------------- golden pins
def test_paper_example_p1():
    g = load_golden("paper_example.txt")
    m, pos, neg, e = g["m"], g["pos"], g["neg"], g["expect"]
    mk = masks_of(pos, neg)
    st, a, picks = oracle.greedy(m, len(pos), mk)
    assert synth.mask_to_vars(a) == [int(x) for x in e["greedy"]]
    assert st == STATUS[e["greedy_status"][0]]
    r = oracle.mhs(m, len(pos), mk)
    assert vars_of(r.assign) == [int(x) for x in e["mhs"]]
    assert r.status == STATUS[e["mhs_status"][0]]
    for reduce in (0, 1):
        r = oracle.pms(m, len(pos), mk, reduce=reduce)
        assert r.status == SAT
        assert vars_of(r.assign) == [int(x) for x in e["pms"]]
        assert r.cost == int(e["pms_cost"][0])


@pytest.mark.parametrize("name", ["unrepairable.txt", "write_write_race.txt"])
def test_case_study_unsat(name):
    g = load_golden(name)
    m, pos, neg, e = g["m"], g["pos"], g["neg"], g["expect"]
    mk = masks_of(pos, neg)
    if "pms_status" in e:
        for reduce in (0, 1):
            assert oracle.pms(m, len(pos), mk, reduce=reduce).status == STATUS[e["pms_status"][0]]
        assert oracle.pms_brute(m, len(pos), mk).status == STATUS[e["pms_status"][0]]
    if "mhs_status" in e:
        assert oracle.mhs(m, len(pos), mk).status == STATUS[e["mhs_status"][0]]
    if "greedy_status" in e:
        assert oracle.greedy(m, len(pos), mk)[0] == STATUS[e["greedy_status"][0]]


def colex_rank(vars1):
    """Combinatorial number system: rank = sum_j C(c_j, j), c_1 < c_2 < ... (0-based)."""
    return sum(math.comb(c - 1, j + 1) for j, c in enumerate(sorted(vars1)))


def test_c1_instances_p2_p3():
    """C1 instances A and B (m = 8).  The candidate count of the
    plain levelled enumeration is fixed by the closed form
    sum_{k<k*} C(m,k) + colex_rank + 1 (first witness ends the search)."""
    cb = synth.c1_instances()
    exp = [([2, 3, 4], 14), ([1, 5, 6], 49)]
    for b in range(2):
        m, npos, mk, _ = cb.instance(b)
        r = oracle.pms(m, npos, mk, reduce=0)
        assert (r.status, r.assign, r.cost) == (SAT, exp[b][1], 3)
        assert vars_of(r.assign) == exp[b][0]
        want = sum(math.comb(8, k) for k in range(3)) + colex_rank(exp[b][0]) + 1
        assert r.decided == want
    assert [41, 54] == [sum(math.comb(8, k) for k in range(3)) + colex_rank(v) + 1 for v, _ in exp]


# ---------------------------------------------------------------- closed forms
def test_triangle_p4_colex_tiebreak():
    mk = masks_of([[1, 2], [1, 3], [2, 3]], [])
    assert vars_of(oracle.mhs(3, 3, mk).assign) == [1, 2]
    assert vars_of(oracle.pms(3, 3, mk).assign) == [1, 2]


@pytest.mark.parametrize("sizes", [[1], [2, 3], [3, 1, 4, 2], [5, 5, 5]])
def test_disjoint_clauses_p5(sizes):
    pos, v = [], 1
    for s in sizes:
        pos.append(list(range(v, v + s)))
        v += s
    m = v - 1
    mk = masks_of(pos, [])
    want = [c[0] for c in pos]
    assert vars_of(oracle.mhs(m, len(pos), mk).assign) == want
    st, a, _ = oracle.greedy(m, len(pos), mk)
    assert st == SAT and synth.mask_to_vars(a) == want


@pytest.mark.parametrize("m,mhs_vars,greedy_vars", [
    (2, [1], [1]), (3, [2], [2]), (4, [1, 3], [2, 3]), (5, [2, 4], None), (7, [2, 4, 6], None)])
def test_path_p6(m, mhs_vars, greedy_vars):
    pos = [[i, i + 1] for i in range(1, m)]
    mk = masks_of(pos, [])
    r = oracle.mhs(m, len(pos), mk)
    assert r.cost == m // 2  # minimum vertex cover of a path on m vertices
    assert vars_of(r.assign) == mhs_vars
    if greedy_vars is not None:
        assert synth.mask_to_vars(oracle.greedy(m, len(pos), mk)[1]) == greedy_vars


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_complete_graph_p7(n):
    pos = [list(e) for e in itertools.combinations(range(1, n + 1), 2)]
    r = oracle.mhs(n, len(pos), masks_of(pos, []))
    assert r.cost == n - 1 and vars_of(r.assign) == list(range(1, n))


def test_star_p8():
    pos = [[1, j] for j in range(2, 6)]
    assert vars_of(oracle.mhs(5, 4, masks_of(pos, [])).assign) == [1]
    r = oracle.pms(5, 4, masks_of(pos, [[1]]))
    assert vars_of(r.assign) == [2, 3, 4, 5] and r.cost == 4


def test_unsat_p9_and_empty_clauses():
    assert oracle.pms(1, 1, masks_of([[1]], [[1]])).status == UNSAT
    # an empty negative clause: all-true and all-false both violate it
    assert oracle.pms(3, 1, masks_of([[1]], [[]])).status == UNSAT
    assert oracle.pms(3, 0, masks_of([], [[]])).status == UNSAT


def test_trivial_cases():
    # m = 0, no clauses -> SAT with the empty assignment
    r = oracle.pms(0, 0, np.zeros((0, 1), np.uint64))
    assert (r.status, r.assign, r.cost) == (SAT, 0, 0)
    # only negative clauses -> all-false (always satisfiable)
    r = oracle.pms(5, 0, masks_of([], [[1, 2], [3]]))
    assert (r.status, r.assign, r.cost) == (SAT, 0, 0)
    # only positive clauses (non-empty) -> always SAT
    r = oracle.pms(5, 2, masks_of([[1, 2], [5]], []))
    assert r.status == SAT


def test_bad_input():
    mk = masks_of([[1, 9]], [])  # b9 with m = 8
    assert oracle.pms(8, 1, mk).status == BAD
    assert oracle.mhs(8, 1, mk).status == BAD
    assert oracle.greedy(8, 1, mk)[0] == BAD
    assert oracle.pms(3, 1, masks_of([[1]], []), w=[1, 0, 2]).status == BAD


def test_nonminimal_greedy_p10():
    pos = [[1, 2, 4], [1, 2, 5], [1, 3, 6], [1, 3, 7], [2], [3]]
    st, a, picks = oracle.greedy(7, len(pos), masks_of(pos, []))
    assert picks.tolist() == [0, 1, 2]  # b1 (4 clauses), then b2, b3
    assert synth.mask_to_vars(a) == [2, 3]  # reverse-delete drops b1


def bipartite_family(n):
    """Johnson's bad family: left = n vertices; for i = 2..n, floor(n/i) right
    vertices each adjacent to i consecutive left vertices.  Right vertices get
    the low indices.  Returns (m, edges as 1-based pairs, n_left, n_right)."""
    right = []
    for i in range(n, 1, -1):
        for j in range(n // i):
            right.append(list(range(j * i, (j + 1) * i)))
    nr = len(right)
    edges = [[r + 1, nr + u + 1] for r, nb in enumerate(right) for u in nb]
    return nr + n, edges, n, nr


def max_matching(edges, m):
    """Kuhn's augmenting paths (independent of the oracle)."""
    adj = {}
    for a, b in edges:
        adj.setdefault(a, []).append(b)
    match = {}

    def aug(u, seen):
        for v in adj.get(u, []):
            if v in seen:
                continue
            seen.add(v)
            if v not in match or aug(match[v], seen):
                match[v] = u
                return True
        return False

    return sum(aug(u, set()) for u in adj)


def test_bipartite_family_p11_bound():
    m, edges, nl, nr = bipartite_family(9)
    assert (m, len(edges), nr) == (23, 60, 14)
    mk = masks_of(edges, [])
    r = oracle.mhs(m, len(edges), mk)
    assert r.cost == nl == max_matching(edges, m)  # Koenig
    st, a, picks = oracle.greedy(m, len(edges), mk)
    g = len(synth.mask_to_vars(a))
    assert g == 14
    # greedy/OPT = 14/9 > H(2) = 3/2: the "H(max clause size)" bound is false
    assert Fraction(g, r.cost) > Fraction(3, 2)
    delta = max(sum(1 for e in edges if v in e) for v in range(1, m + 1))
    assert Fraction(g) <= sum(Fraction(1, i) for i in range(1, delta + 1)) * r.cost


def test_weights_p12_p13():
    r = oracle.pms(2, 1, masks_of([[1, 2]], []), w=[100, 1])
    assert vars_of(r.assign) == [2] and r.cost == 1
    assert synth.mask_to_vars(oracle.greedy(2, 1, masks_of([[1, 2]], []))[1]) == [1]
    # P13: w = gw*gb + lw^ld with gw = 12, lw = 10
    vals = sorted({12 * gb + 10 ** ld for gb in (0, 1) for ld in (0, 1, 2)})
    assert vals == [1, 10, 13, 22, 100, 112]
    rng = np.random.default_rng(0)
    w = synth.paper_weights(rng, 1000)
    assert set(np.unique(w).tolist()) <= set(vals)


# ---------------------------------------------------- independent brute force
def py_brute(m, pos, neg, w):
    """Minimum of (weight, size, colex rank) over all assignments, with the
    clauses as Python sets -- a second, encoding-independent definition."""
    best = None
    for bits in itertools.product((0, 1), repeat=m):
        true = {i + 1 for i in range(m) if bits[i]}
        if all(set(c) & true for c in pos) and all(not set(c) <= true for c in neg):
            key = (sum(w[i - 1] for i in true), len(true), colex_rank(true))
            if best is None or key < best[0]:
                best = (key, sorted(true))
    return best


def rand_instance(rng, m, n, p_neg=0.3, wmax=0):
    pos, neg, seen = [], [], set()
    for _ in range(n):
        s = rng.randint(1, min(m, 4))
        c = tuple(sorted(rng.sample(range(1, m + 1), s)))
        isneg = rng.random() < p_neg
        if (isneg, c) in seen:
            continue
        seen.add((isneg, c))
        (neg if isneg else pos).append(list(c))
    w = [rng.randint(1, wmax) for _ in range(m)] if wmax else [1] * m
    return pos, neg, w


@pytest.mark.parametrize("seed", range(6))
def test_levelled_equals_brute_force(seed):
    rng = random.Random(1000 + seed)
    for trial in range(60):
        m = rng.randint(1, 9)
        wmax = 0 if trial % 2 == 0 else rng.choice([3, 100])
        pos, neg, w = rand_instance(rng, m, rng.randint(1, 12), wmax=wmax)
        mk = masks_of(pos, neg)
        bf = py_brute(m, pos, neg, w)
        ww = w if wmax else None
        results = [oracle.pms(m, len(pos), mk, w=ww, reduce=r) for r in (0, 1)]
        results.append(oracle.pms_brute(m, len(pos), mk, w=ww))
        for r in results:
            if bf is None:
                assert r.status == UNSAT
            else:
                assert r.status == SAT
                assert vars_of(r.assign) == bf[1]
                assert r.cost == bf[0][0]


@pytest.mark.parametrize("seed", range(3))
def test_reduce_matches_plain_larger_m(seed):
    rng = random.Random(77 + seed)
    for trial in range(25):
        m = rng.randint(10, 18)
        pos, neg, w = rand_instance(rng, m, rng.randint(3, 20), wmax=(50 if trial % 3 == 0 else 0))
        mk = masks_of(pos, neg)
        ww = w if trial % 3 == 0 else None
        a = oracle.pms(m, len(pos), mk, w=ww, reduce=0)
        b = oracle.pms(m, len(pos), mk, w=ww, reduce=1)
        c = oracle.pms_brute(m, len(pos), mk, w=ww)
        assert (a.status, a.assign, a.cost) == (b.status, b.assign, b.cost) == (c.status, c.assign, c.cost)


@pytest.mark.parametrize("seed", range(3))
def test_koenig_bipartite(seed):
    rng = random.Random(seed)
    for _ in range(20):
        nl, nr = rng.randint(1, 7), rng.randint(1, 7)
        edges = sorted({(l, nl + r) for l in range(1, nl + 1) for r in range(1, nr + 1)
                        if rng.random() < 0.35})
        if not edges:
            continue
        edges = [list(e) for e in edges]
        r = oracle.mhs(nl + nr, len(edges), masks_of(edges, []))
        assert r.cost == max_matching(edges, nl + nr)


def test_decided_closed_form_reduced():
    """With reduce = 1 and unit weights, the candidates tested are exactly
    sum_{k<k*} C(m_eff, k) + rank(x*) + 1 in the support-relabelled space."""
    rng = random.Random(5)
    for _ in range(80):
        m = rng.randint(2, 14)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 10))
        mk = masks_of(pos, neg)
        r = oracle.pms(m, len(pos), mk, reduce=1)
        if r.status != SAT:
            continue
        sup = sorted({v for c in pos for v in c})
        relabel = {v: i + 1 for i, v in enumerate(sup)}
        x = [relabel[v] for v in vars_of(r.assign)]
        k = len(x)
        assert r.decided == sum(math.comb(len(sup), j) for j in range(k)) + colex_rank(x) + 1


# ------------------------------------------------------------- greedy invariants
def check_greedy_invariants(m, pos, neg, status, chosen, picks):
    S = set(chosen)
    assert all(set(c) & S for c in pos)  # a hitting set of phi+ 
    for x in S:  # minimal: every element has a private clause
        assert any(set(c) & S == {x} for c in pos)
    # pick order: newly covered counts are non-increasing (greedy takes the max)
    unc = [set(c) for c in pos]
    gains = []
    for v in picks:
        gains.append(sum(1 for c in unc if v + 1 in c))
        unc = [c for c in unc if v + 1 not in c]
    assert not unc
    assert all(g > 0 for g in gains)
    assert all(a >= b for a, b in zip(gains, gains[1:]))
    assert set(chosen) <= {v + 1 for v in picks}
    viol = any(set(c) <= S for c in neg)
    assert status == (NEGV if viol else SAT)


@pytest.mark.parametrize("seed", range(4))
def test_greedy_properties_and_bound(seed):
    rng = random.Random(300 + seed)
    for _ in range(60):
        m = rng.randint(2, 12)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 16))
        if not pos:
            continue
        mk = masks_of(pos, neg)
        st, a, picks = oracle.greedy(m, len(pos), mk)
        chosen = synth.mask_to_vars(a)
        check_greedy_invariants(m, pos, neg, st, chosen, picks.tolist())
        opt = py_brute(m, pos, [], [1] * m)[0][1]
        assert oracle.mhs(m, len(pos), mk).cost == opt
        delta = max(sum(1 for c in pos if v in c) for v in range(1, m + 1))
        H = sum(Fraction(1, i) for i in range(1, delta + 1))
        assert opt <= len(chosen) <= H * opt
        # unit PMS relations (P14): |MHS| <= |PMS|; MHS feasible for phi- => PMS == MHS
        r = oracle.pms(m, len(pos), mk)
        rm = oracle.mhs(m, len(pos), mk)
        if r.status == SAT:
            assert rm.cost <= r.cost
        if rm.status == SAT:
            assert (r.status, r.assign) == (SAT, rm.assign)


def test_greedy_csr_equals_masks():
    rng = random.Random(9)
    for _ in range(30):
        m = rng.randint(2, 12)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 14))
        st, a, picks = oracle.greedy(m, len(pos), masks_of(pos, neg))
        po = np.cumsum([0] + [len(c) for c in pos])
        no = np.cumsum([0] + [len(c) for c in neg])
        pv = [v - 1 for c in pos for v in c]
        nv = [v - 1 for c in neg for v in c]
        g = oracle.greedy_csr(m, po, np.array(pv, np.int32), no, np.array(nv, np.int32))
        assert g.status == st
        assert g.picks.tolist() == picks.tolist()
        assert [i + 1 for i in np.nonzero(g.in_S)[0]] == synth.mask_to_vars(a)


def test_invariance_reorder_relabel():
    rng = random.Random(11)
    for _ in range(40):
        m = rng.randint(2, 10)
        pos, neg, w = rand_instance(rng, m, rng.randint(1, 12), wmax=20)
        r0 = oracle.pms(m, len(pos), masks_of(pos, neg), w=w)
        pos2, neg2 = pos[::-1], neg[::-1]
        r1 = oracle.pms(m, len(pos), masks_of(pos2, neg2), w=w)
        assert (r0.status, r0.assign, r0.cost) == (r1.status, r1.assign, r1.cost)
        # insert an unused variable at position 1 (order-preserving relabel)
        sh = lambda cs: [[v + 1 for v in c] for c in cs]
        r2 = oracle.pms(m + 1, len(pos), masks_of(sh(pos), sh(neg)), w=[1] + w)
        assert r2.status == r0.status
        if r0.status == SAT:
            assert vars_of(r2.assign) == [v + 1 for v in vars_of(r0.assign)]


# ------------------------------------------------------------ P15 (C3 shape)
def test_p15_product_reasoning_small():
    """P15 on a shrunken C3: G disjoint groups -> the canonical optimum is the
    min feasible one-per-group set; checked against the levelled oracle."""
    for seed in range(5):
        cb, H, grp = synth.c3_instance(seed=seed, m=15, groups=5, n_rand_pos=12, n_neg=8)
        m, npos, mk, _ = cb.instance(0)
        r = oracle.pms(m, npos, mk)
        n, best = oracle.min_feasible_product(grp, npos, mk)
        assert n >= 1 and r.status == SAT and r.cost == 5 and r.assign == best


def test_c3_structure():
    cb, H, grp = synth.c3_instance()
    m, npos, mk, _ = cb.instance(0)
    assert (m, npos, mk.shape[0]) == (48, 140, 200)
    gm = [sum(1 << v for v in g) for g in grp]
    assert all(a & b == 0 for a, b in itertools.combinations(gm, 2))
    assert all(int(x) in {int(v) for v in mk[:npos, 0]} for x in gm)  # group clauses present
    hm = sum(1 << v for v in H)
    assert oracle.feasible(hm, npos, mk)


# ------------------------------------------------------- composite Solve (f1)
def test_composite_solve_paper_fallback():
    """PAPER.md:26 / SPEC.md:411 (acceptance #6): the mhs strategy on the paper's
    example triggers the MaxSAT fallback and returns 3 true variables."""
    g = load_golden("paper_example.txt")
    cb = synth.batch_from_lists([(g["m"], g["pos"], g["neg"])], W=1)
    r = oracle.batch("solve", cb)
    assert r.decided[0] == 1  # fell back
    assert (r.status[0], r.cost[0]) == (SAT, 3)
    assert synth.mask_to_vars(r.assign[0]) == [2, 3, 4]


def test_composite_solve_properties():
    """Fallback completeness: Solve is UNSAT iff PMS is UNSAT;
    without fallback the answer is the greedy set, with it the PMS optimum."""
    rng = random.Random(21)
    insts = []
    for _ in range(200):
        m = rng.randint(1, 10)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 12))
        insts.append((m, pos, neg))
    cb = synth.batch_from_lists(insts, W=1)
    s, p, g = oracle.batch("solve", cb), oracle.batch("pms", cb), oracle.batch("greedy", cb)
    assert ((s.status == UNSAT) == (p.status == UNSAT)).all()
    fb = s.decided == 1
    assert (fb == (g.status == NEGV)).all()
    assert (s.assign[fb] == p.assign[fb]).all() and (s.assign[~fb] == g.assign[~fb]).all()
    assert (s.status != NEGV).all()


# ------------------------------------------------------- incremental Solve (f2)
def test_incremental_kstart_monotone():
    """phi := phi U {c}.  A feasible set of phi U {c} is feasible
    for phi, so no feasible set lies below phi's optimum level: enumerating
    from k* gives exactly the full answer with fewer candidates."""
    rng = random.Random(31)
    for _ in range(150):
        m = rng.randint(2, 12)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 10))
        r0 = oracle.pms(m, len(pos), masks_of(pos, neg))
        if r0.status != SAT:
            continue
        c = sorted(rng.sample(range(1, m + 1), rng.randint(1, min(3, m))))
        if rng.random() < 0.5:
            pos2, neg2 = pos + [c], neg
        else:
            pos2, neg2 = pos, neg + [c]
        full = oracle.pms(m, len(pos2), masks_of(pos2, neg2))
        inc = oracle.pms_kstart(m, len(pos2), masks_of(pos2, neg2), r0.cost)
        assert (inc.status, inc.assign, inc.cost) == (full.status, full.assign, full.cost)
        assert inc.decided <= full.decided
        assert full.cost >= r0.cost or full.status == UNSAT  # the optimum never decreases


# ------------------------------------------------------- weighted mhs (f4)
def test_weighted_greedy_pins():
    # phi+ = {b1 v b2}, w(b1) = 100, w(b2) = 1 -> only b2 true
    st, a, picks = oracle.greedy(2, 1, masks_of([[1, 2]], []), w=[100, 1])
    assert synth.mask_to_vars(a) == [2] and picks.tolist() == [1]
    # unit (or constant) weights reduce to the unweighted greedy
    rng = random.Random(41)
    for _ in range(60):
        m = rng.randint(2, 12)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 14))
        mk = masks_of(pos, neg)
        ref = oracle.greedy(m, len(pos), mk)
        for c in (1, 7):
            got = oracle.greedy(m, len(pos), mk, w=[c] * m)
            assert got[0] == ref[0] and (got[1] == ref[1]).all() and (got[2] == ref[2]).all()


def test_weighted_greedy_chvatal_bound_and_scaling():
    """Chvatal 1979: the ratio greedy costs at most H(Delta+) x the weighted
    optimum (here: WPMS over phi+ alone); scaling all weights changes nothing."""
    rng = random.Random(43)
    for _ in range(120):
        m = rng.randint(2, 10)
        pos, _, _ = rand_instance(rng, m, rng.randint(1, 12), p_neg=0.0)
        if not pos:
            continue
        w = [rng.randint(1, 30) for _ in range(m)]
        mk = masks_of(pos, [])
        st, a, picks = oracle.greedy(m, len(pos), mk, w=w)
        chosen = synth.mask_to_vars(a)
        check_greedy_invariants_weighted(pos, chosen)
        cost = sum(w[v - 1] for v in chosen)
        opt = oracle.pms(m, len(pos), mk, w=w).cost
        delta = max(sum(1 for c in pos if v in c) for v in range(1, m + 1))
        assert opt <= cost <= sum(Fraction(1, i) for i in range(1, delta + 1)) * opt
        st3, a3, p3 = oracle.greedy(m, len(pos), mk, w=[3 * x for x in w])
        assert (a3 == a).all() and p3.tolist() == picks.tolist()


def check_greedy_invariants_weighted(pos, chosen):
    S = set(chosen)
    assert all(set(c) & S for c in pos)
    for x in S:
        assert any(set(c) & S == {x} for c in pos)


def test_weighted_prune_order_golden():
    """tests/golden/weighted_prune_order.txt: with weights the reverse-delete
    runs in descending-weight order (reading R12), which here
    keeps {b2, b3} (weight 101) where reverse pick order would keep {b1, b3}."""
    g = load_golden("weighted_prune_order.txt")
    m, pos, w, e = g["m"], g["pos"], g["w"], g["expect"]
    mk = masks_of(pos, [])
    st, a, picks = oracle.greedy(m, len(pos), mk, w=w)
    assert [int(p) + 1 for p in picks] == [int(x) for x in e["picks"]]
    assert synth.mask_to_vars(a) == [int(x) for x in e["greedy"]]
    assert sum(w[v - 1] for v in synth.mask_to_vars(a)) == int(e["greedy_cost"][0])
    assert st == STATUS[e["greedy_status"][0]]
    # the CSR entry point agrees
    off = np.cumsum([0] + [len(c) for c in pos]).astype(np.int64)
    var = np.asarray([v - 1 for c in pos for v in c], np.int32)
    g2 = oracle.greedy_csr(m, off, var, np.zeros(1, np.int64), np.zeros(0, np.int32), w=w)
    assert [i + 1 for i in np.flatnonzero(g2.in_S)] == [int(x) for x in e["greedy"]]


def py_weighted_prune(pos, picks, w):
    """Reverse-delete written out over Python sets: descending weight, equal
    weights in reverse pick order (reading R12)."""
    order = sorted(range(len(picks)), key=lambda i: (-w[picks[i] - 1], -i))
    S = set(picks)
    for i in order:
        x = picks[i]
        if all(set(c) & (S - {x}) for c in pos):
            S.discard(x)
    return sorted(S)


def test_weighted_prune_order_random():
    rng = random.Random(4242)
    for _ in range(200):
        m = rng.randint(2, 10)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 14))
        w = [rng.choice([1, 2, 3, 10, 100]) for _ in range(m)]
        st, a, picks = oracle.greedy(m, len(pos), masks_of(pos, neg), w=w)
        if st not in (SAT, NEGV):
            continue
        assert synth.mask_to_vars(a) == py_weighted_prune(pos, [int(p) + 1 for p in picks], w)


# ------------------------------------------------- two-word masks (W = 2)
# Variables above b_64 live in word 1; the oracle then relabels the support of
# phi+ across both words (compress(word0) | compress(word1) << popc(sup0)) and
# expands the optimum back.  These pins fix that branch by closed forms and an
# independent Python-sets brute force over the variables that occur.
def py_brute_support(pos, neg, w=None):
    """min (weight, size, colex rank) over subsets of the variables that occur
    in some clause (a variable in no clause is false in every optimum: it only
    adds weight >= 1), clauses as Python sets, original 1-based indices."""
    V = sorted({v for c in pos + neg for v in c})
    best = None
    for bits in itertools.product((0, 1), repeat=len(V)):
        true = {V[i] for i in range(len(V)) if bits[i]}
        if all(set(c) & true for c in pos) and all(not set(c) <= true for c in neg):
            key = (sum((w[i - 1] if w else 1) for i in true), len(true), colex_rank(true))
            if best is None or key < best[0]:
                best = (key, sorted(true))
    return best


@pytest.mark.parametrize("sizes,start", [([2, 3, 4], 60), ([1, 5, 2, 7], 58), ([3] * 8, 50),
                                         ([4, 4], 63), ([9, 1, 1], 100)])
def test_w2_disjoint_clauses(sizes, start):
    """P5 across the word boundary: MHS = PMS = the lowest variable of each
    disjoint clause; the greedy returns the same set; decided closed form."""
    pos, v = [], start
    for s in sizes:
        pos.append(list(range(v, v + s)))
        v += s
    m = 128
    mk = masks_of(pos, [], W=2)
    want = [c[0] for c in pos]
    for r in (oracle.mhs(m, len(pos), mk, W=2), oracle.pms(m, len(pos), mk, W=2)):
        assert r.status == SAT and vars_of(r.assign) == want and r.cost == len(pos)
        # relabelled: support = the clauses' variables in order; x* = the first
        # of each group; decided = sum_{k<K} C(m_eff, k) + rank + 1
        sup = sorted(v for c in pos for v in c)
        x = [sup.index(c[0]) + 1 for c in pos]
        K = len(pos)
        assert r.decided == sum(math.comb(len(sup), j) for j in range(K)) + colex_rank(x) + 1
    st, a, _ = oracle.greedy(m, len(pos), mk, W=2)
    assert st == SAT and synth.mask_to_vars(a) == want


@pytest.mark.parametrize("lo,n", [(60, 8), (55, 15), (64, 5), (65, 9), (40, 30)])
def test_w2_path(lo, n):
    """P6 across the word boundary: a path b_lo - ... - b_{lo+n-1} has minimum
    vertex cover floor(n/2); canonical (smallest colex rank) = odd positions for
    odd n ({lo+1, lo+3, ...}), and for even n the colex-smallest cover."""
    pos = [[i, i + 1] for i in range(lo, lo + n - 1)]
    mk = masks_of(pos, [], W=2)
    r = oracle.mhs(128, len(pos), mk, W=2)
    assert r.cost == n // 2
    if n % 2 == 1:
        assert vars_of(r.assign) == list(range(lo + 1, lo + n - 1, 2))
    if n <= 15:
        bf = py_brute_support(pos, [])
        assert vars_of(r.assign) == bf[1]


def test_w2_mixed_brute_force():
    """reduce = 1 on two-word instances with support <= 12 spread over both
    words, unit and weighted, against the Python-sets brute force; plus the
    MHS and its phi- flag."""
    rng = random.Random(2022)
    n_sat = 0
    for trial in range(150):
        nv = rng.randint(2, 12)
        vars_ = sorted(rng.sample(range(1, 129), nv))
        if not any(v > 64 for v in vars_) or not any(v <= 64 for v in vars_):
            vars_[0], vars_[-1] = rng.randint(1, 64), rng.randint(65, 128)
            vars_ = sorted(set(vars_))
        pos, neg, seen = [], [], set()
        for _ in range(rng.randint(1, 10)):
            c = tuple(sorted(rng.sample(vars_, rng.randint(1, min(4, len(vars_))))))
            isneg = rng.random() < 0.3
            if (isneg, c) in seen:
                continue
            seen.add((isneg, c))
            (neg if isneg else pos).append(list(c))
        w = [rng.randint(1, 100) for _ in range(128)] if trial % 2 else None
        mk = masks_of(pos, neg, W=2)
        r = oracle.pms(128, len(pos), mk, w=w, reduce=1, W=2)
        # the brute force over the occurring variables; negatives touching a
        # variable outside phi+'s support are satisfied by keeping it false
        bf = py_brute_support(pos, neg, w)
        if bf is None:
            assert r.status == UNSAT
            continue
        n_sat += 1
        assert r.status == SAT and vars_of(r.assign) == bf[1] and r.cost == bf[0][0]
        h = oracle.mhs(128, len(pos), mk, W=2)
        bh = py_brute_support(pos, [])
        assert vars_of(h.assign) == bh[1]
        viol = any(set(c) <= set(bh[1]) for c in neg)
        assert h.status == (NEGV if viol else SAT)
    assert n_sat > 60


def test_w2_greedy_relabel_invariance():
    """The greedy over an instance shifted into word 1 (b_i -> b_{i+s}) picks
    the shifted variables in the same order (ties: the shift preserves the
    index order)."""
    rng = random.Random(7)
    for _ in range(60):
        m = rng.randint(2, 12)
        pos, neg, _ = rand_instance(rng, m, rng.randint(1, 14))
        st, a, picks = oracle.greedy(m, len(pos), masks_of(pos, neg))
        for s in (50, 64, 100):
            sp = [[v + s for v in c] for c in pos]
            sn = [[v + s for v in c] for c in neg]
            st2, a2, p2 = oracle.greedy(128, len(pos), masks_of(sp, sn, W=2), W=2)
            assert st2 == st and p2.tolist() == [p + s for p in picks.tolist()]
            assert synth.mask_to_vars(a2) == [v + s for v in synth.mask_to_vars(a)]


def test_kmax_after_subsumption_r13():
    """Reading R13: with reduce = 1 the levels stop at k_max = min(|support|,
    #positive clauses no other clause subsumes).  Nested clauses {b1} c {b1,b2}
    c {b1,b2,b3} leave one minimal clause, so with not-b1 the UNSAT proof
    enumerates levels 0 and 1 only: 1 + C(3,1) = 4 candidates (the raw clause
    count would give 1 + 3 + 3 + 1 = 8); duplicates count once."""
    pos, neg = [[1], [1, 2], [1, 2, 3]], [[1]]
    r = oracle.pms(3, 3, masks_of(pos, neg), reduce=1)
    assert r.status == UNSAT and r.decided == 1 + 3
    assert oracle.pms(3, 3, masks_of(pos, neg), reduce=0).decided == 8
    assert py_brute(3, pos, neg, [1] * 3) is None
    # two disjoint minimal clauses and a superset: k_max = 2
    pos, neg = [[1, 2], [3, 4], [1, 2, 3]], [[1], [2], [3], [4]]
    r = oracle.pms(4, 3, masks_of(pos, neg), reduce=1)
    assert r.status == UNSAT and r.decided == sum(math.comb(4, k) for k in range(3))
    # a duplicated clause counts once (masks_of keeps both copies)
    pos = [[1, 2], [1, 2]]
    r = oracle.pms(2, 2, masks_of(pos, [[1], [2]]), reduce=1)
    assert r.status == UNSAT and r.decided == 1 + 2
