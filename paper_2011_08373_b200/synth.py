"""Seeded synthetic clause sets shaped like GPURepair's Solve-step workloads.

This module is the ONLY code shared by the CUDA path and the CPU oracle.  It
draws random clause sets and packs clause variable lists into bit masks; it
contains none of the method's arithmetic (no feasibility test, no
enumeration, no greedy step, no cost).  Everything the method computes lives
on one side in ``paper_2011_08373_b200/csrc`` (CUDA) and, independently, in
``oracle/`` (plain C).

Vocabulary follows PAPER.md:3-15 (Se:preliminaries): barrier variables
b_1..b_m, positive monotone clauses phi+ (one per data-race trace,
PAPER.md:24) and negative monotone clauses phi- (one per barrier-divergence
trace).  Encoding (reading R1): b_i <-> bit (i-1), b_1 = LSB of word
0; a clause is ``W`` little-endian uint64 words; polarity is positional: the
first ``n_pos[b]`` clauses of instance b are positive, the rest negative.

Workload recipes are SURVEY.md §8(d) C1..C5 (seed = 2011083730 + cfg); the
m-distribution of C2 is the instrumented-barrier histogram of PAPER.md:593-602
(Fi:kernels_barriers); the batch size 748 is PAPER.md:194.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

SEED_BASE = 2011083730


def seed_for(cfg: int, rank: int = 0) -> int:
    """Seed of config ``cfg`` (1..5); ``rank`` > 0 gives an independent batch per GPU."""
    return SEED_BASE + cfg + 1000 * rank


# --------------------------------------------------------------------------
# containers
# --------------------------------------------------------------------------
@dataclass
class ClauseBatch:
    """A batch of independent Solve-step instances (host numpy arrays).

    m      int32  [B]          number of barrier variables of each instance
    off    int64  [B+1]        instance b owns clauses off[b] .. off[b+1]-1
    n_pos  int32  [B]          the first n_pos[b] of them are positive (phi+)
    masks  uint64 [off[B], W]  bit (i-1) of the clause <-> literal on b_i
    w      uint32 [B, wstride] weight of soft clause (not b_i), or None = unit
    """

    m: np.ndarray
    off: np.ndarray
    n_pos: np.ndarray
    masks: np.ndarray
    w: Optional[np.ndarray] = None

    @property
    def B(self) -> int:
        return int(self.m.shape[0])

    @property
    def W(self) -> int:
        return int(self.masks.shape[1])

    def instance(self, b: int) -> Tuple[int, int, np.ndarray, Optional[np.ndarray]]:
        """(m, n_pos, masks[n, W], w[m] or None) of instance b."""
        lo, hi = int(self.off[b]), int(self.off[b + 1])
        w = None if self.w is None else self.w[b, : int(self.m[b])]
        return int(self.m[b]), int(self.n_pos[b]), self.masks[lo:hi], w

    def subset(self, idx: Sequence[int]) -> "ClauseBatch":
        idx = list(idx)
        ms, offs, nps, parts, ws = [], [0], [], [], []
        for b in idx:
            m, npos, mk, w = self.instance(b)
            ms.append(m)
            nps.append(npos)
            parts.append(mk)
            offs.append(offs[-1] + mk.shape[0])
            if self.w is not None:
                ws.append(self.w[b])
        masks = np.concatenate(parts, 0) if parts else np.zeros((0, self.W), np.uint64)
        return ClauseBatch(
            m=np.asarray(ms, np.int32),
            off=np.asarray(offs, np.int64),
            n_pos=np.asarray(nps, np.int32),
            masks=np.ascontiguousarray(masks.reshape(-1, self.W), dtype=np.uint64),
            w=None if self.w is None else np.ascontiguousarray(np.stack(ws), dtype=np.uint32),
        )


@dataclass
class CSRClauses:
    """Clauses of ONE big instance as variable lists (0-based var ids = i-1).

    Used for the greedy-at-scale workload (C5), whose bit matrix is packed on
    the device.  ``pos_off``/``pos_var`` hold phi+, ``neg_off``/``neg_var`` phi-.
    """

    m: int
    pos_off: np.ndarray  # int64 [n_pos+1]
    pos_var: np.ndarray  # int16/int32 [nnz]
    neg_off: np.ndarray  # int64 [n_neg+1]
    neg_var: np.ndarray  # int32 [nnz_neg]

    @property
    def n_pos(self) -> int:
        return int(self.pos_off.shape[0] - 1)

    @property
    def n_neg(self) -> int:
        return int(self.neg_off.shape[0] - 1)


# --------------------------------------------------------------------------
# packing helpers (pure data layout, no method arithmetic)
# --------------------------------------------------------------------------
def words_for(m: int) -> int:
    return max(1, (m + 63) // 64)


def pack_vars(vars0: Sequence[int], W: int) -> np.ndarray:
    """0-based variable ids -> W little-endian uint64 words."""
    out = np.zeros(W, np.uint64)
    for v in vars0:
        out[v // 64] |= np.uint64(1) << np.uint64(v % 64)
    return out


def batch_from_lists(
    instances: Sequence[Tuple[int, Sequence[Sequence[int]], Sequence[Sequence[int]]]],
    weights: Optional[Sequence[Sequence[int]]] = None,
    W: Optional[int] = None,
) -> ClauseBatch:
    """Build a batch from (m, positive clauses, negative clauses) triples.

    Clauses are given as lists of 1-based barrier-variable ids (b_i -> i), the
    paper's notation.
    """
    if W is None:
        W = max([words_for(m) for m, _, _ in instances] + [1])
    ms, offs, nps, rows = [], [0], [], []
    for m, pos, neg in instances:
        ms.append(m)
        nps.append(len(pos))
        for c in list(pos) + list(neg):
            rows.append(pack_vars([i - 1 for i in c], W))
        offs.append(offs[-1] + len(pos) + len(neg))
    masks = np.stack(rows) if rows else np.zeros((0, W), np.uint64)
    w = None
    if weights is not None:
        ws = max([len(x) for x in weights] + [1])
        w = np.ones((len(instances), ws), np.uint32)
        for b, x in enumerate(weights):
            w[b, : len(x)] = np.asarray(x, np.uint32)
    return ClauseBatch(
        m=np.asarray(ms, np.int32),
        off=np.asarray(offs, np.int64),
        n_pos=np.asarray(nps, np.int32),
        masks=np.ascontiguousarray(masks, dtype=np.uint64),
        w=w,
    )


def mask_to_vars(words: np.ndarray) -> List[int]:
    """W uint64 words -> sorted 1-based barrier ids (b_i)."""
    out = []
    for wi, x in enumerate(np.asarray(words, np.uint64).reshape(-1)):
        x = int(x)
        while x:
            low = x & -x
            out.append(64 * wi + low.bit_length())
            x ^= low
    return out


# --------------------------------------------------------------------------
# C1: the paper's worked example embedded in m = 8
# --------------------------------------------------------------------------
PAPER_EXAMPLE_POS = [[1, 3], [1, 4], [2, 5], [2, 6]]
PAPER_EXAMPLE_NEG = [[1, 2]]  # PAPER.md:26, (not b1 or not b2)


def c1_instances() -> ClauseBatch:
    """instance A (P2) and instance B (P3), m = 8, 6 clauses each."""
    a = (8, PAPER_EXAMPLE_POS, [[1, 2], [7, 8]])
    b = (8, PAPER_EXAMPLE_POS, [[1, 2], [3, 4]])
    return batch_from_lists([a, b], W=1)


# --------------------------------------------------------------------------
# C2: suite-shaped batch (748 kernels; m per PAPER.md:593-602)
# --------------------------------------------------------------------------
# (lo, hi, count) buckets of Fi:kernels_barriers; the top two are clamped to
# the config's m <= 32.
M_HISTOGRAM = [
    (0, 0, 203), (1, 1, 59), (2, 2, 95), (3, 3, 50), (4, 5, 92),
    (6, 10, 110), (11, 20, 61), (21, 32, 59), (32, 32, 5),
]


def _draw_m(rng: np.random.Generator, B: int, hist=M_HISTOGRAM) -> np.ndarray:
    counts = np.array([c for _, _, c in hist], np.float64)
    bucket = rng.choice(len(hist), size=B, p=counts / counts.sum())
    lo = np.array([h[0] for h in hist])[bucket]
    hi = np.array([h[1] for h in hist])[bucket]
    return (lo + (rng.random(B) * (hi - lo + 1)).astype(np.int64)).astype(np.int32)


def _pos_clause(rng, m: int, min_size: int = 1) -> List[int]:
    """70 % contiguous interval (barriers disabled along a trace), 30 % subset."""
    if rng.random() < 0.7:
        # 1 + Geom(0.5) on {0,1,..} == numpy's geometric on {1,2,..}
        length = int(rng.geometric(0.5))
        length = min(max(length, min_size), min(m, 6))
        start = int(rng.integers(0, m - length + 1))
        return list(range(start, start + length))
    size = int(rng.integers((m + 3) // 4, m + 1))
    size = max(size, min(min_size, m), 1)
    return sorted(rng.choice(m, size=size, replace=False).tolist())


def _neg_clause(rng, m: int) -> List[int]:
    size = int(rng.choice([1, 2, 3], p=[0.3, 0.5, 0.2]))
    size = min(size, m)
    return sorted(rng.choice(m, size=size, replace=False).tolist())


def c2_batch(seed: Optional[int] = None, B: int = 748, m_max: int = 32) -> ClauseBatch:
    """B suite-shaped instances, m <= 32, <= 64 clauses, 25 % negative."""
    rng = np.random.default_rng(seed_for(2) if seed is None else seed)
    ms = np.minimum(_draw_m(rng, B), m_max)
    insts = []
    for m in ms.tolist():
        if m == 0:
            insts.append((0, [], []))
            continue
        n = int(rng.integers(1, min(64, 2 * m) + 1))
        pos, neg, seen = [], [], set()
        tries = 0
        while len(pos) + len(neg) < n and tries < 20 * n:
            tries += 1
            if rng.random() < 0.25:
                c, key = _neg_clause(rng, m), "n"
            else:
                c, key = _pos_clause(rng, m), "p"
            t = (key, tuple(c))
            if t in seen:
                continue
            seen.add(t)
            (neg if key == "n" else pos).append([v + 1 for v in c])
        insts.append((m, pos, neg))
    return batch_from_lists(insts, W=1)


# --------------------------------------------------------------------------
# C3: single hard instance, m = 48, 200 clauses, certified k* = 16
# --------------------------------------------------------------------------
def c3_instance(seed: Optional[int] = None, m: int = 48, groups: int = 16,
                n_rand_pos: int = 124, n_neg: int = 60):
    """SURVEY §8(d) C3.  Returns (batch of 1, planted H* as 0-based ids, groups).

    A seeded permutation maps the m vars into ``groups`` disjoint groups of
    m/groups -> one positive clause per group (so k* >= groups); planted H* =
    one var per group; every random positive clause meets H*, every negative
    clause has a var outside H* (so H* is feasible and k* = groups).
    """
    rng = np.random.default_rng(seed_for(3) if seed is None else seed)
    perm = rng.permutation(m)
    gsz = m // groups
    grp = [sorted(perm[g * gsz:(g + 1) * gsz].tolist()) for g in range(groups)]
    H = sorted(int(rng.choice(g)) for g in grp)
    Hs = set(H)
    seen = set(tuple(g) for g in grp)
    pos = [list(g) for g in grp]
    while len(pos) < groups + n_rand_pos:
        s = int(rng.integers(2, 5))
        c = tuple(sorted(rng.choice(m, size=s, replace=False).tolist()))
        if not (set(c) & Hs) or c in seen:
            continue
        seen.add(c)
        pos.append(list(c))
    neg, nseen = [], set()
    while len(neg) < n_neg:
        s = int(rng.integers(2, 4))
        c = tuple(sorted(rng.choice(m, size=s, replace=False).tolist()))
        if set(c) <= Hs or c in nseen:
            continue
        nseen.add(c)
        neg.append(list(c))
    order = rng.permutation(len(pos))
    pos = [pos[i] for i in order]
    inst = (m, [[v + 1 for v in c] for c in pos], [[v + 1 for v in c] for c in neg])
    return batch_from_lists([inst], W=1), H, grp


# --------------------------------------------------------------------------
# C4: weighted batch, m = 40, 10k instances, planted SAT
# --------------------------------------------------------------------------
def c4_batch(seed: Optional[int] = None, B: int = 10000, m: int = 40,
             wlo: int = 50, whi: int = 100, hlo: int = 4, hhi: int = 8) -> ClauseBatch:
    """n ~ U{16..64}, 25 % negative, planted H with |H| ~ U{4..8}.

    Every positive clause meets H and has >= 2 vars; every negative clause has
    a var outside H; weights w_j ~ U{wlo..whi} (soft clause not b_j).
    """
    rng = np.random.default_rng(seed_for(4) if seed is None else seed)
    insts, weights = [], []
    for _ in range(B):
        n = int(rng.integers(16, 65))
        hs = int(rng.integers(hlo, hhi + 1))
        H = set(rng.choice(m, size=hs, replace=False).tolist())
        pos, neg, seen = [], [], set()
        while len(pos) + len(neg) < n:
            if rng.random() < 0.25:
                c = _neg_clause(rng, m)
                if len(c) < 1 or set(c) <= H:
                    continue
                t = ("n", tuple(c))
            else:
                c = _pos_clause(rng, m, min_size=2)
                if not (set(c) & H):
                    continue
                t = ("p", tuple(c))
            if t in seen:
                continue
            seen.add(t)
            (neg if t[0] == "n" else pos).append([v + 1 for v in c])
        insts.append((m, pos, neg))
        weights.append(rng.integers(wlo, whi + 1, size=m).tolist())
    return batch_from_lists(insts, weights=weights, W=1)


def paper_weights(rng: np.random.Generator, m: int, gw: int = 12, lw: int = 10,
                  p_grid: float = 0.3, ld_p=(0.6, 0.3, 0.1)) -> np.ndarray:
    """Barrier weights w = gw*gb + lw**ld (defaults gw=12, lw=10).

    gb ~ Bern(p_grid) (grid-level barrier), ld ~ {0,1,2} (loop depth).
    """
    gb = (rng.random(m) < p_grid).astype(np.int64)
    ld = rng.choice(len(ld_p), size=m, p=np.asarray(ld_p) / np.sum(ld_p))
    return (gw * gb + lw ** ld).astype(np.uint32)


# --------------------------------------------------------------------------
# C5: greedy at scale, m = 4096, n = 2^24 positive clauses
# --------------------------------------------------------------------------
def c5_clauses(seed: Optional[int] = None, m: int = 4096, n: int = 1 << 24,
               n_planted: int = 256, smin: int = 3, smax: int = 16, n_neg: int = 64):
    """SURVEY §8(d) C5.  Returns (CSRClauses, planted H as sorted 0-based ids).

    Clause = 1 var from the planted set H + (s-1) distinct random vars,
    s ~ U{smin..smax}; clauses are distinct (duplicates redrawn); phi- = n_neg
    random negative pairs.  Vectorised: rows are drawn as a padded [n, smax]
    int32 matrix with -1 padding.
    """
    rng = np.random.default_rng(seed_for(5) if seed is None else seed)
    H = np.sort(rng.choice(m, size=n_planted, replace=False)).astype(np.int32)
    sizes = rng.integers(smin, smax + 1, size=n).astype(np.int32)
    rows = np.full((n, smax), -1, np.int32)

    def draw(idx: np.ndarray):
        k = idx.shape[0]
        r = rng.integers(0, m, size=(k, smax)).astype(np.int32)
        r[:, 0] = H[rng.integers(0, n_planted, size=k)]
        col = np.arange(smax)[None, :]
        r[col >= sizes[idx][:, None]] = -1
        rows[idx] = r

    def bad_rows(idx: np.ndarray) -> np.ndarray:
        s = np.sort(rows[idx], axis=1)
        dup = (s[:, 1:] == s[:, :-1]) & (s[:, 1:] >= 0)
        return idx[dup.any(axis=1)]

    todo = np.arange(n)
    while todo.size:
        draw(todo)
        todo = bad_rows(todo)
    rows.sort(axis=1)  # -1 padding first, vars ascending
    # distinct clauses: hash the sorted rows, redraw duplicates
    while True:
        h = np.zeros(n, np.uint64)
        for j in range(smax):
            h = h * np.uint64(1000003) + (rows[:, j].astype(np.int64) + 1).astype(np.uint64)
        order = np.argsort(h, kind="stable")
        hs = h[order]
        same = np.nonzero(hs[1:] == hs[:-1])[0]
        if same.size == 0:
            break
        cand = order[same + 1]
        # confirm real duplicates (not just hash collisions)
        real = np.all(rows[order[same]] == rows[cand], axis=1)
        dupi = np.unique(cand[real])
        if dupi.size == 0:
            break
        todo = dupi
        while todo.size:
            draw(todo)
            todo = bad_rows(todo)
        rows[dupi] = np.sort(rows[dupi], axis=1)
    valid = rows >= 0
    cnt = valid.sum(axis=1)
    pos_off = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=pos_off[1:])
    pos_var = rows[valid].astype(np.int16 if m <= 32767 else np.int32)
    neg = np.array([np.sort(rng.choice(m, size=2, replace=False)) for _ in range(n_neg)],
                   np.int32).reshape(-1)
    neg_off = np.arange(0, 2 * n_neg + 1, 2, dtype=np.int64)
    return CSRClauses(m=m, pos_off=pos_off, pos_var=pos_var, neg_off=neg_off,
                      neg_var=neg), H
