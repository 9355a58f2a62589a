"""Host logic of the multi-GPU drivers on CPU: world_size-2 gloo process
groups run the real driver loop (run_levels_sharded) with its real
all-reduce; the per-shard level work is a CPU stand-in of the device call
(this tests the driver, not the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_08373_b200.multigpu import run_levels_sharded, shard_instances, estimate_costs
from gr_testutil import load_golden

NONE = 2**63 - 1


class FakeSession:
    """Instances given as {level: sorted feasible ranks} plus level sizes;
    level(k, shard, G) mimics the chunk interleave of gr_exact_level."""

    def __init__(self, inst, chunk=3):
        self.inst, self.chunk = inst, chunk
        self.B = len(inst)
        self.keys = torch.full((self.B,), NONE, dtype=torch.int64)
        self.active = list(range(self.B))
        self.result = [None] * self.B
        self.enumerated = [0] * self.B

    def prepare(self):
        return len(self.active)

    def level(self, k, shard, nshard):
        for b in self.active:
            size, feas = self.inst[b]["size"][k], self.inst[b]["feas"].get(k, [])
            nch = (size + self.chunk - 1) // self.chunk
            for c in range(shard, nch, nshard):
                lo, hi = c * self.chunk, min((c + 1) * self.chunk, size)
                self.enumerated[b] += hi - lo
                hit = [r for r in feas if lo <= r < hi]
                if hit:
                    self.keys[b] = min(int(self.keys[b]), hit[0])

    def level_keys(self):
        return self.keys

    def finish(self, k):
        nxt = []
        for b in self.active:
            if int(self.keys[b]) != NONE:
                self.result[b] = (k, int(self.keys[b]))
            elif k >= self.inst[b]["kmax"]:
                self.result[b] = ("UNSAT",)
            else:
                nxt.append(b)
        self.active = nxt
        self.keys.fill_(NONE)
        return len(nxt)


def make_instances(seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(6):
        kmax = int(rng.integers(1, 6))
        size = {k: int(rng.integers(1, 40)) for k in range(1, kmax + 1)}
        feas = {}
        if rng.random() < 0.8:
            kstar = int(rng.integers(1, kmax + 1))
            feas[kstar] = sorted(rng.choice(size[kstar], size=min(3, size[kstar]), replace=False).tolist())
        out.append({"kmax": kmax, "size": size, "feas": feas})
    return out


def _worker(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = FakeSession(make_instances(seed))

    def allreduce_min(t):
        dist.all_reduce(t, op=dist.ReduceOp.MIN)

    levels = run_levels_sharded(s, rank, world, allreduce_min)
    q.put((rank, levels, s.result, s.enumerated))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_level_sharding_gloo_world2(seed):
    ref = FakeSession(make_instances(seed))
    ref_levels = run_levels_sharded(ref, 0, 1, lambda t: None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    for rank, levels, result, enumerated in got:
        assert levels == ref_levels
        assert result == ref.result  # every rank commits the same canonical answer
    # the two shards together enumerate exactly what one rank enumerates
    assert [a + b for a, b in zip(got[0][3], got[1][3])] == ref.enumerated


class FakePairSession:
    """Stand-in of the fused pair session (gr_pair_*): one level loop decides
    two solves per instance -- PMS (feasible ranks feas) and MHS (feasible
    ranks feas_m, a superset: the MHS ignores phi-) -- an instance stays
    listed while either searches, and level_keys() returns both key arrays."""

    def __init__(self, inst, chunk=3):
        self.inst, self.chunk = inst, chunk
        self.B = len(inst)
        self.keys = (torch.full((self.B,), NONE, dtype=torch.int64),
                     torch.full((self.B,), NONE, dtype=torch.int64))
        self.open = [[True] * self.B, [True] * self.B]
        self.result = [[None] * self.B, [None] * self.B]
        self.active = list(range(self.B))

    def prepare(self):
        return len(self.active)

    def level(self, k, shard, nshard):
        for b in self.active:
            size = self.inst[b]["size"][k]
            nch = (size + self.chunk - 1) // self.chunk
            for s, key in enumerate(("feas", "feas_m")):
                if not self.open[s][b]:
                    continue
                feas = self.inst[b][key].get(k, [])
                for c in range(shard, nch, nshard):
                    lo, hi = c * self.chunk, min((c + 1) * self.chunk, size)
                    hit = [r for r in feas if lo <= r < hi]
                    if hit:
                        self.keys[s][b] = min(int(self.keys[s][b]), hit[0])

    def level_keys(self):
        return self.keys

    def finish(self, k):
        nxt = []
        for b in self.active:
            for s in (0, 1):
                if not self.open[s][b]:
                    continue
                if int(self.keys[s][b]) != NONE:
                    self.result[s][b], self.open[s][b] = (k, int(self.keys[s][b])), False
                elif k >= self.inst[b]["kmax"]:
                    self.result[s][b], self.open[s][b] = ("UNSAT",), False
            if self.open[0][b] or self.open[1][b]:
                nxt.append(b)
        self.active = nxt
        for t in self.keys:
            t.fill_(NONE)
        return len(nxt)


def make_pair_instances(seed):
    rng = np.random.default_rng(seed)
    out = make_instances(seed)
    for x in out:
        fm = {}
        for k, size in x["size"].items():
            if rng.random() < 0.4 or k in x["feas"]:
                extra = rng.choice(size, size=min(2, size), replace=False).tolist()
                fm[k] = sorted(set(extra) | set(x["feas"].get(k, [])))
        x["feas_m"] = fm
    return out


def _pair_worker(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = FakePairSession(make_pair_instances(seed))
    levels = run_levels_sharded(s, rank, world, lambda t: dist.all_reduce(t, op=dist.ReduceOp.MIN))
    q.put((rank, levels, s.result))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [3, 4])
def test_pair_level_sharding_gloo_world2(seed):
    """The fused pair session through the sharded driver (both key arrays
    all-reduced per level) at world 2 = world 1, for both solves."""
    ref = FakePairSession(make_pair_instances(seed))
    ref_levels = run_levels_sharded(ref, 0, 1, lambda t: None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_pair_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, levels, result in got:
        assert levels == ref_levels and result == ref.result


def test_shard_instances_balanced_and_complete():
    rng = np.random.default_rng(0)
    m = rng.integers(0, 33, size=748)
    n = rng.integers(1, 65, size=748)
    costs = estimate_costs(m, n)
    for world in (1, 2, 4, 8):
        parts = shard_instances(costs, world)
        allidx = sorted(i for p in parts for i in p)
        assert allidx == list(range(748))
        loads = [costs[p].sum() for p in parts]
        assert max(loads) <= 2.0 * (sum(loads) / world) + costs.max()


# ---- column-sharded greedy (C5 protocol) ------------------------------------------
class FakeGreedyShard:
    """CPU stand-in of one rank's gr_greedy_shard_* calls: this rank's clauses
    (lists of variable ids) and the replicated negatives."""

    def __init__(self, m, clauses, neg, w=None):
        self.m, self.cl, self.neg = m, [set(c) for c in clauses], [set(c) for c in neg]
        self.w = w
        self.counts = torch.zeros(m, dtype=torch.int32)

    def _local_counts(self):
        c = np.zeros(self.m, np.int64)
        for i, cl in enumerate(self.cl):
            if self.unc[i]:
                for v in cl:
                    c[v] += 1
        self.counts.copy_(torch.from_numpy(c.astype(np.int32)))

    def begin(self):
        self.unc = [True] * len(self.cl)
        self.picks, self.done = [], False
        self._local_counts()

    def step(self):  # counts hold the all-reduced global counts
        if not self.done:
            g = self.counts.numpy()
            if g.max() == 0:
                self.done = True
            else:
                if self.w is None:
                    v = int(np.argmax(g))  # first maximum = lowest index on ties
                else:  # ratio rule (R20): max g/w, cross-multiplied, lowest index on ties
                    v = 0
                    for u in range(1, self.m):
                        if int(g[u]) * self.w[v] > int(g[v]) * self.w[u]:
                            v = u
                self.picks.append(v)
                for i, cl in enumerate(self.cl):
                    if v in cl:
                        self.unc[i] = False
        self._local_counts()

    def state(self, picks=None):
        if picks is not None:
            picks[:len(self.picks)] = torch.tensor(self.picks, dtype=torch.int32)
        self.removed = set()
        return len(self.picks), self.done

    def private(self, only, flags):
        live = [p for j, p in enumerate(self.picks) if j not in self.removed]
        js = range(len(self.picks)) if only < 0 else [only]
        for j in js:
            v = self.picks[j]
            for cl in self.cl:
                if v in cl and sum(1 for p in live if p in cl) == 1:
                    flags[j] = 1
                    break

    def remove(self, j):
        self.removed.add(j)

    def finalize(self, removed, assign, status):
        S = {p for j, p in enumerate(self.picks) if not int(removed[j])}
        for v in S:
            assign[v // 64] |= 1 << (v % 64) if v % 64 < 63 else -(1 << 63)
        status[0] = 2 if any(n <= S for n in self.neg) else 0


def greedy_instance(seed):
    rng = np.random.default_rng(seed)
    m, n = 40, 120
    H = rng.choice(m, size=6, replace=False)
    cl = []
    for _ in range(n):
        s = int(rng.integers(2, 6))
        c = {int(rng.choice(H))} | set(rng.choice(m, size=s - 1, replace=False).tolist())
        cl.append(sorted(c))
    neg = [sorted(rng.choice(m, size=2, replace=False).tolist()) for _ in range(4)]
    return m, cl, neg


def weighted_golden_instance():
    """tests/golden/weighted_prune_order.txt as 0-based clause lists + weights"""
    g = load_golden("weighted_prune_order.txt")
    return g["m"], [[v - 1 for v in c] for c in g["pos"]], [], g["w"]


def _greedy_worker(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2011_08373_b200.multigpu import column_range, run_greedy_sharded

    if seed == "weighted":
        m, cl, neg, w = weighted_golden_instance()
    else:
        (m, cl, neg), w = greedy_instance(seed), None
    c0, c1 = column_range(len(cl), rank, world)
    sh = FakeGreedyShard(m, cl[c0:c1], neg, w)

    def red(op):
        return lambda t: dist.all_reduce(t, op=op)

    assign, status, picks, n = run_greedy_sharded(sh, red(dist.ReduceOp.SUM), red(dist.ReduceOp.MAX),
                                                  steps_per_check=4, w=w)
    q.put((rank, assign.tolist(), int(status[0]), picks[:n].tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [0, 1, "weighted"])
def test_greedy_column_sharding_gloo_world2(seed):
    """The sharded protocol over two gloo ranks gives the textbook greedy of
    the whole phi+ (the oracle): same pick order, same pruned set, same phi-
    verdict.  "weighted": the ratio greedy on the golden prune-order instance
    (descending-weight reverse-delete, reading R12)."""
    import oracle

    if seed == "weighted":
        m, cl, neg, w = weighted_golden_instance()
    else:
        (m, cl, neg), w = greedy_instance(seed), None
    off = np.cumsum([0] + [len(c) for c in cl]).astype(np.int64)
    var = np.concatenate([np.array(c, np.int32) for c in cl])
    noff = np.cumsum([0] + [len(c) for c in neg]).astype(np.int64)
    nvar = np.concatenate([np.array(c, np.int32) for c in neg]) if neg else np.zeros(0, np.int32)
    ref = oracle.greedy_csr(m, off, var, noff, nvar, w=w)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_greedy_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_set = sorted(np.nonzero(ref.in_S)[0].tolist())
    for rank, assign, status, picks in got:
        assert picks == ref.picks.tolist()
        got_set = [v for v in range(m) if (assign[v // 64] >> (v % 64)) & 1]
        assert got_set == ref_set
        assert status == (2 if ref.status == oracle.SAT_NEG_VIOLATED else 0)


# ---- batch sharding with result collection ---------------------------------------
def _batch_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2011_08373_b200 import synth
    from paper_2011_08373_b200.multigpu import solve_batch_sharded

    cb = synth.c2_batch()
    cb = cb.subset([b for b in range(cb.B) if cb.m[b] <= 14])

    def solve(sub):  # CPU stand-in for this rank's GPU solve
        r = oracle.batch("pms", sub)
        return {"status": r.status, "assign": r.assign, "cost": r.cost, "decided": r.decided}

    def allgather(t):
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return outs

    out = solve_batch_sharded(cb, rank, world, solve, allgather)
    q.put((rank, {k: v.tolist() for k, v in out.items()}))
    dist.destroy_process_group()


def test_batch_sharding_allgather_gloo_world2():
    """Instances dealt by cost over two ranks + one all-gather = the
    single-rank results, in input order, on every rank."""
    import oracle
    from paper_2011_08373_b200 import synth

    cb = synth.c2_batch()
    cb = cb.subset([b for b in range(cb.B) if cb.m[b] <= 14])
    ref = oracle.batch("pms", cb)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in got:
        assert out["status"] == ref.status.tolist()
        assert np.array_equal(np.asarray(out["assign"], np.uint64).reshape(-1),
                              np.asarray(ref.assign, np.uint64).reshape(-1))
        assert out["decided"] == np.asarray(ref.decided, np.uint64).tolist()


# ---- batch split with the heavy-instance rule (§8(e)) --------------------------
class CpuPmsSession:
    """Unit-weight PMS of a small batch by brute force, level by level: the
    colex ranks of level k are cut into chunks of `chunk` ranks and chunk c
    goes to shard c mod G (gr_exact_level's protocol); level_keys() holds
    each instance's lowest feasible rank seen (NONE if none).  Stand-in for
    the GPU session on CPU (small m only)."""

    def __init__(self, cb, chunk=5):
        import itertools

        self.it = itertools
        self.inst = [cb.instance(b) for b in range(cb.B)]
        self.B, self.chunk = cb.B, chunk
        self.keys = torch.full((self.B,), NONE, dtype=torch.int64)
        self.res = {"status": np.zeros(self.B, np.int32), "cost": np.zeros(self.B, np.uint64),
                    "decided": np.zeros(self.B, np.uint64), "assign": np.zeros((self.B, 1), np.uint64)}
        self.subs = {}

    def _level(self, b, k):
        if (b, k) not in self.subs:
            m = self.inst[b][0]
            self.subs[(b, k)] = sorted(self.it.combinations(range(m), k), key=lambda s: tuple(reversed(s)))
        return self.subs[(b, k)]

    def _feasible(self, b, x):
        m, npos, mk, _ = self.inst[b]
        mk = [int(v) for v in mk[:, 0]]
        return all(mk[j] & x for j in range(npos)) and not any((mk[j] & ~x) == 0 for j in range(npos, len(mk)))

    def prepare(self):
        self.active = []
        for b in range(self.B):
            if self._feasible(b, 0):
                self.res["status"][b] = 0  # level 0: the empty set (no positive clause)
            else:
                self.active.append(b)
        return len(self.active)

    def level(self, k, shard, nshard):
        for b in self.active:
            subs = self._level(b, k)
            nch = (len(subs) + self.chunk - 1) // self.chunk
            for c in range(shard, nch, nshard):
                for r in range(c * self.chunk, min((c + 1) * self.chunk, len(subs))):
                    if self._feasible(b, sum(1 << i for i in subs[r])):
                        self.keys[b] = min(int(self.keys[b]), r)
                        break

    def level_keys(self):
        return self.keys

    def finish(self, k):
        nxt = []
        for b in self.active:
            key = int(self.keys[b])
            if key != NONE:
                self.res["cost"][b] = k
                self.res["assign"][b, 0] = sum(1 << i for i in self._level(b, k)[key])
            elif k >= self.inst[b][0]:
                self.res["status"][b] = 1  # UNSAT
            else:
                nxt.append(b)
        self.active = nxt
        self.keys.fill_(NONE)
        return len(nxt)


def _heavy_batch():
    from paper_2011_08373_b200 import synth

    cb = synth.c2_batch()
    cb = cb.subset([b for b in range(cb.B) if cb.m[b] <= 11][:40])
    costs = np.ones(cb.B)
    costs[3] = 100.0  # heavier than the fair share of two ranks
    return cb, costs


def _heavy_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2011_08373_b200.multigpu import solve_batch_split_heavy

    cb, costs = _heavy_batch()

    def solve(sub):  # CPU stand-in for this rank's GPU solve of its whole instances
        r = oracle.batch("pms", sub)
        return {"status": r.status, "assign": r.assign, "cost": r.cost, "decided": r.decided}

    def solve_heavy(sub):  # the heavy instances: level rank ranges over both ranks
        s = CpuPmsSession(sub)
        run_levels_sharded(s, rank, world, lambda t: dist.all_reduce(t, op=dist.ReduceOp.MIN))
        return s.res

    def allgather(t):
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)
        return outs

    out, heavy = solve_batch_split_heavy(cb, rank, world, costs, solve, solve_heavy, allgather)
    q.put((rank, heavy, {k: v.tolist() for k, v in out.items()}))
    dist.destroy_process_group()


def test_split_heavy_rule():
    from paper_2011_08373_b200.multigpu import split_heavy

    assert split_heavy([1, 1, 10, 1], 2) == ([2], [0, 1, 3])
    assert split_heavy([1, 1, 1, 1], 2) == ([], [0, 1, 2, 3])
    assert split_heavy([5], 1) == ([], [0])


def test_batch_split_heavy_gloo_world2():
    """Light instances dealt whole + one all-gather, the heavy ones split by
    level rank ranges over both ranks (all-reduce MIN per level): the
    single-rank oracle's status, cost and assignment on every rank."""
    import oracle

    cb, _ = _heavy_batch()
    ref = oracle.batch("pms", cb)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_heavy_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, heavy, out in got:
        assert heavy == [3]
        assert out["status"] == ref.status.tolist()
        assert out["cost"] == np.asarray(ref.cost, np.uint64).tolist()
        assert np.array_equal(np.asarray(out["assign"], np.uint64).reshape(-1),
                              np.asarray(ref.assign, np.uint64).reshape(-1))
