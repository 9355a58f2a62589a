"""Multi-GPU drivers: one process per GPU, torch.distributed (NCCL over
NVLink / NVSwitch) for the plumbing.  SURVEY.md §8(e).

Two ways the Solve step shards:

* batch sharding (configs C2, C4): instances are independent, so each rank
  solves its own slice with no data-path collective (``shard_instances``);
  results may be gathered once at the end.
* rank-range sharding of one hard instance (config C3): every cardinality
  level's colex rank range is cut into fixed chunks and chunk c goes to rank
  c % G (``gr_exact_level(.., shard=r, nshard=G)``); after each level the
  per-instance minimum key is all-reduced (MIN, int64; 8 bytes per instance)
  so every rank commits the same level (``run_levels_sharded``).  This is the
  exact solvers' only real exchange step: one 8-byte all-reduce per level.
* column sharding of one huge phi+ for the greedy (config C5): each rank owns
  a contiguous range of clause columns; the counts are sums over clauses, so
  one all-reduce (SUM) of the m counts per pick gives every rank the same
  pick (``run_greedy_sharded`` over the gr_greedy_shard_* protocol).
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import numpy as np


def estimate_costs(m: Sequence[int], n_pos: Sequence[int]) -> np.ndarray:
    """Upper bound on each instance's enumeration work: 2^min(m, n_pos)
    candidates (every level up to k_max = min(m_eff, n_pos), R13)."""
    m = np.asarray(m, np.int64)
    n_pos = np.asarray(n_pos, np.int64)
    return np.exp2(np.minimum(m, np.maximum(n_pos, 0)).astype(np.float64))


def shard_instances(costs: Sequence[float], world: int) -> List[List[int]]:
    """Cost-balanced static split: sort by descending estimated cost and deal
    in a snake pattern (0,1,..,G-1,G-1,..,0,...).  Deterministic."""
    order = np.argsort(-np.asarray(costs, np.float64), kind="stable")
    out: List[List[int]] = [[] for _ in range(world)]
    for i, b in enumerate(order.tolist()):
        lap, pos = divmod(i, world)
        r = pos if lap % 2 == 0 else world - 1 - pos
        out[r].append(b)
    return [sorted(x) for x in out]


def run_levels_sharded(session, rank: int, world: int,
                       allreduce_min: Callable[[object], None]) -> int:
    """Level loop of a rank-range-sharded exact solve.

    ``session`` offers prepare() -> n_active, level(k, shard, nshard),
    level_keys() (a tensor of the B int64 level keys) and finish(k) ->
    n_active (an ExactSession on the GPU).  Every rank runs the same loop; the
    only exchange is ``allreduce_min(level_keys)`` once per level.  Returns
    the number of levels enumerated."""
    n = session.prepare()
    k = 0
    while n > 0:
        k += 1
        session.level(k, rank, world)
        keys = session.level_keys()
        for t in (keys if isinstance(keys, tuple) else (keys,)):  # PairSession: PMS and MHS keys
            allreduce_min(t)
        n = session.finish(k)
    return k


def nccl_allreduce_min(group=None):
    import torch.distributed as dist

    def f(t):
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)

    return f


def solve_exact_sharded(db, which: int, rank: int, world: int, group=None, out=None):
    """Exact PMS (which = 0) or MHS (1) of a batch whose level rank ranges are
    split across the ranks of ``group``; every rank returns the same result."""
    from . import _native as N

    s = N.ExactSession(db, which, out=out)
    levels = run_levels_sharded(s, rank, world,
                                nccl_allreduce_min(group) if world > 1 else (lambda t: None))
    return s.out, levels


def solve_pair_sharded(db, rank: int, world: int, group=None, out_pms=None, out_mhs=None):
    """PMS and MHS of a unit-weight batch decided by ONE fused walk whose
    level rank ranges are split across the ranks of ``group`` (gr_pair_*):
    per level one NCCL all-reduce (MIN) of each key array.  Every rank returns
    the same (out_pms, out_mhs, levels)."""
    from . import _native as N

    s = N.PairSession(db, out_pms=out_pms, out_mhs=out_mhs)
    levels = run_levels_sharded(s, rank, world,
                                nccl_allreduce_min(group) if world > 1 else (lambda t: None))
    return s.out_pms, s.out_mhs, levels


# ---- column-sharded greedy (C5) ------------------------------------------------
def removal_order(picks: Sequence[int], w=None) -> List[int]:
    """Positions 0..n-1 of the picks in reverse-delete order (reading R12):
    reverse pick order; with weights (weighted mhs) descending weight, equal
    weights in reverse pick order."""
    order = list(range(len(picks) - 1, -1, -1))
    if w is not None:
        order.sort(key=lambda j: -int(w[int(picks[j])]))  # stable: ties stay reverse-pick
    return order


def run_greedy_sharded(shard, allreduce_sum: Callable[[object], None],
                       allreduce_max: Callable[[object], None], steps_per_check: int = 32,
                       w=None):
    """Greedy mhs over phi+ split by clause columns across ranks (SURVEY.md
    §8(e) C5).  ``shard`` offers the gr_greedy_shard_* protocol (a
    GreedyShard on the GPU): ``counts`` (int32 tensor [m]), begin(), step(),
    state(picks=None) -> (n_picks, done), private(only, flags), remove(j),
    finalize(removed, assign, status).  The exchanges are one all-reduce (SUM)
    of the m counts per pick and, in the prune, one all-reduce (MAX) of the
    private flags plus one single-flag all-reduce per re-checked pick.
    ``w``: host weights [m] of the weighted mhs (they set the prune order),
    or None.  Returns (assign, status, picks, n_picks), identical on every
    rank."""
    import torch

    counts = shard.counts
    dev, m = counts.device, counts.numel()
    shard.begin()
    steps = 0
    while True:
        for _ in range(steps_per_check):
            allreduce_sum(counts)
            shard.step()
        steps += steps_per_check
        n, done = shard.state()
        if done:
            break
        if steps > m + 2 * steps_per_check:
            raise RuntimeError("sharded greedy did not terminate")
    picks = torch.full((m,), -1, dtype=torch.int32, device=dev)
    n, _ = shard.state(picks)
    # prune (R12): picks that are the sole hitter of a clause on some rank stay
    flags = torch.zeros(m, dtype=torch.int32, device=dev)
    shard.private(-1, flags)
    allreduce_max(flags)
    keep = flags[:n].cpu().tolist()
    removed = torch.zeros(m, dtype=torch.int32, device=dev)
    for j in removal_order(picks[:n].cpu().tolist(), w):  # the others, in removal order
        if keep[j]:
            continue
        fj = flags[j:j + 1]
        fj.zero_()
        shard.private(j, flags)
        allreduce_max(fj)
        if int(fj.item()) == 0:
            removed[j] = 1
            shard.remove(j)
    assign = torch.zeros((m + 63) // 64, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    shard.finalize(removed, assign, status)
    return assign, status, picks, n


def nccl_allreduce(op: str, group=None):
    import torch.distributed as dist

    red = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}[op]

    def f(t):
        dist.all_reduce(t, op=red, group=group)

    return f


def column_range(n_pos: int, rank: int, world: int):
    """Clause columns [c0, c1) of ``rank``: equal contiguous slices."""
    return n_pos * rank // world, n_pos * (rank + 1) // world


def greedy_matrix_sharded(bm_shard, rank: int, world: int, group=None, stream=None):
    """Greedy mhs of a C5-style phi+ whose clause columns are split across
    the ranks of ``group`` (each rank passes its own DeviceBitMatrix shard);
    every rank returns the same (assign, status, picks, n_picks)."""
    from . import _native as N

    sh = N.GreedyShard(bm_shard, stream=stream)
    w = None if bm_shard.w is None else bm_shard.w.cpu().numpy().view(np.uint32)
    if world > 1:
        return run_greedy_sharded(sh, nccl_allreduce("sum", group), nccl_allreduce("max", group),
                                  w=w)
    return run_greedy_sharded(sh, lambda t: None, lambda t: None, w=w)


# ---- batch sharding with result collection (C2 / C4) -------------------------------
def split_heavy(costs: Sequence[float], world: int, factor: float = 1.0):
    """§8(e) heavy-instance rule: an instance whose cost alone exceeds
    ``factor`` x the fair share (total / world) cannot be balanced by dealing
    whole instances; it is split by level rank ranges over all ranks instead.
    Returns (heavy, light) index lists (ascending)."""
    c = np.asarray(costs, np.float64)
    if world <= 1 or c.size == 0:
        return [], list(range(c.size))
    fair = c.sum() / world
    heavy = [int(b) for b in np.nonzero(c > factor * fair)[0]]
    hs = set(heavy)
    return heavy, [b for b in range(c.size) if b not in hs]


def _gather_rows(cb, parts, rank: int, solve_fn: Callable, allgather: Callable):
    """Each rank solves its slice ``parts[rank]`` with solve_fn(sub_batch) ->
    dict (status, assign, cost, decided); one all-gather of (index, status,
    cost, decided, assign) rows gives every rank the results in input order
    (entries of instances in no part stay 0)."""
    import torch

    mine = parts[rank]
    W = cb.W
    width = 4 + W
    maxn = max(max(len(p) for p in parts), 1)
    rows = torch.full((maxn, width), -1, dtype=torch.int64)
    if mine:
        r = solve_fn(cb.subset(mine))
        n = len(mine)
        rows[:n, 0] = torch.tensor(mine, dtype=torch.int64)
        rows[:n, 1] = torch.from_numpy(np.asarray(r["status"], np.int64))
        rows[:n, 2] = torch.from_numpy(np.asarray(r["cost"], np.uint64).view(np.int64))
        rows[:n, 3] = torch.from_numpy(np.asarray(r["decided"], np.uint64).view(np.int64))
        rows[:n, 4:] = torch.from_numpy(np.asarray(r["assign"], np.uint64).reshape(n, W).view(np.int64))
    got = allgather(rows)
    out = {"status": np.zeros(cb.B, np.int32), "cost": np.zeros(cb.B, np.uint64),
           "decided": np.zeros(cb.B, np.uint64), "assign": np.zeros((cb.B, W), np.uint64)}
    for g in got:
        g = g.cpu().numpy()
        g = g[g[:, 0] >= 0]
        idx = g[:, 0]
        out["status"][idx] = g[:, 1].astype(np.int32)
        out["cost"][idx] = g[:, 2].view(np.uint64)
        out["decided"][idx] = g[:, 3].view(np.uint64)
        out["assign"][idx] = g[:, 4:].view(np.uint64)
    return out


def solve_batch_split_heavy(cb, rank: int, world: int, costs: Sequence[float], solve_fn: Callable,
                            solve_heavy_fn: Callable, allgather: Callable, factor: float = 1.0):
    """Batch split with the heavy-instance rule (``split_heavy``): the light
    instances are dealt whole by cost and gathered as in solve_batch_sharded;
    the heavy ones are solved by all ranks together with
    ``solve_heavy_fn(sub_batch) -> dict`` -- a level loop whose rank ranges
    are split over the ranks (solve_exact_sharded / solve_pair_sharded on the
    GPU), which returns the same result on every rank.  Returns (results in
    input order, heavy indices)."""
    heavy, light = split_heavy(costs, world, factor)
    lc = np.asarray(costs, np.float64)[light] if light else np.zeros(0)
    parts = [[light[i] for i in p] for p in shard_instances(lc, world)] if light else [[] for _ in range(world)]
    out = _gather_rows(cb, parts, rank, solve_fn, allgather)
    if heavy:
        r = solve_heavy_fn(cb.subset(heavy))
        out["status"][heavy] = np.asarray(r["status"], np.int32)
        out["cost"][heavy] = np.asarray(r["cost"], np.uint64)
        out["decided"][heavy] = np.asarray(r["decided"], np.uint64)
        out["assign"][heavy] = np.asarray(r["assign"], np.uint64).reshape(len(heavy), cb.W)
    return out, heavy


def solve_batch_sharded(cb, rank: int, world: int, solve_fn: Callable, allgather: Callable):
    """Solve a host ClauseBatch split across ranks: instances are dealt by
    estimated cost (``shard_instances``), each rank solves its slice with
    ``solve_fn(sub_batch) -> dict`` (status int32 [n], assign uint64 [n, W],
    cost uint64 [n], decided uint64 [n]; e.g. a gr.solve_pms on this rank's
    GPU), and one all-gather of (index, status, cost, decided, assign) rows
    gives every rank the whole batch's results in input order.  The gather is
    result collection after the solve, not part of the data path.
    ``allgather(t) -> list of tensors`` (one per rank, same shape as t)."""
    parts = shard_instances(estimate_costs(cb.m, cb.n_pos), world)
    return _gather_rows(cb, parts, rank, solve_fn, allgather)


def measured_costs(cb, device="cuda") -> np.ndarray:
    """Per-instance cost for the batch split, measured: the candidates each
    instance's exact PMS + MHS decides (gr_result.decided of one solve on
    this rank's GPU; the level loop's work grows with it), plus a constant
    per instance for its pack and level commits."""
    from . import _native as N

    db = N.DeviceBatch.from_host(cb, device=device)
    p, h = N.solve_pms_mhs(db)
    r = N.to_host_many([p, h])
    return r[0]["decided"].astype(np.float64) + r[1]["decided"].astype(np.float64) + 1e4


def solve_batch_sharded_device(cb, parts, rank: int, db, outs, allgather):
    """One rank's share of a batch split over the ranks (``parts`` from
    shard_instances): PMS + MHS (one launch) and greedy of the rank's
    sub-batch ``db`` into ``outs`` on its GPU, then one all-gather of
    (index, PMS status/cost/decided/assign, MHS decided) rows -- on the
    device, NCCL -- so every rank holds the whole batch's results in input
    order (host arrays)."""
    import torch

    from . import _native as N

    mine = parts[rank]
    W = cb.W
    width = 5 + W
    maxn = max(max(len(p) for p in parts), 1)
    dev = outs[0].status.device if outs else torch.device("cuda")
    rows = torch.full((maxn, width), -1, dtype=torch.int64, device=dev)
    if mine:
        N.solve_pms_mhs(db, outs[0], outs[1])
        N.mhs_greedy(db, outs[2])
        n = len(mine)
        rows[:n, 0] = torch.tensor(mine, dtype=torch.int64, device=dev)
        rows[:n, 1] = outs[0].status.to(torch.int64)
        rows[:n, 2] = outs[0].cost
        rows[:n, 3] = outs[0].decided
        rows[:n, 4] = outs[1].decided
        rows[:n, 5:] = outs[0].assign
    got = torch.cat(allgather(rows)).cpu().numpy()
    got = got[got[:, 0] >= 0]
    idx = got[:, 0]
    out = {"status": np.zeros(cb.B, np.int32), "cost": np.zeros(cb.B, np.uint64),
           "decided_pms": np.zeros(cb.B, np.uint64), "decided_mhs": np.zeros(cb.B, np.uint64),
           "assign": np.zeros((cb.B, W), np.uint64)}
    out["status"][idx] = got[:, 1].astype(np.int32)
    out["cost"][idx] = got[:, 2].view(np.uint64)
    out["decided_pms"][idx] = got[:, 3].view(np.uint64)
    out["decided_mhs"][idx] = got[:, 4].view(np.uint64)
    out["assign"][idx] = got[:, 5:].view(np.uint64)
    return out


def nccl_allgather(group=None, device=None):
    """all_gather over the group: on the device with NCCL (gloo, e.g. the
    one-GPU functional check, gathers host copies)."""
    import torch
    import torch.distributed as dist

    def f(t):
        if dist.get_backend(group) == "gloo":
            t = t.cpu()
        elif device is not None:
            t = t.to(device)
        outs = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(outs, t, group=group)
        return outs

    return f
