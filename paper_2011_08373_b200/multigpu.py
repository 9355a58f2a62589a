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
  method's only real exchange step: one 8-byte all-reduce per level.
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
        allreduce_min(session.level_keys())
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
