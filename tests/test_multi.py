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
