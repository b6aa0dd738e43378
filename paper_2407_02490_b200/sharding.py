"""Head sharding for multi-GPU pre-fill (one process per GPU, torch.distributed).

Heads are independent (SPEC.md:422 of the reference: "safe to parallelize
across rows and across heads"), so the only partitioning is over q-heads:
every rank runs estimation -> compaction -> sparse attention for its own
q-heads and needs only the kv heads those q-heads read (GQA map
h -> h // (Hq / Hkv)).  There is no collective on the data path; the optional
all-gather of the per-head outputs is the one exchange.

* ``shard_heads`` -- balanced contiguous q-head ranges (sizes differ by at
  most one).  When ``world`` divides ``n_kv_heads`` the ranges are whole kv
  groups (no K/V duplication, LLaMA 32/8 on 8 GPUs = 1 kv head + 4 q-heads
  each); otherwise a kv group is split and its K/V is replicated on the ranks
  that share it (Qwen2 28/4 on 8 GPUs: 4+3 q-heads per group).
* ``plan_heads_lpt`` -- the same with per-head predicted costs (e.g.
  ``patterns.flops_in_kernel`` of each head's pattern, summed over layers):
  longest-processing-time assignment of whole kv groups when ``world`` <= the kv
  head count, of single q-heads otherwise ("use LPT on
  predicted cost").
* ``HeadShard.kv_stack`` -- the global kv heads to stack as the rank's local
  K/V so that the kernels' GQA map (local q-head i reads local kv head
  i // (n_q / n_kv_local)) holds; a rank whose q-heads split kv groups unevenly
  gets one kv entry per q-head.
* ``gather_heads`` -- all-gather of ragged per-rank head blocks, reassembled in
  global head order.
* ``max_over_ranks`` -- the timing rule (device time, max over ranks).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    q_heads: tuple  # global q-head ids owned by this rank, ascending
    q_per_kv: int

    @property
    def n_q(self) -> int:
        return len(self.q_heads)

    @property
    def contiguous(self) -> bool:
        return not self.q_heads or self.q_heads[-1] - self.q_heads[0] + 1 == len(self.q_heads)

    @property
    def q_begin(self) -> int:
        return self.q_heads[0] if self.q_heads else 0

    @property
    def q_end(self) -> int:
        return self.q_heads[-1] + 1 if self.q_heads else 0

    @property
    def kv_heads(self) -> tuple:
        """Distinct global kv heads read by this rank's q-heads, ascending."""
        return tuple(sorted({h // self.q_per_kv for h in self.q_heads}))

    @property
    def kv_begin(self) -> int:
        return self.kv_heads[0] if self.q_heads else 0

    @property
    def kv_end(self) -> int:
        return self.kv_heads[-1] + 1 if self.q_heads else 0

    @property
    def n_kv(self) -> int:
        return len(self.kv_heads)

    @property
    def kv_stack(self) -> tuple:
        """Global kv heads, in order, forming the rank's local K/V for the kernels: the
        distinct kv heads when every one of them serves the same number of local
        q-heads (in q-head order), otherwise one kv head per local q-head."""
        groups = [h // self.q_per_kv for h in self.q_heads]
        kvs = self.kv_heads
        r = len(groups) // len(kvs) if kvs else 0
        if kvs and r * len(kvs) == len(groups) and all(g == kvs[i // r] for i, g in enumerate(groups)):
            return kvs
        return tuple(groups)

    def local_kv_index(self, q_head: int) -> int:
        """Index into ``kv_stack`` of the kv head read by global q-head ``q_head``."""
        i = self.q_heads.index(q_head)
        stack = self.kv_stack
        return i // (len(self.q_heads) // len(stack))


def _ranges(n: int, world: int):
    base, extra = divmod(n, world)
    out, start = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def _check(n_q_heads: int, n_kv_heads: int, world: int, rank: int):
    if n_kv_heads < 1 or n_q_heads % n_kv_heads:
        raise ValueError("n_q_heads must be a positive multiple of n_kv_heads")
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if world > n_q_heads:
        raise ValueError(f"{world} ranks for {n_q_heads} q-heads: some ranks would have no work")


def shard_heads(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> HeadShard:
    _check(n_q_heads, n_kv_heads, world, rank)
    qpk = n_q_heads // n_kv_heads
    if n_kv_heads % world == 0:  # whole kv groups per rank
        kv0, kv1 = _ranges(n_kv_heads, world)[rank]
        return HeadShard(rank, world, tuple(range(kv0 * qpk, kv1 * qpk)), qpk)
    q0, q1 = _ranges(n_q_heads, world)[rank]
    return HeadShard(rank, world, tuple(range(q0, q1)), qpk)


def lpt_assign(costs, world: int):
    """Longest-processing-time list scheduling: units in decreasing cost (ties: lower
    index first) go to the least-loaded rank (ties: lower rank).  Deterministic, so
    every rank computes the same plan.  Returns the ascending unit lists per rank."""
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    loads = [0.0] * world
    bins = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda x: (loads[x], x))
        bins[r].append(i)
        loads[r] += float(costs[i])
    return [sorted(b) for b in bins]


def plan_heads_lpt(head_costs, n_kv_heads: int, world: int, rank: int) -> HeadShard:
    """Cost-balanced head shard (see the module docstring); ``head_costs`` has one
    non-negative predicted cost per q-head."""
    n_q = len(head_costs)
    _check(n_q, n_kv_heads, world, rank)
    qpk = n_q // n_kv_heads
    if world <= n_kv_heads:
        group_costs = [sum(head_costs[g * qpk:(g + 1) * qpk]) for g in range(n_kv_heads)]
        groups = lpt_assign(group_costs, world)[rank]
        heads = tuple(h for g in groups for h in range(g * qpk, (g + 1) * qpk))
    else:
        heads = tuple(lpt_assign(head_costs, world)[rank])
    if not heads:
        raise ValueError("a rank received no heads")
    return HeadShard(rank, world, heads, qpk)


class PendingGather:
    """An in-flight all-gather of per-rank head blocks (gather_heads_async)."""

    def __init__(self, work, bufs, shards, like: torch.Tensor):
        self._work, self._bufs, self._shards, self._like = work, bufs, shards, like

    def wait(self) -> torch.Tensor:
        """Make the current stream wait for the exchange; the full [n_q_total, ...] tensor."""
        self._work.wait()
        bufs, shards, local = self._bufs, self._shards, self._like
        sizes = [s.n_q for s in shards]
        if all(s.contiguous for s in shards) and [s.q_begin for s in shards] == sorted(s.q_begin for s in shards):
            return torch.cat([b[:n] for b, n in zip(bufs, sizes)], dim=0)
        full = torch.empty((sum(sizes),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        for b, s in zip(bufs, shards):
            full[torch.tensor(s.q_heads, device=local.device)] = b[: s.n_q]
        return full


def gather_heads_async(local: torch.Tensor, shards, group=None) -> PendingGather:
    """Start the all-gather of this rank's [n_q_local, ...] block (SURVEY.md 8(e)'s optional
    collective) without blocking: the block is first copied into a padded send buffer on
    the current stream, so the caller may overwrite ``local`` right away (e.g. with the
    next layer's attention) while the exchange overlaps it; ``wait()`` assembles."""
    import torch.distributed as dist

    sizes = [s.n_q for s in shards]
    width = max(sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in shards]
    work = dist.all_gather(bufs, pad, group=group, async_op=True)
    return PendingGather(work, bufs, shards, local)


def gather_heads(local: torch.Tensor, shards, group=None) -> torch.Tensor:
    """All-gather per-rank [n_q_local, ...] blocks into [n_q_total, ...] (global head order)."""
    return gather_heads_async(local, shards, group).wait()


def max_over_ranks(value: float, device=None, group=None) -> float:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    if dist.get_backend(group) == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
