"""Head sharding for multi-GPU pre-fill (one process per GPU, torch.distributed).

Heads are independent (SPEC.md:422 of the reference: "safe to parallelize
across rows and across heads"), so the only partitioning is over q-heads:
every rank runs estimation -> compaction -> sparse attention for its own
contiguous range of q-heads and needs only the kv heads those q-heads read
(GQA map h -> h // (Hq / Hkv)).  There is no collective on the data path; the
optional all-gather of the per-head outputs is the one exchange (SURVEY.md
8(e)).

* ``shard_heads`` -- balanced contiguous q-head ranges (sizes differ by at
  most one).  When ``world`` divides ``n_kv_heads`` the ranges are whole kv
  groups (no K/V duplication, LLaMA 32/8 on 8 GPUs = 1 kv head + 4 q-heads
  each); otherwise a kv group is split and its K/V is replicated on the ranks
  that share it (Qwen2 28/4 on 8 GPUs: 4+3 q-heads per group).
* ``gather_heads`` -- all-gather of ragged per-rank head blocks along dim 0.
* ``max_over_ranks`` -- the timing rule (device time, max over ranks).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    q_begin: int
    q_end: int
    kv_begin: int
    kv_end: int
    q_per_kv: int

    @property
    def n_q(self) -> int:
        return self.q_end - self.q_begin

    @property
    def n_kv(self) -> int:
        return self.kv_end - self.kv_begin

    def local_kv_index(self, q_head: int) -> int:
        """kv head (local to this shard's K/V slice) read by global q-head ``q_head``."""
        return q_head // self.q_per_kv - self.kv_begin


def _ranges(n: int, world: int):
    base, extra = divmod(n, world)
    out, start = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def shard_heads(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> HeadShard:
    if n_kv_heads < 1 or n_q_heads % n_kv_heads:
        raise ValueError("n_q_heads must be a positive multiple of n_kv_heads")
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if world > n_q_heads:
        raise ValueError(f"{world} ranks for {n_q_heads} q-heads: some ranks would have no work")
    qpk = n_q_heads // n_kv_heads
    if n_kv_heads % world == 0:  # whole kv groups per rank
        kv0, kv1 = _ranges(n_kv_heads, world)[rank]
        return HeadShard(rank, world, kv0 * qpk, kv1 * qpk, kv0, kv1, qpk)
    q0, q1 = _ranges(n_q_heads, world)[rank]
    return HeadShard(rank, world, q0, q1, q0 // qpk, (q1 - 1) // qpk + 1, qpk)


def gather_heads(local: torch.Tensor, shards, group=None) -> torch.Tensor:
    """All-gather per-rank [n_q_local, ...] blocks into [n_q_total, ...] (head order)."""
    import torch.distributed as dist

    sizes = [s.n_q for s in shards]
    width = max(sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in shards]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:n] for b, n in zip(bufs, sizes)], dim=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    if dist.get_backend(group) == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
