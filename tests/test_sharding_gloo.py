"""CPU, world_size 2 over gloo: the multi-GPU head sharding (sharding.py) covers
every q-head exactly once, gives each rank the kv heads its q-heads read, and
the optional output all-gather reassembles the full layer in head order.  Each
rank computes its heads with the CPU oracle (no GPU here) on a small layer."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_02490_b200.sharding import shard_heads


def test_shards_partition_heads():
    for hq, hkv in [(32, 8), (56, 8), (28, 4), (8, 8), (4, 1)]:
        for world in (1, 2, 4, 8):
            if world > hq:
                continue
            shards = [shard_heads(hq, hkv, world, r) for r in range(world)]
            owned = [h for s in shards for h in range(s.q_begin, s.q_end)]
            assert owned == list(range(hq)), (hq, hkv, world)
            sizes = [s.n_q for s in shards]
            assert max(sizes) - min(sizes) <= (hq // hkv if hkv % world == 0 else 1)
            for s in shards:
                for h in range(s.q_begin, s.q_end):
                    assert 0 <= s.local_kv_index(h) < s.n_kv
                if hkv % world == 0:  # whole kv groups: no K/V duplication
                    assert s.n_q == s.n_kv * (hq // hkv)
    with pytest.raises(ValueError):
        shard_heads(6, 4, 2, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as orc
        from paper_2407_02490_b200.sharding import gather_heads, max_over_ranks

        s_len, d, b, hq, hkv = 96, 16, 16, 6, 2
        rng = np.random.Generator(np.random.PCG64(3))
        q = rng.standard_normal((hq, s_len, d)).astype(np.float32)
        k = rng.standard_normal((hkv, s_len, d)).astype(np.float32)
        v = rng.standard_normal((hkv, s_len, d)).astype(np.float32)
        shards = [shard_heads(hq, hkv, world, r) for r in range(world)]
        me = shards[rank]
        k_loc, v_loc = k[me.kv_begin:me.kv_end], v[me.kv_begin:me.kv_end]
        outs = []
        for h in range(me.q_begin, me.q_end):
            tiles, cols, _ = orc.build_vs_layout_with_stats(*orc.estimate_vertical_slash(
                q[h], k[h // (hq // hkv)], 8, 12, 16), s_len, b)
            ts, to = orc.flatten(tiles)
            cs, co = orc.flatten(cols)
            kv = me.local_kv_index(h)
            outs.append(orc.sparse_flash_rows(q[h], k_loc[kv], v_loc[kv], d ** -0.5, b, ts, to, cs, co))
        full = gather_heads(torch.from_numpy(np.stack(outs)), shards)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            ref = []
            for h in range(hq):
                tiles, cols, _ = orc.build_vs_layout_with_stats(*orc.estimate_vertical_slash(
                    q[h], k[h // (hq // hkv)], 8, 12, 16), s_len, b)
                ts, to = orc.flatten(tiles)
                cs, co = orc.flatten(cols)
                ref.append(orc.sparse_flash_rows(q[h], k[h // (hq // hkv)], v[h // (hq // hkv)], d ** -0.5, b,
                                                 ts, to, cs, co))
            result["max_err"] = float(np.max(np.abs(full.numpy() - np.stack(ref))))
            result["shape"] = tuple(full.shape)
            result["t"] = t
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_sharded_layer(world):
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    assert result["shape"] == (6, 96, 16)
    assert result["max_err"] == 0.0  # same CPU computation, reassembled in head order
    assert result["t"] == float(world)  # max over ranks
