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

from paper_2407_02490_b200.sharding import lpt_assign, plan_heads_lpt, shard_heads


def _check_kernel_map(s, qpk):
    """The kernels' GQA map over the rank's stacked K/V reads each head's own kv head."""
    stack = s.kv_stack
    ratio = s.n_q // len(stack)
    assert ratio * len(stack) == s.n_q
    for i, h in enumerate(s.q_heads):
        assert stack[i // ratio] == h // qpk
        assert s.local_kv_index(h) == i // ratio


def test_shards_partition_heads():
    for hq, hkv in [(32, 8), (56, 8), (28, 4), (8, 8), (4, 1)]:
        for world in (1, 2, 4, 8):
            if world > hq:
                continue
            shards = [shard_heads(hq, hkv, world, r) for r in range(world)]
            owned = [h for s in shards for h in s.q_heads]
            assert owned == list(range(hq)), (hq, hkv, world)
            sizes = [s.n_q for s in shards]
            assert max(sizes) - min(sizes) <= (hq // hkv if hkv % world == 0 else 1)
            for s in shards:
                _check_kernel_map(s, hq // hkv)
                if hkv % world == 0:  # whole kv groups: no K/V duplication
                    assert s.n_q == s.n_kv * (hq // hkv) and s.kv_stack == s.kv_heads
    # Qwen2 28/4 on 8 GPUs: rank 1 holds q-heads 4..7 = three of group 0 and one of group 1,
    # so its K/V stack has one entry per q-head
    s = shard_heads(28, 4, 8, 1)
    assert s.q_heads == (4, 5, 6, 7) and s.kv_stack == (0, 0, 0, 1)
    with pytest.raises(ValueError):
        shard_heads(6, 4, 2, 0)


def test_lpt_plans():
    # 5 -> r0, 4 -> r1, 3 -> r1 (4 < 5), 2 -> r0 (5 < 7), 1 -> r0 (7 == 7, lower rank)
    assert lpt_assign([5, 1, 4, 2, 3], 2) == [[0, 1, 3], [2, 4]]
    rng = np.random.Generator(np.random.PCG64(7))
    for hq, hkv, world in [(32, 8, 2), (32, 8, 4), (56, 8, 8), (28, 4, 8), (28, 4, 3), (8, 2, 8)]:
        costs = rng.uniform(1.0, 10.0, hq).tolist()
        shards = [plan_heads_lpt(costs, hkv, world, r) for r in range(world)]
        owned = sorted(h for s in shards for h in s.q_heads)
        assert owned == list(range(hq))
        qpk = hq // hkv
        for s in shards:
            _check_kernel_map(s, qpk)
            if world <= hkv:  # whole kv groups
                assert s.n_q == s.n_kv * qpk
        loads = [sum(costs[h] for h in s.q_heads) for s in shards]
        unit = max(costs) * (qpk if world <= hkv else 1)
        assert max(loads) - min(loads) <= unit + 1e-9  # LPT bound: within one unit
        assert [plan_heads_lpt(costs, hkv, world, r) for r in range(world)] == shards  # deterministic
    # a skewed cost vector moves whole groups away from the contiguous split
    costs = [10.0] * 8 + [1.0] * 24  # kv groups 0, 1 expensive (32/8)
    a, b = plan_heads_lpt(costs, 8, 2, 0), plan_heads_lpt(costs, 8, 2, 1)
    assert set(a.kv_heads) & {0, 1} and set(b.kv_heads) & {0, 1}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result, plan):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as orc
        from paper_2407_02490_b200.sharding import gather_heads, gather_heads_async, max_over_ranks

        s_len, d, b, hq, hkv = 96, 16, 16, 6, 2
        rng = np.random.Generator(np.random.PCG64(3))
        q = rng.standard_normal((hq, s_len, d)).astype(np.float32)
        k = rng.standard_normal((hkv, s_len, d)).astype(np.float32)
        v = rng.standard_normal((hkv, s_len, d)).astype(np.float32)
        if plan == "lpt":
            costs = [1.0, 5.0, 2.0, 2.0, 9.0, 1.0]  # groups of 3: {0,1,2} = 8, {3,4,5} = 12
            shards = [plan_heads_lpt(costs, hkv, world, r) for r in range(world)]
            assert shards[0].q_heads == (3, 4, 5)  # the dearer group goes to rank 0: gather reorders
        else:
            shards = [shard_heads(hq, hkv, world, r) for r in range(world)]
        me = shards[rank]
        k_loc, v_loc = k[list(me.kv_stack)], v[list(me.kv_stack)]
        outs = []
        for h in me.q_heads:
            tiles, cols, _ = orc.build_vs_layout_with_stats(*orc.estimate_vertical_slash(
                q[h], k[h // (hq // hkv)], 8, 12, 16), s_len, b)
            ts, to = orc.flatten(tiles)
            cs, co = orc.flatten(cols)
            kv = me.local_kv_index(h)
            outs.append(orc.sparse_flash_rows(q[h], k_loc[kv], v_loc[kv], d ** -0.5, b, ts, to, cs, co))
        full = gather_heads(torch.from_numpy(np.stack(outs)), shards)
        # overlapped form: the block may be overwritten (next layer) right after the call
        loc = torch.from_numpy(np.stack(outs)).clone()
        pending = gather_heads_async(loc, shards)
        loc.fill_(float("nan"))
        full_async = pending.wait()
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
            result["async_equal"] = bool(torch.equal(full_async, full))
            result["shape"] = tuple(full.shape)
            result["t"] = t
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,plan", [(2, "contiguous"), (2, "lpt")])
def test_two_rank_gloo_sharded_layer(world, plan):
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), result, plan), nprocs=world, join=True)
    assert result["shape"] == (6, 96, 16)
    assert result["max_err"] == 0.0  # same CPU computation, reassembled in head order
    assert result["async_equal"]  # the overlapped gather copies the block before returning
    assert result["t"] == float(world)  # max over ranks


def test_bench_spawns_world_size_ranks():
    """`python bench.py --gpus 2` without torchrun env must launch 2 ranks itself (torchrun
    re-exec, 127.0.0.1 rendezvous), take the max over ranks and print ONE JSON line with
    n_gpus 2 from rank 0 (--dry-run: the same launch and reduction over gloo, no GPU)."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=repo)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, res.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] == 2.0  # max over the ranks' 1.0 and 2.0
    assert rec["rank0_q_heads"] == list(range(16))
