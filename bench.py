"""Benchmark: MInference dynamic sparse pre-fill attention on B200.

Metric (BASELINE.json): pre-fill attention latency (ms) at 128K tokens for
LLaMA-3-8B-1M attention, all 32 layers' per-head pattern configs (config
C2: 32 q-heads / 8 kv-heads, d = 128, mixed VS / A-shape / BS heads from
configs/llama3_8b_1m_c2.json), G-local synthetic bf16 inputs (SURVEY.md
8(d)).  One step = estimation + index compaction + sparse attention for all
32 layers (1024 heads), inputs resident in HBM (48 GB > L2, no flush needed).

    python bench.py [--gpus N --steps K --warmup W] [--config c2|c3|c4|c5] [--impl reference]

Multi-GPU (torchrun, one rank per GPU): q-heads are sharded over ranks
(paper_2407_02490_b200/sharding.py: whole kv groups when N divides the kv
heads; no data-path collective; strong scaling of the fixed job), time = max
over ranks.  ``--impl reference`` times the reference's CPU path on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

TILE_FLOPS_PER_CELL = 4  # QK^T + PV, 2 flops per MAC each (patterns.py:196-199)

CONFIGS = {
    # name: (seq_len, q_heads, kv_heads, layers, pattern source, inputs)
    "c2": dict(workload="c2_llama3_8b_1m_attention_32L_128k_mixed", seq_len=131072, hq=32, hkv=8, layers=32,
               patterns="configs/llama3_8b_1m_c2.json", inputs="G-local"),
    "c3": dict(workload="c3_llama3_8b_1m_attention_1L_1m_vs", seq_len=1048576, hq=32, hkv=8, layers=1,
               patterns="VS(1000,6096) all heads", inputs="G-local"),
    "c4": dict(workload="c4_yi_200k_attention_1L_256k_bs", seq_len=262144, hq=56, hkv=8, layers=1,
               patterns="BS(100) all heads", inputs="G-iid"),
    "c5": dict(workload="c5_qwen2_7b_attention_1L_512k_ashape", seq_len=524288, hq=28, hkv=4, layers=1,
               patterns="AShape(128,4096) all heads", inputs="G-iid"),
}


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def layer_configs(cfg):
    from benchmarks.workloads import load_layer_configs
    from paper_2407_02490_b200.patterns import AShape, VerticalSlash

    if cfg["patterns"].endswith(".json"):
        return load_layer_configs(os.path.join(REPO, cfg["patterns"]))
    from paper_2407_02490_b200.patterns import BlockSparse

    if cfg["patterns"].startswith("VS"):
        return [[VerticalSlash(1000, 6096)] * cfg["hq"] for _ in range(cfg["layers"])]
    if cfg["patterns"].startswith("BS"):
        return [[BlockSparse(100)] * cfg["hq"] for _ in range(cfg["layers"])]
    return [[AShape(128, 4096)] * cfg["hq"] for _ in range(cfg["layers"])]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm),
                "power_w_max": max((float(r[2]) for r in self.rows if len(r) >= 7 and r[2].replace(".", "").isdigit()),
                                   default=None)}


# ----------------------------------------------------------------------------- reference arm
def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from benchmarks import cpu_reference

    layers = layer_configs(cfg)
    cores = os.cpu_count() or 1
    vals = []
    info = None
    for step in range(args.warmup + args.steps):
        step_s, info = cpu_reference.run_sample(layers, cfg["seq_len"], 128, 64, cores, items_per_pattern=max(1, min(
            cores, 4)), n_sample_rows=args.ref_rows, step_seed=step)
        if step >= args.warmup:
            vals.append(step_s * 1e3)
    value = statistics.median(vals)
    sample = (f"{info['items']} (layer, head) items per step (per pattern) of {cfg['workload']}: full estimation + "
              f"full index build, kernel on {args.ref_rows} sampled row blocks extrapolated by tiles+chips; "
              f"code = {info['impl']}; step latency = sum(item s)/cores")
    line = {"impl": "reference", "modeled": True,
            "value_kind": (f"modeled: each step times a bounded sample ({info['items']} (layer, head) items; kernel on "
                           f"{args.ref_rows} row blocks each) and extrapolates to the whole workload by tile count"),
            "sample_items_per_step": info["items"],
            "metric": metric_name(args, cfg), "value": round(value, 3), "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 storage)", "data": "synthetic",
            # the workload identity keys of the GPU arm's config (same workload, shapes and patterns)
            "config": {"workload": cfg["workload"], "seq_len": cfg["seq_len"], "layers": cfg["layers"],
                       "q_heads": cfg["hq"], "kv_heads": cfg["hkv"], "head_dim": 128, "block_size": 64,
                       "patterns": cfg["patterns"], "inputs": cfg["inputs"] + " (SURVEY.md 8d)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "ms", "cores": cores, "kind": "reference"
                             if info["ref_kernel"] else "port", "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": info["patterns"]}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- helpers
def metric_name(args, cfg) -> str:
    if args.config == "c2":
        return "pre-fill attention latency (ms), LLaMA-3-8B-1M attention, 32 layers mixed per-head patterns @128K"
    return f"pre-fill attention latency (ms), {cfg['workload']}"


def union_steps(tiles_np, toff_np, n_rows, hq, paired=None):
    """Kernel steps of the 128-row CTAs: |tiles(2p) U tiles(2p+1)| per pair of row blocks
    (union kernel), or max(n(2p), n(2p+1)) for the heads in ``paired`` (paired-box
    kernel).  Returns (union steps, paired steps)."""
    import numpy as np

    counts = np.diff(toff_np)
    rows = np.repeat(np.arange(hq * n_rows, dtype=np.int64), counts)
    head = rows // n_rows
    pair = head * ((n_rows + 1) // 2) + (rows % n_rows) // 2
    keys = np.unique(pair * (np.int64(1) << 32) + tiles_np.astype(np.int64))
    u_head = np.bincount(keys >> 32, minlength=hq * ((n_rows + 1) // 2)).reshape(hq, -1).sum(axis=1)
    listed = [] if paired is None else [int(h) for h in np.asarray(paired).reshape(-1)]
    n_union, n_paired = int(u_head.sum()), 0
    for h in listed:
        c = counts[h * n_rows:(h + 1) * n_rows]
        if n_rows % 2:
            c = np.append(c, 0)
        m = int(np.maximum(c[0::2], c[1::2]).sum())
        # the library's routing (spf_internal.h pair_preferred): a listed head stays on the union
        # kernel unless its union steps exceed 1.6x its paired steps (Block-Sparse heads have no
        # residual columns, the other condition)
        if 5 * int(u_head[h]) > 8 * m:
            n_union -= int(u_head[h])
            n_paired += m
    return n_union, n_paired


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` launched directly (no WORLD_SIZE): re-exec under torchrun, one
    rank per GPU, rendezvous on 127.0.0.1; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    # communicator setup lines (one per rank) on stderr, so stdout keeps the one JSON line
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def dry_run(args, world, rank):
    """CPU plumbing check of the multi-rank path (no GPU): gloo process group, the same
    shard plan and max-over-ranks rule; each rank reports a synthetic per-rank time."""
    import torch.distributed as dist

    from paper_2407_02490_b200.sharding import max_over_ranks, shard_heads

    cfg = CONFIGS[args.config]
    if world > 1:
        dist.init_process_group("gloo")
    shard = shard_heads(cfg["hq"], cfg["hkv"], world, rank)
    ms = max_over_ranks(1.0 + rank, device=None)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": metric_name(args, cfg), "value": ms, "unit": "ms",
                          "n_gpus": world, "ms_per_step": ms, "rank0_q_heads": list(shard.q_heads)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def vs_bytes_min(cfgs_layer, S, D, HQ, HKV):
    """SURVEY 8(d) algorithmic bytes of one layer's estimation (bf16, e = 2):
    VS: K read once per kv head its VS heads use + the Q tail + the fp32 vertical/slash
    vectors written and read back + the selected indices; BS: Q and K read once."""
    from paper_2407_02490_b200.patterns import BlockSparse, VerticalSlash

    e, hpk = 2, HQ // HKV
    vs = [h for h, c in enumerate(cfgs_layer) if isinstance(c, VerticalSlash)]
    bs = [h for h, c in enumerate(cfgs_layer) if isinstance(c, BlockSparse)]
    out = 0
    if vs:
        kv = {h // hpk for h in vs}
        out += len(kv) * S * D * e + sum(cfgs_layer[h].last_q for h in vs) * D * e + len(vs) * S * 4 * 2 * 2
        out += sum(min(cfgs_layer[h].k_v, S) + min(cfgs_layer[h].k_s, S) for h in vs) * 4
    if bs:
        out += len(bs) * S * D * e + len({h // hpk for h in bs}) * S * D * e
    return out


def run_config(args, cfg, world, rank, local, dev, with_cpu, with_e2e, steps, label):
    """Measure one workload: estimation + compaction + sparse attention for every layer
    of this rank's heads, inputs resident in HBM.  Returns the per-config record."""
    import numpy as np
    import torch

    import paper_2407_02490_b200 as P
    from benchmarks.workloads import g_iid_qkv, g_local_qkv
    from paper_2407_02490_b200 import _lib, kernels
    from paper_2407_02490_b200.driver import PatternTable, SparsePrefill
    from paper_2407_02490_b200.prefill import _pair_heads
    from paper_2407_02490_b200.sharding import (gather_heads, gather_heads_async, max_over_ranks, plan_heads_lpt,
                                                shard_heads)

    S, HQ, HKV, L, D, B = cfg["seq_len"], cfg["hq"], cfg["hkv"], cfg["layers"], 128, 64
    all_cfgs = layer_configs(cfg)[:L]
    if args.shard == "lpt":  # whole kv groups (or heads) balanced on the patterns' modeled kernel FLOPs
        from paper_2407_02490_b200.patterns import flops_in_kernel

        head_costs = [sum(flops_in_kernel(all_cfgs[layer][h], S, D, B) for layer in range(L)) for h in range(HQ)]
        shards = [plan_heads_lpt(head_costs, HKV, world, r) for r in range(world)]
    else:
        shards = [shard_heads(HQ, HKV, world, r) for r in range(world)]
    shard = shards[rank]
    hq_loc = shard.n_q
    q_idx = torch.tensor(shard.q_heads, dtype=torch.long, device=dev)
    kv_idx = torch.tensor(shard.kv_stack, dtype=torch.long, device=dev)
    cfgs = [[row[h] for h in shard.q_heads] for row in all_cfgs]
    table = PatternTable(cfgs)  # this rank's heads; device head groups cached per layer
    gen = g_local_qkv if cfg["inputs"] == "G-local" else g_iid_qkv

    # ---- inputs resident in HBM (per layer; this rank's kv groups) ----
    Q, K, V = [], [], []
    for layer in range(L):
        q, k, v = gen(HQ, HKV, S, D, seed=1000 * layer, device=dev)
        Q.append(q.index_select(0, q_idx))
        K.append(k.index_select(0, kv_idx))
        V.append(v.index_select(0, kv_idx))
        del q, k, v
    out = torch.empty((hq_loc, S, D), dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    scale = 1.0 / math.sqrt(D)
    lib = _lib.load()
    pair_masks = [_pair_heads(cfgs[layer], dev) for layer in range(L)]  # Block-Sparse heads: paired-box candidates
    est_events, attn_events = [], []
    model = SparsePrefill(table, B)
    layers_qkv = list(zip(Q, K, V))
    outs = [out] * L  # every layer writes the same buffer (stream-ordered)

    def step(record=False):
        # the public model pass (SparsePrefill.prefill): per layer estimation, compaction into the
        # speculatively sized CSR (checked on the device; one read-back per step) and the attention
        # launch; --pipeline overlaps layer l+1's estimation with layer l's attention instead
        pending = []

        def after_layer(layer, o):
            # the optional output all-gather, overlapped with the next layers' compute
            # (at most two exchanges in flight)
            pending.append(gather_heads_async(o, shards))
            if len(pending) > 2:
                pending.pop(0).wait()

        model.prefill(layers_qkv, outs, attn_events if record else None,
                      after_layer if (args.gather and world > 1) else None, pipeline=args.pipeline)
        for pg in pending:
            pg.wait()

    # ---- warm-up + layout statistics (deterministic inputs -> fixed layouts) ----
    step()
    torch.cuda.synchronize()
    n_rows = (S + B - 1) // B
    tiles_tot = chips_tot = union_tot = paired_tot = cols_tot = 0
    area_tot = 0
    pattern_counts = {}
    for layer in range(L):
        lay = P.build_layer_layout(Q[layer], K[layer], cfgs[layer], B)
        tiles_tot += lay.n_tiles
        cols_tot += lay.n_cols
        chips_tot += lay.chips()
        area_tot += int(lay.area().sum().item())
        plist = pair_masks[layer]
        nu, npr = union_steps(lay.tiles.cpu().numpy(), lay.tile_offsets.cpu().numpy(), n_rows, hq_loc,
                              None if plist is None else plist.cpu().numpy())
        union_tot += nu
        paired_tot += npr
        for c in cfgs[layer]:
            pattern_counts[type(c).__name__] = pattern_counts.get(type(c).__name__, 0) + 1
    for _ in range(args.warmup - 1):
        step()
    torch.cuda.synchronize()

    # ---- timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.spf_kernel_launches()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step(record=True)
    t1.record(stream)
    torch.cuda.synchronize()
    launches = lib.spf_kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = max_over_ranks(t0.elapsed_time(t1), device=dev)
    ms_per_step = elapsed / steps
    attn_ms = [a.elapsed_time(b) for a, b in attn_events]
    attn_avg = sum(attn_ms) / len(attn_ms)
    attn_step_ms = sum(attn_ms) / steps
    if not est_events:
        # the pipelined step overlaps estimation with attention: time estimation + compaction
        # alone (serial, every layer, CUDA events) for its roofline, outside the timed region;
        # the median of three passes when there are few layers (one sample is noisy)
        passes = []
        for _ in range(3 if L < 4 else 1):
            evs = []
            for layer in range(L):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                P.build_layer_layout(Q[layer], K[layer], cfgs[layer], B, groups=table.device_groups(layer, dev))
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            passes.append(sum(a.elapsed_time(b) for a, b in evs))
        est_step_ms = sorted(passes)[len(passes) // 2]
    else:
        est_step_ms = sum(a.elapsed_time(b) for a, b in est_events) / steps

    # ---- roofline of the dominant kernel (sparse attention) ----
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    tile_flops = TILE_FLOPS_PER_CELL * D * B * B
    flops_issued_layer = tile_flops * (tiles_tot + chips_tot) / L      # reference-layout algorithmic FLOPs
    achieved_tf = flops_issued_layer / (attn_avg * 1e-3) / 1e12
    # what the M=128 CTAs issue: union step = M128xN64 QK + K64 PV; paired step = N128 QK + K128 PV
    mma_flops_layer = (2 * tile_flops * (union_tot + chips_tot) + 4 * tile_flops * paired_tot) / L
    traffic, traffic_src = None, None
    tpath = os.path.join(REPO, "profiles", "attn_traffic.json")
    if world == 1 and os.path.exists(tpath):  # an ncu capture of this config's full-size (unsharded) launch
        try:
            with open(tpath) as f:
                rec = json.load(f).get(label, {})
            traffic, traffic_src = rec.get("dram_bytes_per_launch"), rec.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(achieved_tf, 2), "peak": tf_sust, "unit": "TFLOP/s",
                "frac": round(achieved_tf / tf_sust, 4), "traffic": traffic,
                "traffic_source": traffic_src if traffic is not None else
                ("omitted: sharded run (the ncu capture is of the full unsharded launch)" if world > 1 else None),
                "frac_of_burst_peak": round(achieved_tf / tf_burst, 4),
                "kernel": ("sparse_attn_pair_kernel<128>" if union_tot + chips_tot == 0 else
                           "sparse_attn_fwd_kernel<128,false>" + (" + sparse_attn_pair_kernel<128>" if paired_tot else "")),
                "peak_source": f"{peak_src} bf16 sustained (burst {tf_burst})",
                "flops_per_launch": flops_issued_layer, "avg_launch_ms": round(attn_avg, 4),
                "mma_flops_per_launch": mma_flops_layer,
                "mma_frac": round(mma_flops_layer / (attn_avg * 1e-3) / 1e12 / tf_sust, 4),
                "attn_share_of_step": round(attn_step_ms / ms_per_step, 4)}
    # ---- estimation + compaction against the HBM roofline (SURVEY 8d "HBM fraction") ----
    bmin = sum(vs_bytes_min(cfgs[layer], S, D, hq_loc, len(set(shard.kv_stack))) for layer in range(L))
    csr_bytes = 4 * (tiles_tot + cols_tot) + L * 2 * 8 * (hq_loc * n_rows + 1)
    est_roof = {"bound": "hbm", "bytes_min_per_step": int(bmin), "csr_bytes_per_step": int(csr_bytes),
                "ms_per_step": round(est_step_ms, 3), "ms_per_layer": round(est_step_ms / L, 4),
                "achieved_gbs": round(bmin / (est_step_ms * 1e-3) / 1e9, 1) if est_step_ms > 0 else None,
                "peak_gbs": hbm, "frac": round(bmin / (est_step_ms * 1e-3) / 1e9 / hbm, 4) if est_step_ms > 0 else None,
                "note": "CUDA events around build_layer_layout (estimation, certification / exact fp64 path, "
                        "index compaction, CSR sizing) on the launch stream, every layer run alone (in the timed "
                        "step it overlaps the previous layer's attention); bytes_min per SURVEY 8(d)"}

    e2e = None
    if with_e2e:
        e2e = run_e2e(args, SparsePrefill(table, B), torch, Q, K, V, L, stream)
        e2e["value"] = round(max_over_ranks(e2e["value"], device=dev), 3)

    dense = None
    if rank == 0 and not args.no_dense:
        dense = dense_baseline(torch, Q[0], K[0], V[0], L, ms_per_step)

    cpu = None
    if rank == 0 and world == 1 and with_cpu:
        cpu = cpu_baseline(cfg, all_cfgs)

    sparsity = 1.0 - area_tot / (L * hq_loc * S * (S + 1) / 2)
    rec = {
        "value": round(ms_per_step, 3), "ms_per_step": round(ms_per_step, 3), "steps": steps,
        "config": {"workload": cfg["workload"], "seq_len": S, "layers": L, "q_heads": HQ, "kv_heads": HKV,
                   "head_dim": D, "block_size": B, "patterns": cfg["patterns"],
                   "pattern_heads_this_rank": pattern_counts, "inputs": cfg["inputs"] + " (SURVEY.md 8d)",
                   "l2": "inputs (%.1f GB) exceed the 126 MB L2; no flush" % (
                       sum(t.numel() * 2 for t in Q + K + V) / 1e9),
                   "parallelism": (f"q-heads sharded over {world} GPU(s) (whole kv groups when {world} "
                                   f"divides {HKV}), no data-path collective" if args.shard == "contiguous" else
                                   f"q-heads sharded over {world} GPU(s) by LPT on modeled kernel FLOPs (whole kv "
                                   f"groups when {world} <= {HKV}), no data-path collective"),
                   "realized_kernel_sparsity": round(sparsity, 4), "tiles": tiles_tot, "column_chips": chips_tot,
                   "union_steps": union_tot, "paired_steps": paired_tot,
                   "output_all_gather": bool(args.gather and world > 1)},
        "roofline": roofline,
        "estimate_roofline": est_roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
        "gpu_launches": int(launches),
        "attention_ms_per_step": round(attn_step_ms, 3),
        "estimate_index_ms_per_step": round(est_step_ms, 3),
        "estimate_index_exposed_ms_per_step": round(ms_per_step - attn_step_ms, 3),
        "layer_pipeline": ("SparsePrefill.prefill(pipeline=True): layer l+1 estimation + compaction on a "
                           "high-priority side stream under layer l's attention") if args.pipeline else
                          ("SparsePrefill.prefill: one stream, CSR sized from the previous step and checked on the "
                           "device (spf_csr_guard), one host read-back per step"),
        "dense_baseline": dense,
    }
    del Q, K, V, out
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=None, help="override layer count (profiling only)")
    ap.add_argument("--ref-rows", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the 1M Vertical-Slash sub-record of the C2 line")
    ap.add_argument("--pipeline", action="store_true",
                    help="time the pipelined model pass (layer l+1's estimation under layer l's attention on a side "
                         "stream); measured equal to the serial step on C2 (494.3 vs 494.7 ms), but the attention "
                         "launches then absorb the estimation kernels' SM time, so the default one-stream pass keeps "
                         "the kernel roofline clean")
    ap.add_argument("--dry-run", action="store_true", help="CPU plumbing check of the rank launch (gloo, no GPU)")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="head chunks (whole kv groups) per layer in the host-buffer pipeline of the e2e leg; "
                         "0 = auto: 1 when the job has several layers (layer l+1's copy hides behind layer l), "
                         "one per kv group for a single layer (C2 1 chunk 1115 ms vs 4: 1138; C4 1: 187 vs 8: 165)")
    ap.add_argument("--shard", default="contiguous", choices=["contiguous", "lpt"],
                    help="q-head partition over ranks: contiguous kv-group ranges, or LPT on modeled kernel FLOPs")
    ap.add_argument("--gather", action="store_true",
                    help="all-gather every layer's per-rank outputs into the full [Hq, S, d] on every rank "
                         "(the optional collective of SURVEY 8e), inside the timed step")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["layers"] = args.layers
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        return dry_run(args, world, rank)

    import torch
    import torch.distributed as dist

    # test hooks for exercising the multi-rank path on a one-GPU box: every rank on GPU 0,
    # gloo for the barriers / max-reduction (the data path has no collective either way)
    if os.environ.get("BENCH_SINGLE_DEVICE") == "1":
        local = 0
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group(backend, **({"device_id": dev} if backend == "nccl" else {}))

    rec = run_config(args, cfg, world, rank, local, dev, with_cpu=not args.no_cpu, with_e2e=not args.no_e2e,
                     steps=args.steps, label=args.config)
    c3 = None
    if args.config == "c2" and not args.no_c3 and not args.layers:
        # the 1M Vertical-Slash headline (C3) in the same run, sharded the same way
        c3cfg = dict(CONFIGS["c3"])
        c3 = run_config(args, c3cfg, world, rank, local, dev, with_cpu=False, with_e2e=not args.no_e2e,
                        steps=min(args.steps, 5), label="c3")
        c3 = {"metric": metric_name(argparse.Namespace(config="c3"), c3cfg), "unit": "ms", **c3}
        if c3.get("dense_baseline") and "ms_per_layer" in c3["dense_baseline"]:
            c3["speedup_vs_dense_device"] = round(c3["dense_baseline"]["ms_per_layer"] / c3["ms_per_step"], 2)
            if c3.get("e2e"):
                c3["speedup_vs_dense_e2e"] = round(c3["dense_baseline"]["ms_per_layer"] / c3["e2e"]["value"], 2)

    if rank == 0:
        line = {"metric": metric_name(args, cfg), "value": rec["value"], "unit": "ms", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic"}
        line.update({k: v for k, v in rec.items() if k not in ("value", "ms_per_step", "steps")})
        if c3 is not None:
            line["c3_1m"] = c3
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, model, torch, Q, K, V, L, stream):
    """Public API with host buffers: driver.SparsePrefill.prefill_host -- per (layer, head
    chunk) unit, H2D of Q/K/V from pinned host memory on a copy stream (unit u+1 while
    unit u computes), the layer's estimation, compaction and attention for the chunk's
    heads, and D2H of its output into pinned host memory on a third stream."""
    slots = 2  # pinned host inputs for two layers, reused round-robin (host RAM)
    host_q = [Q[i % L].cpu().pin_memory() for i in range(slots)]
    host_k = [K[i % L].cpu().pin_memory() for i in range(slots)]
    host_v = [V[i % L].cpu().pin_memory() for i in range(slots)]
    host_o = [torch.empty_like(host_q[0]).pin_memory() for _ in range(slots)]
    host_layers = [(host_q[layer % slots], host_k[layer % slots], host_v[layer % slots]) for layer in range(L)]
    host_out = [host_o[layer % slots] for layer in range(L)]
    comp = stream
    chunks = args.e2e_chunks if args.e2e_chunks > 0 else (1 if L > 2 else K[0].shape[0])

    def one_step():
        model.prefill_host(host_layers, host_out, chunks=chunks)

    one_step()
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    for _ in range(n):
        one_step()
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    h2d_bytes = L * (Q[0].numel() + K[0].numel() + V[0].numel()) * 2
    d2h_bytes = L * Q[0].numel() * 2
    return {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d_bytes),
            "d2h_bytes_per_step": int(d2h_bytes), "steps": n, "head_chunks": chunks,
            "note": "public API driver.SparsePrefill.prefill_host: pinned host buffers (inputs of two layers reused "
                    "round-robin), per (layer, kv-group chunk) H2D on one stream overlapping the previous unit's "
                    "estimation + attention and the D2H of the one before on another"}


def dense_baseline(torch, q, k, v, L, ms_per_step):
    import torch.nn.functional as F

    from torch.nn.attention import SDPBackend, sdpa_kernel

    rep = q.shape[0] // k.shape[0]
    qq = q.unsqueeze(0)
    kk = k.repeat_interleave(rep, dim=0).unsqueeze(0)
    vv = v.repeat_interleave(rep, dim=0).unsqueeze(0)
    try:
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION]):
            F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    except Exception as ex:  # pragma: no cover
        return {"error": str(ex)[:200]}
    finally:
        del kk, vv
    hq, s, d = q.shape
    flops = 4 * d * hq * s * (s + 1) / 2
    return {"impl": "torch.nn.functional.scaled_dot_product_attention(is_causal, enable_gqa) bf16",
            "ms_per_layer": round(ms, 3), "ms_per_step_est": round(ms * L, 3),
            "tflops": round(flops / (ms * 1e-3) / 1e12, 1), "speedup_sparse_vs_dense": round(ms * L / ms_per_step, 3)}


def cpu_baseline(cfg, all_cfgs):
    from benchmarks import cpu_reference

    cores = os.cpu_count() or 1
    t0 = time.time()
    step_s, info = cpu_reference.run_sample(all_cfgs, cfg["seq_len"], 128, 64, cores,
                                            items_per_pattern=max(1, min(cores, 2)), n_sample_rows=16)
    return {"value": round(step_s * 1e3, 3), "unit": "ms", "cores": cores,
            "kind": "reference" if info["ref_kernel"] else "port",
            "sample": f"{info['items']} (layer, head) items of {cfg['workload']} (full estimation + index, kernel on "
                      f"16 sampled row blocks extrapolated by tiles+chips; code = {info['impl']}); "
                      f"step = sum(item s)/cores; sampled in {time.time() - t0:.1f}s wall",
            "patterns": info["patterns"]}


if __name__ == "__main__":
    main()
