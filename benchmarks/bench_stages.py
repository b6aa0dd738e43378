"""Per-stage device timing of one layer (estimation / index compaction / attention).

    python benchmarks/bench_stages.py [--seq 131072] [--hq 32] [--hkv 8] [--gen local|iid] [--reps 10]

CUDA events on the launching stream, median of --reps after warm-up; the
inputs are regenerated per layer seed so the K tiles are not L2-resident.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps, torch):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--gen", default="local")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--exact", action="store_true", help="also time the fp64 estimation path")
    args = ap.parse_args()
    import torch

    import paper_2407_02490_b200 as P
    from benchmarks.workloads import g_iid_qkv, g_local_qkv
    from paper_2407_02490_b200 import kernels, layouts
    from paper_2407_02490_b200.estimator import vs_estimate_async

    gen = g_local_qkv if args.gen == "local" else g_iid_qkv
    q, k, v = gen(args.hq, args.hkv, args.seq, 128, seed=0, device="cuda")
    cfg = P.VerticalSlash(1000, 6096, 64)
    cfgs = [cfg] * args.hq
    res = {"seq": args.seq, "hq": args.hq, "hkv": args.hkv, "gen": args.gen}
    for _ in range(3):
        vs_estimate_async(q, k, cfg, mode="fast")
    torch.cuda.synchronize()
    res["estimate_fast_ms"] = timed(lambda: vs_estimate_async(q, k, cfg, mode="fast"), args.reps, torch)
    vert, sl, _, _, flags = vs_estimate_async(q, k, cfg, mode="fast")
    res["uncertain_heads"] = int(flags.sum().item())
    if args.exact:
        res["estimate_exact_ms"] = timed(lambda: vs_estimate_async(q, k, cfg, mode="exact"), max(2, args.reps // 5),
                                         torch)
        ve, se, _, _, _ = vs_estimate_async(q, k, cfg, mode="exact")
        res["fast_equals_exact_heads"] = int(sum(bool(torch.equal(vert[h], ve[h]) and torch.equal(sl[h], se[h]))
                                                 for h in range(args.hq)))
    n = (args.seq + 63) // 64
    tc = torch.zeros(args.hq * n, dtype=torch.int64, device="cuda")
    cc = torch.zeros_like(tc)
    res["vs_count_ms"] = timed(lambda: layouts.vs_count(vert, sl, None, args.seq, 64, tc, cc), args.reps, torch)
    toff, nt = layouts.csr_offsets(tc)
    coff, nc = layouts.csr_offsets(cc)
    tiles = torch.empty(max(nt, 1), dtype=torch.int32, device="cuda")
    cols = torch.empty(max(nc, 1), dtype=torch.int32, device="cuda")
    res["vs_fill_ms"] = timed(lambda: layouts.vs_fill(vert, sl, None, args.seq, 64, toff, coff, tiles, cols),
                              args.reps, torch)
    res["build_layer_layout_ms"] = timed(lambda: P.build_layer_layout(q, k, cfgs, 64), args.reps, torch)
    lay = P.build_layer_layout(q, k, cfgs, 64)
    out = torch.empty_like(q)
    res["attention_ms"] = timed(lambda: kernels.sparse_flash_attention_gpu(
        q, k, v, 128 ** -0.5, 64, lay.tiles, lay.tile_offsets, lay.cols, lay.col_offsets, out=out), args.reps, torch)
    res["tiles"] = lay.n_tiles
    res["chips"] = lay.chips()
    # estimation roofline: K read once per pass (two passes), Q tail, score vectors written + read by top-k
    kbytes = args.hkv * args.seq * 128 * 2
    res["estimate_bytes_min"] = kbytes + args.hq * 64 * 128 * 2 + args.hq * args.seq * 8 * 2 * 2
    res["estimate_gbs_min"] = res["estimate_bytes_min"] / (res["estimate_fast_ms"] * 1e-3) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
