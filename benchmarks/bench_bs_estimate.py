"""Device time of Block-Sparse estimation (pool -> pooled scores -> row softmax/top-k) for
one layer, the C4 shape by default (256K tokens, 56 q / 8 kv heads, BS(100), G-iid).

    python benchmarks/bench_bs_estimate.py [--seq 262144] [--hq 56] [--hkv 8] [--reps 5]

CUDA events on the launching stream, median of --reps after one warm-up; also prints
a checksum of the tile starts so two builds can be compared for identical output.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=262144)
    ap.add_argument("--hq", type=int, default=56)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--kb", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from benchmarks.workloads import g_iid_qkv
    from paper_2407_02490_b200 import estimator, layouts
    from paper_2407_02490_b200.patterns import BlockSparse

    q, k, _ = g_iid_qkv(args.hq, args.hkv, args.seq, 128, seed=4)
    cfg = BlockSparse(args.kb)
    b = cfg.block_size
    n = (args.seq + b - 1) // b
    cnt = torch.zeros(args.hq * n, dtype=torch.int64, device="cuda")
    layouts.bs_count(None, args.hq, args.seq, b, cfg.k_b, cnt)
    offs = torch.zeros(args.hq * n + 1, dtype=torch.int64, device="cuda")
    offs[1:] = torch.cumsum(cnt, 0)
    starts = torch.empty(int(offs[-1].item()), dtype=torch.int32, device="cuda")
    ts = []
    for r in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        estimator.estimate_block_sparse_gpu(q, k, cfg, None, offs, starts)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    chk = int((starts.to(torch.int64) * torch.arange(1, starts.numel() + 1, device="cuda") % 1000003).sum().item())
    print(json.dumps({"seq": args.seq, "hq": args.hq, "bs_estimate_ms": round(statistics.median(ts), 3),
                      "tiles": starts.numel(), "checksum": chk}))


if __name__ == "__main__":
    main()
