"""Column-chip path cost: a column-heavy Vertical-Slash layout
(many verticals, few slashes) vs the tile-only layout of the same heads, per kernel step.

    python benchmarks/bench_columns.py [--seq 32768] [--hq 16] [--hkv 4] [--kv 2000] [--ks 64]

Reports attention ms, tiles, column chips and the per-step cost of each kind
(least squares over the two layouts: t = a * tile_steps + b * chip_steps)."""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--hq", type=int, default=16)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--kv", type=int, default=2000)
    ap.add_argument("--ks", type=int, default=64)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_2407_02490_b200 as P
    from benchmarks.workloads import g_iid_qkv
    from paper_2407_02490_b200 import kernels

    q, k, v = g_iid_qkv(args.hq, args.hkv, args.seq, 128, seed=3, device="cuda")
    res = {"seq": args.seq, "hq": args.hq, "hkv": args.hkv}
    out = torch.empty_like(q)

    def timed(lay):
        f = lambda: kernels.sparse_flash_attention_gpu(q, k, v, 128 ** -0.5, 64, lay.tiles, lay.tile_offsets,
                                                       lay.cols, lay.col_offsets, out=out)
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for name, cfg in (("columns", P.VerticalSlash(args.kv, args.ks)), ("tiles", P.AShape(64, args.kv))):
        lay = P.build_layer_layout(q, k, [cfg] * args.hq, 64)
        res[name] = {"cfg": repr(cfg), "attention_ms": round(timed(lay), 4), "tiles": lay.n_tiles,
                     "columns": lay.n_cols, "column_chips": lay.chips()}
    c, t = res["columns"], res["tiles"]
    # two equations, two unknowns: ms per tile step and per column chip (128-row CTAs see both row
    # blocks' union, so these are per-(64-row block) step equivalents)
    import numpy as np

    a = np.array([[c["tiles"], c["column_chips"]], [t["tiles"], t["column_chips"]]], dtype=np.float64)
    b = np.array([c["attention_ms"], t["attention_ms"]])
    try:
        per_tile, per_chip = np.linalg.solve(a, b) if abs(np.linalg.det(a)) > 0 else (t["attention_ms"] / max(1, t["tiles"]), float("nan"))
    except np.linalg.LinAlgError:
        per_tile, per_chip = float("nan"), float("nan")
    res["us_per_tile"] = round(float(per_tile) * 1e3, 6)
    res["us_per_chip"] = round(float(per_chip) * 1e3, 6)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
