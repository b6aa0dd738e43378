"""Small-shape run of every libspf kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python benchmarks/sanitize_smoke.py
    compute-sanitizer --tool racecheck python benchmarks/sanitize_smoke.py
    compute-sanitizer --tool synccheck python benchmarks/sanitize_smoke.py

VS (fast + exact estimation, merge), A-shape and BS layouts, the bf16 attention
kernel over a mixed layer (incl. the log-sum-exp output) and the fp32 (split)
attention path, at S = 1000 / 2048 so the tools finish in minutes."""

import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2407_02490_b200 as P
from paper_2407_02490_b200 import kernels
from paper_2407_02490_b200.estimator import vs_estimate_async


def main():
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    s, d, hq, hkv = 2048, 128, 4, 2
    q, k, v = (torch.randn(h, s, d, generator=g, device=dev).to(torch.bfloat16) for h in (hq, hkv, hkv))
    cfg = P.VerticalSlash(64, 256)
    vs_estimate_async(q, k, cfg, mode="fast")
    vs_estimate_async(q, k, cfg, mode="exact")
    cfgs = [P.VerticalSlash(64, 256), P.AShape(64, 512), P.BlockSparse(8), P.VerticalSlash(16, 64, 32)]
    out, lay = P.sparse_prefill_attention(q, k, v, cfgs, 64, return_layout=True)
    lse = torch.empty(hq, s, dtype=torch.float32, device=dev)
    kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), 64, lay.tiles, lay.tile_offsets, lay.cols,
                                       lay.col_offsets, lse=lse)
    # paired-box kernel for the Block-Sparse head, union kernel for the rest (one call)
    pair = torch.tensor([0, 0, 1, 0], dtype=torch.uint8, device=dev)
    kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), 64, lay.tiles, lay.tile_offsets, lay.cols,
                                       lay.col_offsets, pair_heads=pair)
    P.argtopk(torch.randn(5000, generator=g, device=dev).double().cpu().numpy(), 300)
    qf, kf, vf = (x[:, :1000].float().contiguous() for x in (q, k, v))
    lay32 = P.build_layer_layout(qf, kf, [P.VerticalSlash(32, 128)] * hq, 64)
    kernels.sparse_flash_attention_gpu(qf, kf, vf, 1 / math.sqrt(d), 64, lay32.tiles, lay32.tile_offsets,
                                       lay32.cols, lay32.col_offsets)
    # round-2 paths: G-local heads (rigorous bound -> the DMMA fp64 fallback), a column-heavy
    # layout (cp.async chip gathers), the speculative model pass with an overflow (CSR guard),
    # Block-Sparse pooled scores on DMMA (even block count)
    from benchmarks.workloads import g_local_qkv
    from paper_2407_02490_b200.driver import PatternTable, SparsePrefill

    ql, kl, vl = g_local_qkv(hq, hkv, s, d, seed=1, device=dev)
    vs_estimate_async(ql, kl, P.VerticalSlash(100, 300), mode="fast")
    lay_c = P.build_layer_layout(q, k, [P.VerticalSlash(600, 16)] * hq, 64)
    kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), 64, lay_c.tiles, lay_c.tile_offsets, lay_c.cols,
                                       lay_c.col_offsets)
    model = SparsePrefill(PatternTable([cfgs, [P.BlockSparse(6)] * hq]))
    model.prefill([(q, k, v), (ql, kl, vl)])
    model._caps = {key: (5, 3) for key in model._caps}
    model.prefill([(q, k, v), (ql, kl, vl)])
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out).all()) and bool(torch.isfinite(lse).all())
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
