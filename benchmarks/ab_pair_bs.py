"""Interleaved timing of a Block-Sparse layer (BS(100), G-iid) through the union kernel and the
paired-box kernel (spf_sparse_flash_rows_ex pair_heads).  S / HQ env: sequence length, q-heads."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_02490_b200 as P
from paper_2407_02490_b200 import kernels
from benchmarks.workloads import g_iid_qkv, g_local_qkv
S = int(os.environ.get("S", "262144")); HQ = int(os.environ.get("HQ", "56")); HKV = 8
q, k, v = g_iid_qkv(HQ, HKV, S, 128, seed=0, device="cuda")
lay = P.build_layer_layout(q, k, [P.BlockSparse(100)] * HQ, 64)
out = torch.empty_like(q)
mask = torch.ones(HQ, dtype=torch.uint8, device="cuda")
ts = [[], []]
for r in range(8):
    for i, pm in enumerate((None, mask)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kernels.sparse_flash_attention_gpu(q, k, v, 128 ** -0.5, 64, lay.tiles, lay.tile_offsets, lay.cols, lay.col_offsets, out=out, pair_heads=pm)
        e1.record(); torch.cuda.synchronize()
        if r >= 2: ts[i].append(e0.elapsed_time(e1))
a, b = statistics.median(ts[0]), statistics.median(ts[1])
tiles = lay.n_tiles
flops = 4 * 128 * 64 * 64 * tiles
print("S=%d BS(100): union %.2f ms (%.0f TF/s)  pair %.2f ms (%.0f TF/s)  pair/union %.3f" % (S, a, flops / a / 1e9, b, flops / b / 1e9, b / a))
