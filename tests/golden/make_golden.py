"""Generate the golden parity fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    make -C oracle            # builds oracle/_ref/spf_ref_core (reference _core.pyx)
    python tests/golden/make_golden.py

The reference package is imported from /root/reference/pkg/src; its compiled
Cython kernel is the one oracle/Makefile built from /root/reference
(registered as ``sparseprefill._core`` so ``kernels.py`` picks the Cython
backend exactly as an installed copy would, kernels.py:17-25).

Inputs are regenerated from seeds by ``oracle.port.seeded_gaussian`` (the
reference's tensor.py:81-90 generator) and pinned with a SHA-256 so a numpy
generator drift is detected; only small planted inputs are stored verbatim.
Outputs stored: index sets, score vectors, CSR layouts and attention outputs.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import port  # noqa: E402

ref_core = port.load_ref_core()
if ref_core is not None:
    sys.modules["sparseprefill._core"] = ref_core

import sparseprefill  # noqa: E402
from sparseprefill import kernels  # noqa: E402
from sparseprefill.attention_ref import AttentionInputs  # noqa: E402
from sparseprefill.estimator import estimate_block_sparse, estimate_vertical_slash  # noqa: E402
from sparseprefill.patterns import AShape, BlockSparse, VerticalSlash, a_shape_layout, layout_area  # noqa: E402
from sparseprefill.sparse_attn import block_indices_to_layout  # noqa: E402
from sparseprefill.vs_index import build_vs_layout_with_stats  # noqa: E402
from sparseprefill.workload import PlantedLine, WorkloadSpec, synth_planted_qkv  # noqa: E402


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (nearest-even), returned as fp32 (exact)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def gaussian_qkv(s, d, seed, bf16):
    q = port.seeded_gaussian(s, d, seed)
    k = port.seeded_gaussian(s, d, seed + 1)
    v = port.seeded_gaussian(s, d, seed + 2)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v


def digest(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sample_rows(s, b, out):
    """Keep every row for small S; at S >= 2048 keep 8 evenly spaced row
    blocks (first and last included) so the fixture stays small."""
    n = (s + b - 1) // b
    if s < 2048:
        blocks = np.arange(n)
    else:
        blocks = np.unique(np.linspace(0, n - 1, 8).round().astype(np.int64))
    rows = np.concatenate([np.arange(r * b, min(r * b + b, s)) for r in blocks])
    return blocks, out[rows]


def csr(per_row):
    flat, off = kernels._flatten(per_row, len(per_row))
    return flat, off


def main():
    out = {}
    print("reference backend:", kernels.BACKEND, sparseprefill.__version__)
    out["meta_backend"] = np.array(kernels.BACKEND)

    # ---- Vertical-Slash: estimation + merge + kernel --------------------------------
    vs_cases = [
        # name, S, d, k_v, k_s, last_q, seed, bf16, B
        ("vs_s8k_d128_bf16", 8192, 128, 1000, 6096, 64, 11, True, 64),
        ("vs_s8k_d128_sparse", 8192, 128, 64, 256, 64, 12, True, 64),
        ("vs_s4k_d64_f32", 4096, 64, 100, 300, 64, 13, False, 64),
        ("vs_s1000_d128_odd", 1000, 128, 30, 70, 64, 14, True, 64),
        ("vs_s257_d16_b16", 257, 16, 5, 4, 16, 15, False, 16),
        ("vs_s95_d16_b16", 95, 16, 4, 4, 16, 8, False, 16),
        ("vs_s64_d16_clip", 64, 16, 100, 100, 32, 16, False, 16),
    ]
    for name, s, d, kv, ks, lq, seed, bf16, b in vs_cases:
        q, k, v = gaussian_qkv(s, d, seed, bf16)
        idx = estimate_vertical_slash(q, k, VerticalSlash(kv, ks, lq))
        vert_score, slash_score = port.vs_scores(q, k, lq)
        layout, ops = build_vs_layout_with_stats(idx, s, b)
        ts, to = csr(layout.block_starts)
        cs, co = csr(layout.column_indices)
        inp = AttentionInputs(q, k, v)
        want = kernels.sparse_flash_attention(q, k, v, inp.scale, b, layout.block_starts, layout.column_indices)
        out[f"{name}__params"] = np.array([s, d, kv, ks, lq, seed, int(bf16), b], np.int64)
        out[f"{name}__digest"] = np.array(digest(q, k, v))
        out[f"{name}__vertical"] = idx.vertical
        out[f"{name}__slash"] = idx.slash
        out[f"{name}__vscore"] = vert_score
        out[f"{name}__sscore"] = slash_score
        out[f"{name}__tiles"], out[f"{name}__tile_off"] = ts, to
        out[f"{name}__cols"], out[f"{name}__col_off"] = cs, co
        out[f"{name}__ops"] = np.asarray(ops, np.int64)
        out[f"{name}__area"] = np.array(layout_area(layout), np.int64)
        out[f"{name}__out_blocks"], out[f"{name}__out"] = sample_rows(s, b, want)
        print(name, "tiles", ts.size, "cols", cs.size, "area", layout_area(layout))

    # ---- Block-Sparse -----------------------------------------------------------
    bs_cases = [
        ("bs_s8k_d128_bf16", 8192, 128, 100, 64, 21, True),
        ("bs_s4k_d128_k8", 4096, 128, 8, 64, 22, True),
        ("bs_s1000_d64_f32", 1000, 64, 5, 64, 23, False),
        ("bs_s257_d16_b16", 257, 16, 3, 16, 24, False),
    ]
    for name, s, d, kb, b, seed, bf16 in bs_cases:
        q, k, v = gaussian_qkv(s, d, seed, bf16)
        blocks = estimate_block_sparse(q, k, BlockSparse(kb, b))
        layout = block_indices_to_layout(blocks, s, b)
        ts, to = csr(layout.block_starts)
        inp = AttentionInputs(q, k, v)
        want = kernels.sparse_flash_attention(q, k, v, inp.scale, b, layout.block_starts, layout.column_indices)
        out[f"{name}__params"] = np.array([s, d, kb, b, seed, int(bf16)], np.int64)
        out[f"{name}__digest"] = np.array(digest(q, k, v))
        out[f"{name}__tiles"], out[f"{name}__tile_off"] = ts, to
        out[f"{name}__out_blocks"], out[f"{name}__out"] = sample_rows(s, b, want)
        out[f"{name}__area"] = np.array(layout_area(layout), np.int64)
        print(name, "tiles", ts.size)

    # ---- A-shape ----------------------------------------------------------------
    as_cases = [
        ("as_s8k_d128_bf16", 8192, 128, 128, 4096, 64, 31, True),
        ("as_s2k_d128_g1024", 2048, 128, 1024, 512, 64, 32, True),
        ("as_s100_d16_b64", 100, 16, 8, 16, 64, 33, False),
        ("as_s17_d16_b4", 17, 16, 8, 16, 4, 34, False),
    ]
    for name, s, d, g, w, b, seed, bf16 in as_cases:
        q, k, v = gaussian_qkv(s, d, seed, bf16)
        layout = a_shape_layout(s, AShape(g, w), b)
        ts, to = csr(layout.block_starts)
        inp = AttentionInputs(q, k, v)
        want = kernels.sparse_flash_attention(q, k, v, inp.scale, b, layout.block_starts, layout.column_indices)
        out[f"{name}__params"] = np.array([s, d, g, w, b, seed, int(bf16)], np.int64)
        out[f"{name}__digest"] = np.array(digest(q, k, v))
        out[f"{name}__tiles"], out[f"{name}__tile_off"] = ts, to
        out[f"{name}__out_blocks"], out[f"{name}__out"] = sample_rows(s, b, want)
        out[f"{name}__area"] = np.array(layout_area(layout), np.int64)
        print(name, "tiles", ts.size)

    # ---- planted workload (estimator recall; inputs stored verbatim) -------------
    spec = WorkloadSpec(512, 64, seed=5, planted=(
        PlantedLine("vertical", 12.0, column=137), PlantedLine("slash", 12.0, offset=33)))
    inp = synth_planted_qkv(spec)
    idx = estimate_vertical_slash(inp.q, inp.k, VerticalSlash(4, 4, 64))
    blocks = estimate_block_sparse(inp.q, inp.k, BlockSparse(2, 64))
    out["planted__q"], out["planted__k"], out["planted__v"] = inp.q, inp.k, inp.v
    out["planted__vertical"], out["planted__slash"] = idx.vertical, idx.slash
    bt, bo = csr([[b * 64 for b in row] for row in blocks.rows])
    out["planted__bs_tiles"], out["planted__bs_off"] = bt, bo

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
