"""Production entry: one layer of dynamic sparse pre-fill attention on a B200.

``sparse_prefill_attention(q, k, v, head_cfgs)`` runs, for a whole layer of
q-heads with per-head pattern configs (patterns.py:23-57, as loaded from the
config JSON v1 of patterns.py:236-266), the hot path of the reference's
``run_head`` (sparse_attn.py:67-94) for every head at once:

  1. online estimation      VS heads grouped by (k_v, k_s, last_q): spf_vs_estimate
                            on the tensor cores; heads whose top-k boundary is
                            too close for its error model are re-run on the
                            fp64 path inside the same stream-ordered call
  2. index compaction       per-row counts for VS / A-shape / BS heads -> one
                            CSR over all q-heads (spf_*_layout_count,
                            spf_csr_offsets, spf_*_layout_fill); BS heads'
                            pooled estimation writes its tiles directly
  3. sparse attention       ONE launch of the sm_100a kernel over all heads
                            and patterns (GQA head map), bf16 I/O.

Everything stays on the device; the only host sync is the read-back of the
two CSR totals needed to size the layout.
"""

from __future__ import annotations

import math
from collections import OrderedDict
from dataclasses import dataclass

import torch

from . import _dev, kernels, layouts
from .estimator import estimate_block_sparse_gpu, vs_estimate_async
from .patterns import AShape, BlockSparse, HeadPatternConfig, VerticalSlash, n_block_rows


@dataclass
class LayerLayout:
    """Device CSR over (q-head, query-block row) for one layer."""

    seq_len: int
    block_size: int
    n_heads: int
    tiles: torch.Tensor
    tile_offsets: torch.Tensor
    cols: torch.Tensor
    col_offsets: torch.Tensor

    @property
    def n_tiles(self) -> int:
        return int(self.tiles.numel())

    @property
    def n_cols(self) -> int:
        return int(self.cols.numel())

    def chips(self) -> int:
        """Column chips of B per row, summed (the kernel's gathered steps)."""
        per_row = self.col_offsets[1:] - self.col_offsets[:-1]
        return int(((per_row + self.block_size - 1) // self.block_size).sum().item())

    def area(self) -> torch.Tensor:
        """Per-head computed-cell area (patterns.py:147-184)."""
        return layouts.layout_area_dev(self.n_heads, self.seq_len, self.block_size, self.tiles, self.tile_offsets,
                                       self.col_offsets)

    def head_rows(self, h: int):
        n = n_block_rows(self.seq_len, self.block_size)
        return self.tile_offsets[h * n: (h + 1) * n + 1], self.col_offsets[h * n: (h + 1) * n + 1]


def _group_heads(head_cfgs, device):
    groups: "OrderedDict[HeadPatternConfig, list[int]]" = OrderedDict()
    for h, cfg in enumerate(head_cfgs):
        if not isinstance(cfg, (AShape, VerticalSlash, BlockSparse)):
            raise TypeError(f"unknown pattern config: {cfg!r}")
        groups.setdefault(cfg, []).append(h)
    return [(cfg, torch.tensor(ids, dtype=torch.int32, device=device), len(ids)) for cfg, ids in groups.items()]


def build_layer_layout(q: torch.Tensor, k: torch.Tensor, head_cfgs, block_size: int = 64,
                       stream=None, groups=None) -> LayerLayout:
    """Estimation + index compaction for every head of a layer (steps 1-2).

    ``groups`` may pass the layer's precomputed device head groups
    (driver.PatternTable.device_groups) instead of regrouping ``head_cfgs``.  With a
    ``stream``, every allocation, kernel and copy of the layer is ordered on it."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return _build_layer_layout(q, k, head_cfgs, block_size, stream, groups)
    return _build_layer_layout(q, k, head_cfgs, block_size, None, groups)


def _layout_counts(q, k, head_cfgs, block_size, stream, groups):
    """Estimation + per-row counts + the two CSR scans (device only, no host sync)."""
    dev = _dev.require_cuda(q.device)
    hq, s_len, _ = q.shape
    if len(head_cfgs) != hq:
        raise ValueError(f"need one pattern config per q-head ({len(head_cfgs)} != {hq})")
    for cfg in head_cfgs:
        if isinstance(cfg, BlockSparse) and cfg.block_size != block_size:
            raise ValueError("all heads of a layer must share one block size "
                             f"(BlockSparse block_size {cfg.block_size} != {block_size})")
    if groups is None:
        groups = _group_heads(head_cfgs, dev)
    n = n_block_rows(s_len, block_size)
    tc = torch.zeros(hq * n, dtype=torch.int64, device=dev)
    cc = torch.zeros(hq * n, dtype=torch.int64, device=dev)
    vs_sel = {}
    for cfg, ids, m in groups:
        if isinstance(cfg, VerticalSlash):
            vert, sl, _, _, _ = vs_estimate_async(q, k, cfg, ids, mode="fast", stream=stream)
            vs_sel[cfg] = (vert, sl)
            layouts.vs_count(vert, sl, ids, s_len, block_size, tc, cc, stream)
        elif isinstance(cfg, AShape):
            layouts.ashape_count(ids, m, s_len, block_size, cfg, tc, stream)
        else:
            layouts.bs_count(ids, m, s_len, block_size, cfg.k_b, tc, stream)
    toff, _ = layouts.csr_offsets(tc, stream, want_total=False)
    coff, _ = layouts.csr_offsets(cc, stream, want_total=False)
    return dict(groups=groups, vs_sel=vs_sel, toff=toff, coff=coff, s_len=s_len, hq=hq)


def _layout_fill(q, k, ctx, block_size, tiles, cols, stream):
    s_len = ctx["s_len"]
    for cfg, ids, m in ctx["groups"]:
        if isinstance(cfg, VerticalSlash):
            vert, sl = ctx["vs_sel"][cfg]
            layouts.vs_fill(vert, sl, ids, s_len, block_size, ctx["toff"], ctx["coff"], tiles, cols, stream)
        elif isinstance(cfg, AShape):
            layouts.ashape_fill(ids, m, s_len, block_size, cfg, ctx["toff"], tiles, stream)
        else:
            estimate_block_sparse_gpu(q, k, cfg, ids, ctx["toff"], tiles, stream)


def _build_layer_layout(q, k, head_cfgs, block_size, stream, groups) -> LayerLayout:
    dev = _dev.require_cuda(q.device)
    ctx = _layout_counts(q, k, head_cfgs, block_size, stream, groups)
    toff, coff = ctx["toff"], ctx["coff"]
    totals = torch.stack([toff[-1], coff[-1]]).cpu()  # the host read-back that sizes the layout
    nt, nc = int(totals[0]), int(totals[1])
    tiles = torch.empty(max(nt, 1), dtype=torch.int32, device=dev)
    cols = torch.empty(max(nc, 1), dtype=torch.int32, device=dev)
    _layout_fill(q, k, ctx, block_size, tiles, cols, stream)
    return LayerLayout(ctx["s_len"], block_size, ctx["hq"], tiles[:nt], toff, cols[:nc], coff)


def build_layer_layout_into(q, k, head_cfgs, block_size, tiles_buf, cols_buf, overflow, totals, stream=None,
                            groups=None):
    """Estimation + compaction into caller-owned buffers of fixed capacity, with no host
    sync: ``spf_csr_guard`` compares the totals with the capacities on the device and, if
    they do not fit, empties every row (nothing is written past a buffer; the attention
    then yields zero rows) and sets ``overflow`` (an int32 device scalar), while
    ``totals`` (int64 [2] on the device) receives the true sizes.  The caller checks the
    flag later and redoes an overflowed layer with ``build_layer_layout``."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return build_layer_layout_into(q, k, head_cfgs, block_size, tiles_buf, cols_buf, overflow, totals, None,
                                           groups)
    ctx = _layout_counts(q, k, head_cfgs, block_size, None, groups)
    layouts.csr_guard(ctx["toff"], ctx["coff"], tiles_buf.numel(), cols_buf.numel(), overflow, totals)
    _layout_fill(q, k, ctx, block_size, tiles_buf, cols_buf, None)
    return LayerLayout(ctx["s_len"], block_size, ctx["hq"], tiles_buf, ctx["toff"], cols_buf, ctx["coff"])


_PAIR_CACHE: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()


def _pair_heads(head_cfgs, device):
    """Device int32 list of the Block-Sparse heads (no residual columns, row blocks that
    rarely share tiles): the attention runs them with the paired-box kernel."""
    key = (str(device), tuple(isinstance(c, BlockSparse) for c in head_cfgs))
    if not any(key[1]):
        return None
    m = _PAIR_CACHE.get(key)
    if m is None:
        m = torch.tensor([h for h, bs in enumerate(key[1]) if bs], dtype=torch.int32, device=device)
        _PAIR_CACHE[key] = m
        if len(_PAIR_CACHE) > 64:
            _PAIR_CACHE.popitem(last=False)
    return m


def sparse_prefill_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, head_cfgs, block_size: int = 64,
                             scale: float | None = None, out: torch.Tensor | None = None, stream=None,
                             return_layout: bool = False, groups=None):
    """Full layer: q [Hq, S, d], k/v [Hkv, S, d] (bf16) -> out [Hq, S, d]."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return sparse_prefill_attention(q, k, v, head_cfgs, block_size, scale, out, None, return_layout, groups)
    layout = build_layer_layout(q, k, head_cfgs, block_size, stream, groups)
    d = q.shape[-1]
    sc = 1.0 / math.sqrt(d) if scale is None else float(scale)
    out = kernels.sparse_flash_attention_gpu(q, k, v, sc, block_size, layout.tiles, layout.tile_offsets,
                                             layout.cols, layout.col_offsets, out=out, stream=stream,
                                             pair_heads=_pair_heads(head_cfgs, q.device))
    return (out, layout) if return_layout else out
