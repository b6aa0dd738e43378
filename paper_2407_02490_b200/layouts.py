"""GPU index compaction: CSR layouts for the three patterns (libspf wrappers).

Device-level API used by the production pipeline (``prefill.py``) plus the
host-facing builders behind the drop-in functions ``patterns.a_shape_layout``,
``vs_index.build_vs_layout`` and ``patterns.layout_area``.

CSR convention (include/spf.h): rows are (head, query-block row) with
row = h * n_rows + r; offsets int64 [H * n_rows + 1]; entries int32.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _dev, _lib
from .patterns import AShape, SparseLayout, n_block_rows


def _i64_host():
    return (ctypes.c_int64 * 1)()


def csr_offsets(counts: torch.Tensor, stream=None, want_total: bool = True):
    """Exclusive scan of int64 row counts -> (offsets [n+1], total or None)."""
    lib = _lib.load()
    n = counts.numel()
    offsets = torch.empty(n + 1, dtype=torch.int64, device=counts.device)
    ws_bytes = lib.spf_scan_workspace_size(n)
    ws = _dev.workspace(ws_bytes, counts.device, stream)
    total = _i64_host() if want_total else None
    _lib.check(lib.spf_csr_offsets(_dev.ptr(counts), n, _dev.ptr(offsets), total, _dev.ptr(ws), ws_bytes,
                                   _dev.stream_handle(stream)), "spf_csr_offsets")
    return offsets, (int(total[0]) if want_total else None)


def csr_guard(tile_offsets: torch.Tensor, col_offsets: torch.Tensor, cap_tiles: int, cap_cols: int,
              overflow: torch.Tensor, totals: torch.Tensor, stream=None):
    """spf_csr_guard: speculative CSR sizing checked on the device (see prefill.build_layer_layout_into)."""
    lib = _lib.load()
    _lib.check(lib.spf_csr_guard(_dev.ptr(tile_offsets), _dev.ptr(col_offsets), tile_offsets.numel() - 1,
                                 int(cap_tiles), int(cap_cols), _dev.ptr(overflow), _dev.ptr(totals),
                                 _dev.stream_handle(stream)), "spf_csr_guard")


def vs_count(vertical: torch.Tensor, slash: torch.Tensor, head_ids, seq_len: int, block_size: int,
             tile_counts: torch.Tensor, col_counts: torch.Tensor, stream=None):
    lib = _lib.load()
    n_heads, n_v = vertical.shape
    n_s = slash.shape[1]
    _lib.check(lib.spf_vs_layout_count(_dev.ptr(vertical), n_v, _dev.ptr(slash), n_s, _dev.ptr(head_ids), n_heads,
                                       seq_len, block_size, _dev.ptr(tile_counts), _dev.ptr(col_counts),
                                       _dev.stream_handle(stream)), "spf_vs_layout_count")


def vs_fill(vertical, slash, head_ids, seq_len, block_size, tile_offsets, col_offsets, tiles, cols, stream=None):
    lib = _lib.load()
    n_heads, n_v = vertical.shape
    n_s = slash.shape[1]
    _lib.check(lib.spf_vs_layout_fill(_dev.ptr(vertical), n_v, _dev.ptr(slash), n_s, _dev.ptr(head_ids), n_heads,
                                      seq_len, block_size, _dev.ptr(tile_offsets), _dev.ptr(col_offsets),
                                      _dev.ptr(tiles if tiles.numel() else None),
                                      _dev.ptr(cols if cols.numel() else None), _dev.stream_handle(stream)),
               "spf_vs_layout_fill")


def ashape_count(head_ids, n_heads, seq_len, block_size, cfg: AShape, tile_counts, stream=None):
    lib = _lib.load()
    _lib.check(lib.spf_ashape_layout_count(_dev.ptr(head_ids), n_heads, seq_len, block_size, cfg.global_tokens,
                                           cfg.local_window, _dev.ptr(tile_counts), _dev.stream_handle(stream)),
               "spf_ashape_layout_count")


def ashape_fill(head_ids, n_heads, seq_len, block_size, cfg: AShape, tile_offsets, tiles, stream=None):
    lib = _lib.load()
    _lib.check(lib.spf_ashape_layout_fill(_dev.ptr(head_ids), n_heads, seq_len, block_size, cfg.global_tokens,
                                          cfg.local_window, _dev.ptr(tile_offsets), _dev.ptr(tiles),
                                          _dev.stream_handle(stream)), "spf_ashape_layout_fill")


def bs_count(head_ids, n_heads, seq_len, block_size, k_b, tile_counts, stream=None):
    lib = _lib.load()
    _lib.check(lib.spf_bs_layout_count(_dev.ptr(head_ids), n_heads, seq_len, block_size, k_b,
                                       _dev.ptr(tile_counts), _dev.stream_handle(stream)), "spf_bs_layout_count")


def layout_area_dev(n_heads, seq_len, block_size, tiles, tile_offsets, col_offsets, stream=None) -> torch.Tensor:
    """Per-head computed-cell area (patterns.py:147-184) of a device CSR."""
    lib = _lib.load()
    area = torch.empty(n_heads, dtype=torch.int64, device=tile_offsets.device)
    _lib.check(lib.spf_layout_area(n_heads, seq_len, block_size, _dev.ptr(tiles if tiles.numel() else None),
                                   _dev.ptr(tile_offsets), _dev.ptr(col_offsets), _dev.ptr(area),
                                   _dev.stream_handle(stream)), "spf_layout_area")
    return area


# ------------------------------------------------------------------ host-facing builders
def _csr_to_host(seq_len, block_size, tiles, toff, cols, coff) -> SparseLayout:
    return SparseLayout.from_csr(seq_len, block_size, tiles.cpu().numpy().astype(np.int64), toff.cpu().numpy(),
                                 cols.cpu().numpy().astype(np.int64), coff.cpu().numpy())


def ashape_layout_host(seq_len: int, cfg: AShape, block_size: int) -> SparseLayout:
    dev = _dev.require_cuda()
    n = n_block_rows(seq_len, block_size)
    cnt = torch.zeros(n, dtype=torch.int64, device=dev)
    ashape_count(None, 1, seq_len, block_size, cfg, cnt)
    toff, total = csr_offsets(cnt)
    tiles = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    ashape_fill(None, 1, seq_len, block_size, cfg, toff, tiles)
    empty_cols = torch.zeros(0, dtype=torch.int32, device=dev)
    coff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    return _csr_to_host(seq_len, block_size, tiles[:total], toff, empty_cols, coff)


def vs_layout_dev(vertical: torch.Tensor, slash: torch.Tensor, seq_len: int, block_size: int, head_ids=None,
                  n_q_heads: int | None = None, stream=None):
    """Full VS CSR on device for heads given by (vertical [n, n_v], slash [n, n_s])."""
    dev = vertical.device
    n_heads = vertical.shape[0]
    hq = n_heads if n_q_heads is None else n_q_heads
    n = n_block_rows(seq_len, block_size)
    tc = torch.zeros(hq * n, dtype=torch.int64, device=dev)
    cc = torch.zeros(hq * n, dtype=torch.int64, device=dev)
    vs_count(vertical, slash, head_ids, seq_len, block_size, tc, cc, stream)
    toff, tt = csr_offsets(tc, stream)
    coff, ct = csr_offsets(cc, stream)
    tiles = torch.empty(max(tt, 1), dtype=torch.int32, device=dev)
    cols = torch.empty(max(ct, 1), dtype=torch.int32, device=dev)
    vs_fill(vertical, slash, head_ids, seq_len, block_size, toff, coff, tiles, cols, stream)
    return tiles[:tt], toff, cols[:ct], coff


def vs_layout_host(vertical, slash, seq_len: int, block_size: int) -> SparseLayout:
    dev = _dev.require_cuda()
    v = torch.from_numpy(np.ascontiguousarray(np.asarray(vertical, dtype=np.int64).astype(np.int32))).to(dev)
    s = torch.from_numpy(np.ascontiguousarray(np.asarray(slash, dtype=np.int64).astype(np.int32))).to(dev)
    tiles, toff, cols, coff = vs_layout_dev(v.view(1, -1), s.view(1, -1), seq_len, block_size)
    return _csr_to_host(seq_len, block_size, tiles, toff, cols, coff)


def layout_area_host(layout: SparseLayout) -> int:
    dev = _dev.require_cuda()
    t, to, c, co = layout.csr()
    area = layout_area_dev(1, layout.seq_len, layout.block_size, _dev.to_device_i32(t, dev),
                           _dev.to_device_i64(to, dev), _dev.to_device_i64(co, dev))
    return int(area.cpu()[0])
