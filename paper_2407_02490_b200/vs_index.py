"""Point-range two-way merge: VSIndices -> SparseLayout, on the GPU.

Drop-in mirror of /root/reference/pkg/src/sparseprefill/vs_index.py
(Alg. 4, vs_index.py:28-95).  The merge itself runs in libspf
(spf_vs_layout_count / spf_vs_layout_fill, one thread per query-block row,
bit-exact with the reference); this module keeps the reference signatures,
range checks and the per-row operation count of ``build_vs_layout_with_stats``.
"""

from __future__ import annotations

import numpy as np

from . import layouts
from .estimator import VSIndices
from .patterns import SparseLayout, n_block_rows


def _check(idx: VSIndices, seq_len: int, block_size: int):
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    points = np.asarray(idx.vertical, dtype=np.int64)
    slashes = np.asarray(idx.slash, dtype=np.int64)
    if points.size and (points.max() >= seq_len or points.min() < 0):
        raise ValueError("vertical index out of range")
    if slashes.size and (slashes.max() >= seq_len or slashes.min() < 0):
        raise ValueError("slash offset out of range")
    return points, slashes


def build_vs_layout(idx: VSIndices, seq_len: int, block_size: int) -> SparseLayout:
    points, slashes = _check(idx, seq_len, block_size)
    return layouts.vs_layout_host(points, slashes, seq_len, block_size)


def build_vs_layout_with_stats(idx: VSIndices, seq_len: int, block_size: int) -> tuple[SparseLayout, list[int]]:
    """Build the layout and return the merge-loop operation count per row.

    ops(r) = (#slash offsets < q_end) + (#points, each inspected once)
             + (#tiles emitted), which is what vs_index.py:44-94 counts.
    """
    points, slashes = _check(idx, seq_len, block_size)
    layout = layouts.vs_layout_host(points, slashes, seq_len, block_size)
    n = n_block_rows(seq_len, block_size)
    q_end = np.minimum((np.arange(n, dtype=np.int64) + 1) * block_size, seq_len)
    asc = np.sort(slashes)
    active = np.searchsorted(asc, q_end, side="left")
    tiles = np.diff(layout.block_starts.offsets)
    ops = active + points.size + tiles
    return layout, [int(x) for x in ops]
