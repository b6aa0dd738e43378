"""Pattern configurations, the sparse layout type, and FLOP accounting.

Drop-in mirror of /root/reference/pkg/src/sparseprefill/patterns.py:

* ``AShape`` / ``VerticalSlash`` / ``BlockSparse`` (patterns.py:23-57) with the
  same fields, defaults (B = 64, last_q = 64, patterns.py:19-20) and
  ``ValueError`` validation; ``HeadPatternConfig``; ``PATTERN_NAMES``;
* ``SparseLayout`` (patterns.py:69-106): per query-block row, tile starts and
  residual columns.  A layout built by the GPU is CSR-backed (int64 arrays),
  one built by hand keeps plain lists; both expose ``block_starts`` /
  ``column_indices`` as per-row sequences, and ``validate()`` enforces the
  reference invariants (vectorised instead of the reference's
  O(cols x tiles) loop);
* ``a_shape_layout`` (patterns.py:109-128) and ``layout_area`` (147-184) run
  on the GPU through libspf (spf_ashape_layout_*, spf_layout_area);
* ``flops_in_kernel`` (191-233), ``causal_area``, ``layout_to_mask`` and the
  config JSON document (236-266) are host-side metadata, as in the reference.
"""

from __future__ import annotations

import json
from collections.abc import Sequence
from dataclasses import dataclass, field
from typing import Union

import numpy as np

CONFIG_FORMAT_VERSION = 1

DEFAULT_BLOCK_SIZE = 64
DEFAULT_LAST_Q = 64


@dataclass(frozen=True)
class AShape:
    """Static pattern: initial (sink) tokens plus a local diagonal window."""

    global_tokens: int
    local_window: int

    def __post_init__(self):
        if self.global_tokens < 1 or self.local_window < 1:
            raise ValueError("A-shape counts must be >= 1")


@dataclass(frozen=True)
class VerticalSlash:
    """Dynamic pattern: top key columns plus top diagonal offsets."""

    k_v: int
    k_s: int
    last_q: int = DEFAULT_LAST_Q

    def __post_init__(self):
        if self.k_v < 1 or self.k_s < 1 or self.last_q < 1:
            raise ValueError("Vertical-Slash counts must be >= 1")


@dataclass(frozen=True)
class BlockSparse:
    """Dynamic pattern: top key blocks per query-block row."""

    k_b: int
    block_size: int = DEFAULT_BLOCK_SIZE

    def __post_init__(self):
        if self.k_b < 1 or self.block_size < 1:
            raise ValueError("Block-Sparse counts must be >= 1")


HeadPatternConfig = Union[AShape, VerticalSlash, BlockSparse]

PATTERN_NAMES = {AShape: "a_shape", VerticalSlash: "vertical_slash", BlockSparse: "block_sparse"}


def n_block_rows(seq_len: int, block_size: int) -> int:
    return (seq_len + block_size - 1) // block_size


class RaggedRows(Sequence):
    """Read-only per-row view of a CSR (flat int64 + offsets int64)."""

    __slots__ = ("flat", "offsets")

    def __init__(self, flat, offsets):
        self.flat = np.asarray(flat, dtype=np.int64)
        self.offsets = np.asarray(offsets, dtype=np.int64)

    def __len__(self):
        return int(self.offsets.size - 1)

    def __getitem__(self, r):
        if isinstance(r, slice):
            return [self[i] for i in range(*r.indices(len(self)))]
        n = len(self)
        if r < 0:
            r += n
        if not 0 <= r < n:
            raise IndexError(r)
        return [int(x) for x in self.flat[self.offsets[r]: self.offsets[r + 1]]]

    def __eq__(self, other):
        if isinstance(other, RaggedRows):
            return np.array_equal(self.offsets, other.offsets) and np.array_equal(self.flat, other.flat)
        try:
            return len(other) == len(self) and all(list(a) == list(b) for a, b in zip(self, other))
        except TypeError:
            return NotImplemented

    def __repr__(self):
        return f"RaggedRows(rows={len(self)}, entries={self.flat.size})"


def _to_csr(rows) -> tuple[np.ndarray, np.ndarray]:
    if isinstance(rows, RaggedRows):
        return rows.flat, rows.offsets
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    for r, row in enumerate(rows):
        off[r + 1] = off[r] + len(row)
    flat = np.fromiter((int(x) for row in rows for x in row), dtype=np.int64, count=int(off[-1]))
    return flat, off


@dataclass
class SparseLayout:
    seq_len: int
    block_size: int
    block_starts: list = field(default_factory=list)  # per row: sorted key-start offsets
    column_indices: list = field(default_factory=list)  # per row: sorted residual columns

    @classmethod
    def from_csr(cls, seq_len, block_size, tiles, tile_offsets, cols, col_offsets) -> "SparseLayout":
        return cls(seq_len, block_size, RaggedRows(tiles, tile_offsets), RaggedRows(cols, col_offsets))

    def n_rows(self) -> int:
        return n_block_rows(self.seq_len, self.block_size)

    def query_range(self, row: int) -> tuple[int, int]:
        start = row * self.block_size
        return start, min(start + self.block_size, self.seq_len)

    def csr(self):
        """(tile_starts, tile_offsets, col_indices, col_offsets) as int64 arrays."""
        t, to = _to_csr(self.block_starts)
        c, co = _to_csr(self.column_indices)
        return t, to, c, co

    def validate(self) -> None:
        """patterns.py:83-106 invariants, vectorised over the CSR."""
        n = self.n_rows()
        if len(self.block_starts) != n or len(self.column_indices) != n:
            raise ValueError("layout must have one tile list and one column list per row")
        b = self.block_size
        t, to, c, co = self.csr()
        rows_t = np.repeat(np.arange(n, dtype=np.int64), np.diff(to))
        rows_c = np.repeat(np.arange(n, dtype=np.int64), np.diff(co))
        q_end_t = np.minimum((rows_t + 1) * b, self.seq_len)
        q_end_c = np.minimum((rows_c + 1) * b, self.seq_len)
        same_t = rows_t[1:] == rows_t[:-1]
        dt = np.diff(t)
        bad = np.nonzero(same_t & (dt <= 0))[0]
        if bad.size:
            raise ValueError(f"row {rows_t[bad[0]]}: tile starts must be strictly increasing")
        bad = np.nonzero(same_t & (dt < b))[0]
        if bad.size:
            raise ValueError(f"row {rows_t[bad[0]]}: tiles overlap")
        same_c = rows_c[1:] == rows_c[:-1]
        bad = np.nonzero(same_c & (np.diff(c) <= 0))[0]
        if bad.size:
            raise ValueError(f"row {rows_c[bad[0]]}: columns must be strictly increasing")
        bad = np.nonzero((t < 0) | (t >= q_end_t))[0]
        if bad.size:
            raise ValueError(f"row {rows_t[bad[0]]}: tile start {t[bad[0]]} outside causal range")
        bad = np.nonzero((c < 0) | (c >= q_end_c))[0]
        if bad.size:
            raise ValueError(f"row {rows_c[bad[0]]}: column {c[bad[0]]} outside causal range")
        if c.size and t.size:
            # disjointness: the last tile start <= c in the same row must not cover c
            key_t = rows_t * (np.int64(1) << 40) + t
            key_c = rows_c * (np.int64(1) << 40) + c
            pos = np.searchsorted(key_t, key_c, side="right") - 1
            ok = pos >= 0
            hit = np.zeros(c.size, dtype=bool)
            hit[ok] = (rows_t[pos[ok]] == rows_c[ok]) & (t[pos[ok]] + b > c[ok])
            bad = np.nonzero(hit)[0]
            if bad.size:
                i = bad[0]
                s = t[pos[i]]
                raise ValueError(f"row {rows_c[i]}: column {c[i]} duplicates tile [{s}, {s + b})")


def a_shape_layout(seq_len: int, cfg: AShape, block_size: int) -> SparseLayout:
    """patterns.py:109-128, built on the GPU (spf_ashape_layout_count/fill)."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    from . import layouts

    return layouts.ashape_layout_host(seq_len, cfg, block_size)


def layout_to_mask(layout: SparseLayout) -> np.ndarray:
    """patterns.py:131-144: dense boolean mask (causally clipped); O(S^2)."""
    s_len = layout.seq_len
    b = layout.block_size
    mask = np.zeros((s_len, s_len), dtype=bool)
    for r in range(layout.n_rows()):
        q_start, q_end = layout.query_range(r)
        for s in layout.block_starts[r]:
            mask[q_start:q_end, max(s, 0):min(s + b, s_len)] = True
        for c in layout.column_indices[r]:
            mask[q_start:q_end, c] = True
    rows = np.arange(s_len)
    mask &= rows[:, None] >= rows[None, :]
    return mask


def layout_area(layout: SparseLayout) -> int:
    """patterns.py:147-163: computed cells at kernel granularity (GPU)."""
    from . import layouts

    return int(layouts.layout_area_host(layout))


def causal_area(seq_len: int) -> int:
    return seq_len * (seq_len + 1) // 2


def flops_in_kernel(cfg: HeadPatternConfig, seq_len: int, head_dim: int, block_size: int) -> int:
    """patterns.py:191-218: modeled kernel FLOPs = 4 * d * computed-cell area."""
    return 4 * head_dim * _model_area(cfg, seq_len, block_size)


def _model_area(cfg: HeadPatternConfig, seq_len: int, block_size: int) -> int:
    """patterns.py:221-233 (A-shape: realized layout; BS: exact; VS: model)."""
    b = block_size
    if isinstance(cfg, AShape):
        # area of the realized layout (patterns.py:109-128), closed form per row: the
        # aligned sink tiles [0, a) and window tiles [w0, r] are all below the diagonal
        # except tile r (the triangle), so no layout needs to be built for the model
        n = n_block_rows(seq_len, b)
        r = np.arange(n, dtype=np.int64)
        q_start = r * b
        q_end = np.minimum(q_start + b, seq_len)
        h = q_end - q_start
        a = (np.minimum(cfg.global_tokens, q_end) + b - 1) // b
        w0 = np.maximum(0, q_start - cfg.local_window) // b
        n_tiles = (r + 1 - w0) + np.minimum(a, w0)
        return int(np.sum((n_tiles - 1) * h * b + h * (h + 1) // 2))
    if isinstance(cfg, BlockSparse):
        b = cfg.block_size
        n = n_block_rows(seq_len, b)
        r = np.arange(n, dtype=np.int64)
        h = np.minimum(b, seq_len - r * b)
        n_sel = np.minimum(cfg.k_b, r + 1)
        return int(np.sum((n_sel - 1) * h * b + h * (h + 1) // 2))
    if isinstance(cfg, VerticalSlash):
        n = n_block_rows(seq_len, b)
        r = np.arange(n, dtype=np.int64)
        q_start = r * b
        q_end = np.minimum(q_start + b, seq_len)
        h = q_end - q_start
        w = q_end
        slash_tiles = np.minimum((cfg.k_s + b - 1 + b - 1) // b, (w + b - 1) // b)
        col_chips = (np.minimum(cfg.k_v, w) + b - 1) // b
        cells = np.minimum(h * (slash_tiles * b + col_chips * b), q_start * h + h * (h + 1) // 2)
        return int(np.sum(cells))
    raise TypeError(f"unknown pattern config: {cfg!r}")


# --- pattern config document (JSON), patterns.py:236-266 --------------------


def config_to_entry(layer: int, head: int, cfg: HeadPatternConfig) -> dict:
    params = {k: getattr(cfg, k) for k in cfg.__dataclass_fields__}
    return {"layer": layer, "head": head, "pattern": PATTERN_NAMES[type(cfg)], "params": params}


def config_from_entry(entry: dict) -> tuple[int, int, HeadPatternConfig]:
    by_name = {v: k for k, v in PATTERN_NAMES.items()}
    name = entry["pattern"]
    if name not in by_name:
        raise ValueError(f"unknown pattern name: {name!r}")
    cfg = by_name[name](**entry["params"])
    return int(entry["layer"]), int(entry["head"]), cfg


def save_pattern_configs(path, entries: list[dict]) -> None:
    doc = {"format_version": CONFIG_FORMAT_VERSION, "heads": entries}
    with open(path, "w") as f:
        json.dump(doc, f, indent=2, sort_keys=True)
        f.write("\n")


def load_pattern_configs(path) -> list[dict]:
    with open(path) as f:
        doc = json.load(f)
    version = doc.get("format_version")
    if version != CONFIG_FORMAT_VERSION:
        raise ValueError(f"unsupported pattern config format_version: {version!r}")
    return doc["heads"]
