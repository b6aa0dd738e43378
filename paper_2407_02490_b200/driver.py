"""Per-model pre-fill driver over a pattern-config document.

The reference stores one searched pattern per (layer, head) in the config
JSON v1 document (patterns.py:236-266, written by ``cmd_search``, read by
``cmd_run``, cli.py:55-126) and runs heads one at a time.  ``PatternTable``
holds that document for a whole model, validates it once (every (layer, head)
present exactly once, one head count, one block size per layer) and keeps,
per layer, the device-side head groups the layer pipeline needs (q-head ids
per distinct config), so a model pass uploads nothing per layer.
``SparsePrefill`` runs layers through ``prefill.sparse_prefill_attention``:
per layer one grouped estimation pass per config, one CSR compaction and ONE
attention launch over all heads and patterns.
"""

from __future__ import annotations

import math
from collections import OrderedDict

import torch

from .patterns import (AShape, BlockSparse, HeadPatternConfig, VerticalSlash, config_from_entry, config_to_entry,
                       flops_in_kernel, load_pattern_configs, save_pattern_configs)
from .prefill import sparse_prefill_attention


class PatternTable:
    """[layer][head] -> pattern config, plus cached per-layer device head groups."""

    def __init__(self, layers):
        layers = [list(row) for row in layers]
        if not layers or not layers[0]:
            raise ValueError("pattern table needs at least one layer and one head")
        n_heads = len(layers[0])
        for li, row in enumerate(layers):
            if len(row) != n_heads:
                raise ValueError(f"layer {li} has {len(row)} heads, layer 0 has {n_heads}")
            for hi, cfg in enumerate(row):
                if not isinstance(cfg, (AShape, VerticalSlash, BlockSparse)):
                    raise TypeError(f"layer {li} head {hi}: unknown pattern config {cfg!r}")
            sizes = {cfg.block_size for cfg in row if isinstance(cfg, BlockSparse)}
            if len(sizes) > 1:
                raise ValueError(f"layer {li}: Block-Sparse heads use different block sizes {sorted(sizes)}")
        self.layers = layers
        self._groups = {}

    @classmethod
    def from_entries(cls, entries) -> "PatternTable":
        cells = {}
        for e in entries:
            layer, head, cfg = config_from_entry(e)
            if layer < 0 or head < 0:
                raise ValueError(f"negative layer/head in entry {e!r}")
            if (layer, head) in cells:
                raise ValueError(f"duplicate entry for layer {layer} head {head}")
            cells[(layer, head)] = cfg
        if not cells:
            raise ValueError("pattern config document has no heads")
        n_layers = 1 + max(l for l, _ in cells)
        n_heads = 1 + max(h for _, h in cells)
        missing = [(l, h) for l in range(n_layers) for h in range(n_heads) if (l, h) not in cells]
        if missing:
            raise ValueError(f"pattern config missing entries for (layer, head): {missing[:8]}"
                             + (" ..." if len(missing) > 8 else ""))
        return cls([[cells[(l, h)] for h in range(n_heads)] for l in range(n_layers)])

    @classmethod
    def load(cls, path) -> "PatternTable":
        return cls.from_entries(load_pattern_configs(path))

    def save(self, path) -> None:
        save_pattern_configs(path, [config_to_entry(l, h, c) for l, row in enumerate(self.layers)
                                    for h, c in enumerate(row)])

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    @property
    def n_heads(self) -> int:
        return len(self.layers[0])

    def layer(self, layer: int) -> list:
        return self.layers[layer]

    def block_size(self, layer: int, default: int = 64) -> int:
        """The layer's tile size: its Block-Sparse heads' block_size if any (they must
        run at their own size, sparse_attn.py:87-90), else ``default``."""
        for cfg in self.layers[layer]:
            if isinstance(cfg, BlockSparse):
                return cfg.block_size
        return default

    def device_groups(self, layer: int, device) -> list:
        """[(config, int32 q-head ids on ``device``, count)] in first-appearance order."""
        key = (layer, str(torch.device(device)))
        if key not in self._groups:
            groups: "OrderedDict[HeadPatternConfig, list[int]]" = OrderedDict()
            for h, cfg in enumerate(self.layers[layer]):
                groups.setdefault(cfg, []).append(h)
            self._groups[key] = [(cfg, torch.tensor(ids, dtype=torch.int32, device=device), len(ids))
                                 for cfg, ids in groups.items()]
        return self._groups[key]

    def pattern_counts(self) -> dict:
        out = {}
        for row in self.layers:
            for cfg in row:
                name = type(cfg).__name__
                out[name] = out.get(name, 0) + 1
        return out

    def modeled_flops(self, seq_len: int, head_dim: int, block_size: int = 64) -> list:
        """Per-layer sum of flops_in_kernel (patterns.py:191-218) over the layer's heads."""
        return [sum(flops_in_kernel(c, seq_len, head_dim, block_size) for c in row) for row in self.layers]


class SparsePrefill:
    """Run a model's attention layers with their searched per-head patterns."""

    def __init__(self, table: PatternTable, block_size: int = 64, scale: float | None = None):
        self.table = table
        self.default_block = block_size
        self.scale = scale

    def layer(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out=None, stream=None,
              return_layout: bool = False):
        if q.shape[0] != self.table.n_heads:
            raise ValueError(f"layer {layer}: q has {q.shape[0]} heads, the table has {self.table.n_heads}")
        cfgs = self.table.layer(layer)
        sc = self.scale if self.scale is not None else 1.0 / math.sqrt(q.shape[-1])
        return sparse_prefill_attention(q, k, v, cfgs, self.table.block_size(layer, self.default_block), sc, out,
                                        stream, return_layout, groups=self.table.device_groups(layer, q.device))

    def __call__(self, layers_qkv, stream=None):
        """``layers_qkv``: iterable of (q, k, v) per layer, in layer order; yields outputs."""
        for layer, (q, k, v) in enumerate(layers_qkv):
            if layer >= self.table.n_layers:
                raise ValueError(f"more layers than the pattern table holds ({self.table.n_layers})")
            yield self.layer(layer, q, k, v, stream=stream)
