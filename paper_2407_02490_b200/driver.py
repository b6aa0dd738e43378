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

from . import kernels
from .patterns import (AShape, BlockSparse, HeadPatternConfig, VerticalSlash, config_from_entry, config_to_entry,
                       flops_in_kernel, load_pattern_configs, save_pattern_configs)
from .prefill import _pair_heads, build_layer_layout, build_layer_layout_into, sparse_prefill_attention


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

    def device_groups(self, layer: int, device, heads: tuple | None = None) -> list:
        """[(config, int32 q-head ids on ``device``, count)] in first-appearance order;
        ``heads`` = (h0, h1) restricts to that head range (ids then relative to h0)."""
        h0, h1 = heads if heads is not None else (0, self.n_heads)
        key = (layer, str(torch.device(device)), h0, h1)
        if key not in self._groups:
            groups: "OrderedDict[HeadPatternConfig, list[int]]" = OrderedDict()
            for h, cfg in enumerate(self.layers[layer][h0:h1]):
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

    def layer_heads(self, layer: int, h0: int, h1: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out=None,
                    stream=None):
        """The layer restricted to q-heads [h0, h1) (whole kv groups): q [h1-h0, S, d] and
        the k/v heads they read."""
        if q.shape[0] != h1 - h0:
            raise ValueError(f"layer {layer}: q has {q.shape[0]} heads for the head range [{h0}, {h1})")
        cfgs = self.table.layer(layer)[h0:h1]
        sc = self.scale if self.scale is not None else 1.0 / math.sqrt(q.shape[-1])
        return sparse_prefill_attention(q, k, v, cfgs, self.table.block_size(layer, self.default_block), sc, out,
                                        stream, groups=self.table.device_groups(layer, q.device, (h0, h1)))

    def prefill_host(self, host_layers, host_out, chunks: int = 1, device=None):
        """Host-resident model pass: ``host_layers`` = [(q, k, v)] per layer (pinned CPU
        tensors [Hq, S, d] / [Hkv, S, d]), outputs into ``host_out`` (pinned CPU [Hq, S, d]
        per layer).  Each layer is split into ``chunks`` head ranges of whole kv groups;
        unit u = (layer, chunk) is copied in on one stream while unit u-1 computes and
        unit u-2 is copied out on a third, through two device slots, so the PCIe
        transfers in both directions overlap the kernels (the first and last units'
        copies are the only exposed ones: finer chunks shrink them).  Returns after
        enqueueing; the caller synchronises."""
        if len(host_layers) > self.table.n_layers or len(host_out) != len(host_layers):
            raise ValueError("one output per layer, at most the table's layers")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        q0, k0, _ = host_layers[0]
        hq, hkv = q0.shape[0], k0.shape[0]
        if hq != self.table.n_heads or hq % hkv:
            raise ValueError("head counts do not match the pattern table")
        qpk = hq // hkv
        chunks = max(1, min(int(chunks), hkv))
        bounds = [(hkv * c // chunks, hkv * (c + 1) // chunks) for c in range(chunks)]
        units = [(layer, g0, g1) for layer in range(len(host_layers)) for g0, g1 in bounds]
        gmax = max(g1 - g0 for g0, g1 in bounds)
        S, d = q0.shape[1], q0.shape[2]
        slots = [dict(q=torch.empty((gmax * qpk, S, d), dtype=q0.dtype, device=dev),
                      k=torch.empty((gmax, S, d), dtype=q0.dtype, device=dev),
                      v=torch.empty((gmax, S, d), dtype=q0.dtype, device=dev),
                      o=torch.empty((gmax * qpk, S, d), dtype=q0.dtype, device=dev)) for _ in range(2)]
        comp = torch.cuda.current_stream(dev)
        if not hasattr(self, "_copy_streams") or self._copy_streams[0].device != dev:
            self._copy_streams = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        h2d, d2h = self._copy_streams
        ready, freed = [None, None], [None, None]

        def issue_in(u):
            layer, g0, g1 = units[u]
            s = slots[u % 2]
            qh, kh, vh = host_layers[layer]
            with torch.cuda.stream(h2d):
                if freed[u % 2] is not None:
                    h2d.wait_event(freed[u % 2])  # compute of unit u-2 has read the slot
                s["q"][: (g1 - g0) * qpk].copy_(qh[g0 * qpk:g1 * qpk], non_blocking=True)
                s["k"][: g1 - g0].copy_(kh[g0:g1], non_blocking=True)
                s["v"][: g1 - g0].copy_(vh[g0:g1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
            ready[u % 2] = ev

        out_done = [None, None]
        issue_in(0)
        for u, (layer, g0, g1) in enumerate(units):
            if u + 1 < len(units):
                issue_in(u + 1)
            s = slots[u % 2]
            n_q = (g1 - g0) * qpk
            comp.wait_event(ready[u % 2])
            if out_done[u % 2] is not None:
                comp.wait_event(out_done[u % 2])  # the slot's previous output has been copied out
            self.layer_heads(layer, g0 * qpk, g1 * qpk, s["q"][:n_q], s["k"][: g1 - g0], s["v"][: g1 - g0],
                             out=s["o"][:n_q])
            ev = torch.cuda.Event()
            ev.record(comp)
            freed[u % 2] = ev
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev)
                host_out[layer][g0 * qpk:g1 * qpk].copy_(s["o"][:n_q], non_blocking=True)
                e2 = torch.cuda.Event()
                e2.record(d2h)
            out_done[u % 2] = e2
        comp.wait_stream(d2h)
        comp.wait_stream(h2d)

    def _side_stream(self, dev):
        if getattr(self, "_est_stream", None) is None or self._est_stream.device != dev:
            # high priority: when an SM frees up, estimation CTAs go before pending attention CTAs
            lo, hi = torch.cuda.Stream.priority_range()
            self._est_stream = torch.cuda.Stream(dev, priority=hi)
        return self._est_stream

    def prefill(self, layers_qkv, outs=None, attn_events=None, after_layer=None, pipeline: bool = False):
        """Device-resident model pass: ``layers_qkv`` = [(q, k, v)] per layer ([Hq, S, d] /
        [Hkv, S, d] bf16 on the device); returns the outputs (``outs`` if given), enqueued on
        the current stream.  ``attn_events`` (optional list) receives a (start, end) CUDA event
        pair around every layer's attention launch; ``after_layer(layer, out)`` (optional) is
        called once a layer's attention is enqueued (e.g. to start its output all-gather while
        the next layer computes, sharding.gather_heads_async).

        Default (``pipeline=False``): one stream and no per-layer host sync.  A layer's CSR
        is sized from what the same layer needed on the previous call (+12.5 %), in one
        grow-only buffer pair shared by the layers; ``spf_csr_guard`` checks the sizes on the
        device and empties an overflowing layer instead of overrunning anything.  One
        read-back per call checks the flags and recomputes an overflowed layer with an exact
        size (calling ``after_layer`` again for it).  A layer seen for the first time is
        sized exactly (one host read-back).

        ``pipeline=True``: layer l+1's estimation and compaction run on a high-priority side
        stream while layer l's attention runs (exact sizing; the read-back waits for the
        side stream only)."""
        layers = list(layers_qkv)
        if len(layers) > self.table.n_layers:
            raise ValueError(f"more layers than the pattern table holds ({self.table.n_layers})")
        if not layers:
            return []
        for layer, (q, _, _) in enumerate(layers):
            if q.shape[0] != self.table.n_heads:
                raise ValueError(f"layer {layer}: q has {q.shape[0]} heads, the table has {self.table.n_heads}")
        if pipeline:
            return self._prefill_pipelined(layers, outs, attn_events, after_layer)
        return self._prefill_speculative(layers, outs, attn_events, after_layer)

    def _attend(self, layer, q, k, v, lay, b, out, stream, attn_events):
        sc = self.scale if self.scale is not None else 1.0 / math.sqrt(q.shape[-1])
        if attn_events is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        kernels.sparse_flash_attention_gpu(q, k, v, sc, b, lay.tiles, lay.tile_offsets, lay.cols, lay.col_offsets,
                                           out=out, stream=stream, pair_heads=_pair_heads(self.table.layer(layer),
                                                                                          q.device))
        if attn_events is not None:
            e1.record(stream)
            attn_events.append((e0, e1))

    def _prefill_speculative(self, layers, outs, attn_events, after_layer):
        dev = layers[0][0].device
        comp = torch.cuda.current_stream(dev)
        if not hasattr(self, "_caps"):
            self._caps = {}
        n_layers = len(layers)
        flags = torch.zeros(n_layers, dtype=torch.int32, device=dev)
        totals = torch.zeros((n_layers, 2), dtype=torch.int64, device=dev)
        keys = [(layer, tuple(q.shape), tuple(k.shape), str(dev)) for layer, (q, k, _) in enumerate(layers)]

        if not hasattr(self, "_arenas"):
            self._arenas = {}
        akey = (str(dev), int(comp.cuda_stream))  # one buffer pair per stream: passes on two streams never share

        def arena(nt, nc):
            cur = self._arenas.get(akey)
            if cur is None or cur[0].numel() < nt or cur[1].numel() < nc:
                nt2 = max(nt, cur[0].numel() if cur is not None else 0)
                nc2 = max(nc, cur[1].numel() if cur is not None else 0)
                cur = (torch.empty(max(nt2, 1), dtype=torch.int32, device=dev),
                       torch.empty(max(nc2, 1), dtype=torch.int32, device=dev))
                self._arenas[akey] = cur
            return cur

        speculated = []
        results = []
        for layer, (q, k, v) in enumerate(layers):
            cfgs = self.table.layer(layer)
            b = self.table.block_size(layer, self.default_block)
            groups = self.table.device_groups(layer, dev)
            out = outs[layer] if outs is not None else torch.empty_like(q)
            cap = self._caps.get(keys[layer])
            if cap is None:
                lay = build_layer_layout(q, k, cfgs, b, groups=groups)
                self._caps[keys[layer]] = (lay.n_tiles + lay.n_tiles // 8 + 64, lay.n_cols + lay.n_cols // 8 + 64)
            else:
                t_buf, c_buf = arena(*cap)
                lay = build_layer_layout_into(q, k, cfgs, b, t_buf[:cap[0]], c_buf[:cap[1]], flags[layer:layer + 1],
                                              totals[layer], groups=groups)
                speculated.append(layer)
            self._attend(layer, q, k, v, lay, b, out, comp, attn_events)
            results.append(out)
            if after_layer is not None:
                after_layer(layer, out)
        if speculated:
            f = flags.cpu()  # the one read-back of the call
            if int(f.sum()):
                tot = totals.cpu()
                for layer in speculated:
                    if int(f[layer]):
                        q, k, v = layers[layer]
                        nt, nc = int(tot[layer, 0]), int(tot[layer, 1])
                        self._caps[keys[layer]] = (nt + nt // 8 + 64, nc + nc // 8 + 64)
                        b = self.table.block_size(layer, self.default_block)
                        lay = build_layer_layout(q, k, self.table.layer(layer), b,
                                                 groups=self.table.device_groups(layer, dev))
                        self._attend(layer, q, k, v, lay, b, results[layer], comp, None)
                        if after_layer is not None:
                            after_layer(layer, results[layer])
        return results

    def graph_layer(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor):
        """Capture one layer (estimation, compaction into a fixed-capacity CSR, attention) in a
        CUDA graph over the static buffers ``q``, ``k``, ``v``, ``out``; returns ``replay()``,
        which re-runs the layer on whatever those buffers then hold and returns the overflow
        flag (an int32 device scalar: 1 = the layout outgrew the captured capacity and ``out``
        is not valid; re-capture after an exact run).  The layer is first run eagerly to size
        the CSR (with the same +12.5 % slack as ``prefill``) and to finish one-time setup."""
        dev = q.device
        cfgs = self.table.layer(layer)
        b = self.table.block_size(layer, self.default_block)
        groups = self.table.device_groups(layer, dev)
        lay = build_layer_layout(q, k, cfgs, b, groups=groups)
        nt, nc = lay.n_tiles + lay.n_tiles // 8 + 64, lay.n_cols + lay.n_cols // 8 + 64
        tiles = torch.empty(nt, dtype=torch.int32, device=dev)
        cols = torch.empty(nc, dtype=torch.int32, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        totals = torch.zeros(2, dtype=torch.int64, device=dev)

        def body():
            lay2 = build_layer_layout_into(q, k, cfgs, b, tiles, cols, flag, totals, groups=groups)
            self._attend(layer, q, k, v, lay2, b, out, torch.cuda.current_stream(dev), None)

        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up on the capture stream (workspaces, attributes)
            body()
        torch.cuda.current_stream(dev).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            flag.zero_()
            body()

        def replay():
            graph.replay()
            return flag

        replay.graph = graph
        return replay

    def _prefill_pipelined(self, layers, outs, attn_events, after_layer):
        dev = layers[0][0].device
        comp = torch.cuda.current_stream(dev)
        est = self._side_stream(dev)
        est.wait_stream(comp)  # inputs produced on the current stream are visible to estimation
        results = []

        def build(layer):
            q, k, _ = layers[layer]
            cfgs = self.table.layer(layer)
            b = self.table.block_size(layer, self.default_block)
            with torch.cuda.stream(est):
                lay = build_layer_layout(q, k, cfgs, b, stream=est, groups=self.table.device_groups(layer, dev))
                ev = torch.cuda.Event()
                ev.record(est)
            return lay, ev, b

        nxt = build(0)
        for layer, (q, k, v) in enumerate(layers):
            lay, ev, b = nxt
            comp.wait_event(ev)
            for t in (lay.tiles, lay.tile_offsets, lay.cols, lay.col_offsets):
                t.record_stream(comp)  # allocated on the side stream, read by the attention
            out = outs[layer] if outs is not None else torch.empty_like(q)
            self._attend(layer, q, k, v, lay, b, out, comp, attn_events)
            results.append(out)
            if after_layer is not None:
                after_layer(layer, out)
            if layer + 1 < len(layers):
                nxt = build(layer + 1)  # its host read-back waits for the side stream only
        return results

    def __call__(self, layers_qkv, stream=None):
        """``layers_qkv``: iterable of (q, k, v) per layer, in layer order; yields outputs."""
        for layer, (q, k, v) in enumerate(layers_qkv):
            if layer >= self.table.n_layers:
                raise ValueError(f"more layers than the pattern table holds ({self.table.n_layers})")
            yield self.layer(layer, q, k, v, stream=stream)
