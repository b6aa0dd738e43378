"""Per-head run reports computed on the GPU.

Mirror of the reference's report module (/root/reference/pkg/src/sparseprefill/
metrics.py:30-95) with the two S x S computations replaced by streaming ones:

* dense ground truth -- the reference materialises the causal probability
  matrix (attention_ref.py:65-75); here the same sm_100a kernel runs a dense
  causal layout (every aligned tile of every row, ``dense_layout``) and
  returns the dense output and each row's log-sum-exp;
* ``attention_recall`` -- the reference sums probs[mask] / probs.sum()
  (attention_ref.py:128-139).  Per row, the mass a layout keeps is
  sum_{j in cells(i)} p_ij = exp(lse_layout(i) - lse_dense(i)), and every
  causal row's probabilities sum to one, so a head's recall is the mean of
  that ratio over its rows: two kernel passes, O(S) memory.

``report_layer`` reports every head of a layer from one sparse and one dense
launch; ``report_head`` keeps the reference's single-head NumPy signature.
Recall and output error use the kernel's arithmetic (bf16 tensor cores; fp32
inputs go through the bf16x2 split), so they agree with the reference's fp64
values to ~1e-5 (fp32 inputs), not bit for bit; sparsity and modeled FLOPs are
exact integers.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, kernels
from .patterns import (PATTERN_NAMES, AShape, BlockSparse, HeadPatternConfig, SparseLayout, causal_area,
                       flops_in_kernel, layout_area)
from .prefill import LayerLayout, build_layer_layout

CSV_COLUMNS = ["head", "pattern", "recall", "kernel_sparsity", "modeled_flops", "output_mae"]
CSV_TIMING_COLUMNS = ["t_estimate", "t_sparse"]


@dataclass
class RunReport:
    head: str
    pattern: str
    recall: float
    kernel_sparsity: float
    modeled_flops: int
    output_mae: float
    t_estimate: float
    t_sparse: float


def kernel_sparsity(layout: SparseLayout) -> float:
    """metrics.py:43-45: fraction of causal cells the kernel does NOT compute."""
    return 1.0 - layout_area(layout) / causal_area(layout.seq_len)


def modeled_kernel_sparsity(cfg: HeadPatternConfig, seq_len: int, block_size: int) -> float:
    """metrics.py:48-51: sparsity from the cost model alone (head_dim cancels)."""
    area = flops_in_kernel(cfg, seq_len, 1, block_size) / 4
    return 1.0 - area / causal_area(seq_len)


def dense_layout(q: torch.Tensor, k: torch.Tensor, block_size: int = 64, stream=None) -> LayerLayout:
    """Every aligned causal tile of every query-block row (the dense causal mask at
    kernel granularity: AShape with one sink token and a window of S)."""
    hq, s_len, _ = q.shape
    return build_layer_layout(q, k, [AShape(1, s_len)] * hq, block_size, stream)


def _attention_with_lse(q, k, v, lay: LayerLayout, scale: float, stream=None):
    lse = torch.empty(q.shape[0], q.shape[1], dtype=torch.float32, device=q.device)
    out = kernels.sparse_flash_attention_gpu(q, k, v, scale, lay.block_size, lay.tiles, lay.tile_offsets, lay.cols,
                                             lay.col_offsets, stream=stream, lse=lse)
    return out, lse


def recall_from_lse(lse_layout: torch.Tensor, lse_dense: torch.Tensor) -> torch.Tensor:
    """Per-head recall [H] (fp64) from per-row log-sum-exps [H, S]."""
    ratio = torch.exp(lse_layout.double() - lse_dense.double())
    ratio = torch.where(torch.isfinite(lse_layout) & torch.isfinite(lse_dense), ratio, torch.zeros_like(ratio))
    rows = torch.isfinite(lse_dense).sum(dim=1).clamp(min=1)
    return ratio.sum(dim=1) / rows


def attention_recall_gpu(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: LayerLayout,
                         scale: float | None = None, dense: tuple | None = None) -> torch.Tensor:
    """Fraction of dense causal attention mass each head's layout covers
    (attention_ref.py:128-139), [Hq] fp64 on the device.  ``dense`` may pass a
    precomputed (out, lse) of the dense layout."""
    sc = 1.0 / math.sqrt(q.shape[-1]) if scale is None else float(scale)
    if dense is None:
        dense = _attention_with_lse(q, k, v, dense_layout(q, k, layout.block_size), sc)
    _, lse_s = _attention_with_lse(q, k, v, layout, sc)
    return recall_from_lse(lse_s, dense[1])


def _elapsed(fn, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    res = fn()
    e1.record(s)
    e1.synchronize()
    return res, e0.elapsed_time(e1) * 1e-3


def report_layer(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, head_cfgs, block_size: int = 64,
                 scale: float | None = None, head_names=None, stream=None) -> list[RunReport]:
    """One report per q-head of a layer (metrics.py:54-70 for every head at once).

    t_estimate / t_sparse are the layer's device times (estimation + index, attention)
    divided evenly over its heads."""
    dev = _dev.require_cuda(q.device)
    hq, s_len, d = q.shape
    sc = 1.0 / math.sqrt(d) if scale is None else float(scale)
    with torch.cuda.device(dev):
        lay, t_est = _elapsed(lambda: build_layer_layout(q, k, head_cfgs, block_size, stream), stream)
        (out, lse_s), t_sp = _elapsed(lambda: _attention_with_lse(q, k, v, lay, sc, stream), stream)
        dense_out, lse_d = _attention_with_lse(q, k, v, dense_layout(q, k, block_size, stream), sc, stream)
        mae = (out.double() - dense_out.double()).abs().mean(dim=(1, 2))
        recall = recall_from_lse(lse_s, lse_d)
        area = lay.area()
        vals = torch.stack([recall, mae, area.double()]).cpu().numpy()
    total = causal_area(s_len)
    names = head_names if head_names is not None else [str(h) for h in range(hq)]
    reports = []
    for h, cfg in enumerate(head_cfgs):
        reports.append(RunReport(
            head=names[h], pattern=PATTERN_NAMES[type(cfg)], recall=float(vals[0, h]),
            kernel_sparsity=1.0 - int(vals[2, h]) / total,
            modeled_flops=flops_in_kernel(cfg, s_len, d, block_size), output_mae=float(vals[1, h]),
            t_estimate=t_est / hq, t_sparse=t_sp / hq))
    return reports


def report_head(inputs, cfg: HeadPatternConfig, head: str = "0", block_size: int = 64) -> RunReport:
    """metrics.py:54-70 on the GPU: ``inputs`` is a sparse_attn.AttentionInputs (fp32 [S, d])."""
    dev = _dev.require_cuda()
    q = torch.from_numpy(np.ascontiguousarray(inputs.q, dtype=np.float32)).to(dev)[None]
    k = torch.from_numpy(np.ascontiguousarray(inputs.k, dtype=np.float32)).to(dev)[None]
    v = torch.from_numpy(np.ascontiguousarray(inputs.v, dtype=np.float32)).to(dev)[None]
    bs = cfg.block_size if isinstance(cfg, BlockSparse) else block_size  # sparse_attn.py:87-90
    rep = report_layer(q, k, v, [cfg], bs, inputs.scale, head_names=[head])[0]
    # the reference models FLOPs with the caller's block size
    rep.modeled_flops = flops_in_kernel(cfg, inputs.seq_len, inputs.head_dim, block_size)
    return rep


def _format_value(value) -> str:
    return format(value, ".10g") if isinstance(value, float) else str(value)


def reports_to_csv(reports: list[RunReport], path, include_timings: bool = False) -> None:
    """metrics.py:79-86: fixed column order, header row."""
    columns = CSV_COLUMNS + (CSV_TIMING_COLUMNS if include_timings else [])
    lines = [",".join(columns)] + [",".join(_format_value(getattr(r, c)) for c in columns) for r in reports]
    with open(path, "w", newline="") as f:
        f.write("\n".join(lines) + "\n")


def reports_to_json(reports: list[RunReport], path) -> None:
    """metrics.py:89-95."""
    rows = [{c: getattr(r, c) for c in CSV_COLUMNS + CSV_TIMING_COLUMNS} for r in reports]
    with open(path, "w") as f:
        json.dump(rows, f, indent=2)
        f.write("\n")
