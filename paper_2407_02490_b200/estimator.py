"""Online sparsity estimation on the GPU.

Drop-in mirror of /root/reference/pkg/src/sparseprefill/estimator.py:

* ``VSIndices`` / ``BlockIndices`` (estimator.py:20-56) with the same
  ordering/causality validation;
* ``argtopk`` (59-67): stable descending order, ties to the lower index;
* ``estimate_vertical_slash(q, k, cfg)`` (82-114) and
  ``estimate_block_sparse(q, k, cfg)`` (117-143) take NumPy [S, d] arrays
  like the reference (fp32).  They call the production entry (mode "fast"),
  whose tensor-core path takes bf16 inputs only, so fp32 inputs run libspf's
  fp64 estimation kernels (the SPF_VS_EXACT path / spf_bs_estimate) and the
  selected index sets are the reference's.  bf16 device tensors (the
  production path) score on the tensor cores; a head's selection is kept only
  when a rigorous bound on the score error separates its top-k boundary
  (estimate_vs_tc.cu), otherwise the head is re-run on the fp64 path in the
  same call -- the sets equal the fp64 path's either way.

``estimate_vertical_slash_gpu`` / ``estimate_block_sparse_gpu`` are the
batched multi-head (GQA) device entries used by ``prefill.py``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib, layouts
from .patterns import BlockSparse, VerticalSlash, n_block_rows


@dataclass(frozen=True)
class VSIndices:
    """Selected key columns (ascending) and slash offsets (descending).

    Offset o means the diagonal key = query - o.
    """

    vertical: np.ndarray
    slash: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.vertical, dtype=np.int64)
        s = np.asarray(self.slash, dtype=np.int64)
        object.__setattr__(self, "vertical", v)
        object.__setattr__(self, "slash", s)
        if v.size and np.any(np.diff(v) <= 0):
            raise ValueError("vertical indices must be strictly ascending")
        if s.size and np.any(np.diff(s) >= 0):
            raise ValueError("slash offsets must be strictly descending")
        if (v.size and v.min() < 0) or (s.size and s.min() < 0):
            raise ValueError("indices must be non-negative")


@dataclass(frozen=True)
class BlockIndices:
    """Per query-block row: sorted selected key-block indices (b <= row)."""

    rows: tuple

    def __post_init__(self):
        rows = tuple(tuple(int(b) for b in row) for row in self.rows)
        object.__setattr__(self, "rows", rows)
        for r, row in enumerate(rows):
            if any(row[i] >= row[i + 1] for i in range(len(row) - 1)):
                raise ValueError(f"row {r}: block indices must be strictly ascending")
            if any(b < 0 or b > r for b in row):
                raise ValueError(f"row {r}: block index outside causal range")


ARGTOPK_MAX_K = 16384


def argtopk(values, k: int) -> np.ndarray:
    """estimator.py:59-67: indices of the k largest values in descending-value
    order, ties toward the smaller index -- spf_argtopk (radix select + bitonic
    ordering of the k picks on the device)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    dev = _dev.require_cuda()
    vals = torch.as_tensor(np.asarray(values, dtype=np.float64).reshape(-1), device=dev).contiguous()
    n = int(vals.numel())
    m = min(int(k), n)
    if m == 0:
        return np.zeros(0, dtype=np.int64)
    if m > ARGTOPK_MAX_K:
        raise ValueError(f"argtopk supports k <= {ARGTOPK_MAX_K} on the device (got {m})")
    lib = _lib.load()
    out = torch.empty(m, dtype=torch.int32, device=dev)
    ws_bytes = lib.spf_argtopk_workspace_size(n)
    ws = _dev.workspace(ws_bytes, dev)
    _lib.check(lib.spf_argtopk(_dev.ptr(vals), n, m, _dev.ptr(out), _dev.ptr(ws), ws_bytes, _dev.stream_handle()),
               "spf_argtopk")
    return out.cpu().numpy().astype(np.int64)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SPF_DTYPE_BF16
    if t.dtype == torch.float32:
        return _lib.SPF_DTYPE_F32
    raise TypeError("q/k must be bf16 or fp32")


def vs_estimate_async(q: torch.Tensor, k: torch.Tensor, cfg: VerticalSlash, head_ids=None, mode: str = "fast",
                      with_scores: bool = False, stream=None):
    """One stream-ordered spf_vs_estimate call (no host sync).

    Returns (vertical, slash, vscore, sscore, uncertain): vertical
    [n, min(k_v, S)] int32 ascending, slash [n, min(k_s, S)] int32 descending,
    fp64 score vectors [n, S] (or None) and the per-head int32 flags of the
    tensor-core path (1 = the selection was too close to certify and the head
    was re-estimated on the fp64 path inside the same call).
    """
    dev = _dev.require_cuda(q.device)
    hq, s_len, d = q.shape
    hkv = k.shape[0]
    if cfg.last_q > s_len:
        raise ValueError(f"last_q={cfg.last_q} exceeds seq_len={s_len}")
    n = hq if head_ids is None else int(head_ids.numel())
    kv, ks = min(cfg.k_v, s_len), min(cfg.k_s, s_len)
    vert = torch.empty((n, kv), dtype=torch.int32, device=dev)
    sl = torch.empty((n, ks), dtype=torch.int32, device=dev)
    vsc = torch.empty((n, s_len), dtype=torch.float64, device=dev) if with_scores else None
    ssc = torch.empty((n, s_len), dtype=torch.float64, device=dev) if with_scores else None
    flags = torch.empty(n, dtype=torch.int32, device=dev)
    codes = {"fast": _lib.SPF_VS_FAST, "exact": _lib.SPF_VS_EXACT, "uncertified": _lib.SPF_VS_FAST_UNCERTIFIED}
    if mode not in codes:
        raise ValueError(f"unknown estimation mode {mode!r}")
    code = codes[mode]
    dt = _dtype_code(q)
    lib = _lib.load()
    ws_bytes = lib.spf_vs_estimate_workspace_size(code, dt, hq, hkv, n, s_len, d, cfg.last_q)
    ws = _dev.workspace(ws_bytes, dev, stream)
    _lib.check(lib.spf_vs_estimate(code, dt, _dev.ptr(q.contiguous()), _dev.ptr(k.contiguous()), hq, hkv, s_len, d,
                                   _dev.ptr(head_ids), n, cfg.last_q, cfg.k_v, cfg.k_s, _dev.ptr(vert), _dev.ptr(sl),
                                   _dev.ptr(vsc), _dev.ptr(ssc), _dev.ptr(flags), _dev.ptr(ws), ws_bytes,
                                   _dev.stream_handle(stream)), "spf_vs_estimate")
    return vert, sl, vsc, ssc, flags


def estimate_vertical_slash_gpu(q: torch.Tensor, k: torch.Tensor, cfg: VerticalSlash, head_ids=None,
                                with_scores: bool = False, stream=None, mode: str = "fast"):
    """Batched VS estimation: q [Hq, S, d], k [Hkv, S, d] (bf16/fp32).

    Returns (vertical [n, min(k_v, S)] int32 ascending, slash [n, min(k_s, S)]
    int32 descending[, vscore, sscore fp64 [n, S]]) for the heads in
    ``head_ids`` (int32 device tensor; None = all q-heads).  ``mode="fast"``
    runs the tensor-core path (uncertified heads are re-run on the fp64 path
    in the same stream); ``mode="exact"`` runs the fp64 path only.
    """
    vert, sl, vsc, ssc, _ = vs_estimate_async(q, k, cfg, head_ids, mode, with_scores, stream)
    if with_scores:
        return vert, sl, vsc, ssc
    return vert, sl


def bs_workspace_bytes(hq, hkv, s_len, d, block_size, n_heads) -> int:
    n = n_block_rows(s_len, block_size)
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    return al(hq * n * d * 4) + al(hkv * n * d * 4) + al(n_heads * n * n * 8)


def estimate_block_sparse_gpu(q: torch.Tensor, k: torch.Tensor, cfg: BlockSparse, head_ids, tile_offsets,
                              tile_starts, stream=None):
    """Batched BS estimation writing tile starts into an existing CSR."""
    dev = _dev.require_cuda(q.device)
    hq, s_len, d = q.shape
    hkv = k.shape[0]
    n = hq if head_ids is None else int(head_ids.numel())
    lib = _lib.load()
    ws_bytes = bs_workspace_bytes(hq, hkv, s_len, d, cfg.block_size, n)
    ws = _dev.workspace(ws_bytes, dev, stream)
    _lib.check(lib.spf_bs_estimate(_dtype_code(q), _dev.ptr(q.contiguous()), _dev.ptr(k.contiguous()), hq, hkv, s_len,
                                   d, _dev.ptr(head_ids), n, cfg.k_b, cfg.block_size, _dev.ptr(tile_offsets),
                                   _dev.ptr(tile_starts), _dev.ptr(ws), ws_bytes, _dev.stream_handle(stream)),
               "spf_bs_estimate")


def _as_device_matrix(x, dev) -> torch.Tensor:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if a.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return torch.from_numpy(a).to(dev).unsqueeze(0)


def estimate_vertical_slash(q, k, cfg: VerticalSlash) -> VSIndices:
    """estimator.py:82-114 (single head, NumPy in, VSIndices out)."""
    dev = _dev.require_cuda()
    tq, tk = _as_device_matrix(q, dev), _as_device_matrix(k, dev)
    vert, sl = estimate_vertical_slash_gpu(tq, tk, cfg)
    return VSIndices(vertical=vert[0].cpu().numpy().astype(np.int64), slash=sl[0].cpu().numpy().astype(np.int64))


def estimate_block_sparse(q, k, cfg: BlockSparse) -> BlockIndices:
    """estimator.py:117-143 (single head, NumPy in, BlockIndices out)."""
    dev = _dev.require_cuda()
    tq, tk = _as_device_matrix(q, dev), _as_device_matrix(k, dev)
    s_len = tq.shape[1]
    b = cfg.block_size
    n = n_block_rows(s_len, b)
    cnt = torch.zeros(n, dtype=torch.int64, device=dev)
    layouts.bs_count(None, 1, s_len, b, cfg.k_b, cnt)
    toff, total = layouts.csr_offsets(cnt)
    tiles = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    estimate_block_sparse_gpu(tq, tk, cfg, None, toff, tiles)
    t = tiles[:total].cpu().numpy().astype(np.int64) // b
    off = toff.cpu().numpy()
    return BlockIndices(rows=tuple(tuple(int(x) for x in t[off[r]: off[r + 1]]) for r in range(n)))
