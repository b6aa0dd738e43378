"""The kernel plugin: a ``b200`` backend with the reference's backend contract.

Mirrors /root/reference/pkg/src/sparseprefill/kernels.py:

* ``BACKEND_NAME`` + ``sparse_flash_rows(q, k, v, scale, block_size,
  tile_starts, tile_offsets, col_indices, col_offsets)`` is the exact module
  contract of ``_core.pyx:72-82`` / ``_core_py.py:17-27`` (NumPy fp32 in, a
  newly allocated NumPy fp32 [S, d] out, int64 CSR layout), so this module can
  be dropped into the reference's backend dict;
* ``sparse_flash_attention(q, k, v, scale, block_size, tile_starts,
  column_indices, backend=None)`` keeps kernels.py:38-70 (row-count
  ``ValueError``, per-row list flattening, optional explicit backend module);
* ``available_backends()`` keeps kernels.py:73-82.

All compute runs in libspf.so on the GPU (fp32 I/O is handled by the bf16x2
split path of the sm_100a kernel); there is no CPU fallback.
``sparse_flash_attention_gpu`` is the batched multi-head torch entry used by
the production pipeline (bf16, GQA).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib

BACKEND_NAME = "b200"
BACKEND = BACKEND_NAME


def _flatten(per_row, n_rows: int):
    """kernels.py:28-35: per-row lists -> (flat int64, offsets int64)."""
    off = np.zeros(n_rows + 1, dtype=np.int64)
    for r in range(n_rows):
        off[r + 1] = off[r] + len(per_row[r])
    flat = np.fromiter((int(x) for row in per_row for x in row), dtype=np.int64, count=int(off[-1]))
    return flat, off


def _pair_list(pair_heads, hq: int, dev) -> torch.Tensor | None:
    """Device int32 list of the paired-box kernel's heads (see sparse_flash_attention_gpu)."""
    if pair_heads is None:
        return None
    if not isinstance(pair_heads, torch.Tensor):
        pair_heads = torch.as_tensor(pair_heads)
    if pair_heads.dtype in (torch.bool, torch.uint8):
        if pair_heads.numel() != hq:
            raise ValueError("a pair_heads mask must have one entry per q-head")
        pair_heads = torch.nonzero(pair_heads.reshape(-1)).reshape(-1)
    elif pair_heads.dtype not in (torch.int32, torch.int64):
        raise ValueError("pair_heads must be a head-id list or a bool/uint8 mask")
    if pair_heads.numel() == 0:
        return None
    if pair_heads.numel() > hq:
        raise ValueError("more pair heads than q-heads")
    if pair_heads.device.type == "cpu":  # host ids: validate here (device lists are routed by the
        ids = pair_heads.reshape(-1)    # library, which never leaves a head unwritten)
        if int(ids.min()) < 0 or int(ids.max()) >= hq:
            raise ValueError(f"pair head ids must lie in [0, {hq})")
        if torch.unique(ids).numel() != ids.numel():
            raise ValueError("pair head ids must be distinct")
    return pair_heads.to(device=dev, dtype=torch.int32).contiguous()


def sparse_flash_attention_gpu(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float, block_size: int,
                               tile_starts: torch.Tensor, tile_offsets: torch.Tensor, col_indices: torch.Tensor,
                               col_offsets: torch.Tensor, out: torch.Tensor | None = None,
                               stream: torch.cuda.Stream | None = None,
                               lse: torch.Tensor | None = None,
                               pair_heads: torch.Tensor | None = None) -> torch.Tensor:
    """Batched sparse FlashAttention on device tensors.

    q [Hq, S, d], k/v [Hkv, S, d] (bf16 or fp32, contiguous, same dtype);
    CSR over (head, row): offsets int64 [Hq*n_rows+1], entries int32.
    Returns out [Hq, S, d] in the input dtype.  ``lse`` (optional fp32 [Hq, S])
    receives each row's natural-log sum of exp(scale * q.k) over its cells.
    ``pair_heads`` (optional) names candidate heads for the paired-box kernel (Block-Sparse
    heads, whose row blocks rarely share tiles); the library measures each listed head's
    layout on the device and runs it there only when it has no residual columns and the
    paired steps beat the union steps (include/spf.h, spf_sparse_flash_rows_ex); every other
    head runs the union kernel.  Either a device int32 tensor of head ids (the hot path: its
    length is host metadata, no sync), a host id list (validated: distinct, in range), or a
    bool / uint8 [Hq] mask (converted here).
    """
    dev = _dev.require_cuda(q.device)
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
        raise ValueError("q/k/v must be [heads, seq_len, head_dim]")
    hq, s_len, d = q.shape
    hkv = k.shape[0]
    if k.shape != (hkv, s_len, d) or v.shape != k.shape:
        raise ValueError("k/v shape mismatch")
    if q.dtype != k.dtype or q.dtype != v.dtype or q.dtype not in (torch.bfloat16, torch.float32):
        raise TypeError("q/k/v must share dtype bf16 or fp32")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    dtype = _lib.SPF_DTYPE_BF16 if q.dtype == torch.bfloat16 else _lib.SPF_DTYPE_F32
    n_rows = (s_len + block_size - 1) // block_size
    if tile_offsets.numel() != hq * n_rows + 1 or col_offsets.numel() != hq * n_rows + 1:
        raise ValueError("need one tile list and one column list per query-block row")
    if out is None:
        out = torch.empty_like(q)
    lib = _lib.load()
    ws_bytes = lib.spf_sparse_flash_workspace_size(dtype, hq, hkv, s_len, d)
    ws = _dev.workspace(ws_bytes, dev, stream)
    ts = tile_starts if tile_starts.numel() else None
    cs = col_indices if col_indices.numel() else None
    if lse is not None and (lse.dtype != torch.float32 or lse.numel() != hq * s_len or not lse.is_contiguous()):
        raise ValueError("lse must be a contiguous fp32 [Hq, S] tensor")
    pair_list = _pair_list(pair_heads, hq, dev)
    _lib.check(lib.spf_sparse_flash_rows_ex(
        dtype, _dev.ptr(q), _dev.ptr(k), _dev.ptr(v), hq, hkv, s_len, d, float(scale), int(block_size),
        _dev.ptr(ts), _dev.ptr(tile_offsets), _dev.ptr(cs), _dev.ptr(col_offsets), _dev.ptr(pair_list),
        0 if pair_list is None else int(pair_list.numel()), _dev.ptr(out), _dev.ptr(lse), _dev.ptr(ws), ws_bytes, _dev.stream_handle(stream)), "spf_sparse_flash_rows_ex")
    return out


def sparse_flash_rows(q, k, v, scale, block_size, tile_starts, tile_offsets, col_indices, col_offsets):
    """Backend-module contract of _core.pyx:72-82 (single head, NumPy fp32)."""
    dev = _dev.require_cuda()
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    if q.ndim != 2 or k.shape != q.shape or v.shape != q.shape:
        raise ValueError("q, k, v must share the same [S, d] shape")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    tq = torch.from_numpy(q).to(dev).unsqueeze(0)
    tk = torch.from_numpy(k).to(dev).unsqueeze(0)
    tv = torch.from_numpy(v).to(dev).unsqueeze(0)
    out = sparse_flash_attention_gpu(
        tq, tk, tv, float(scale), int(block_size),
        _dev.to_device_i32(tile_starts, dev), _dev.to_device_i64(tile_offsets, dev),
        _dev.to_device_i32(col_indices, dev), _dev.to_device_i64(col_offsets, dev))
    return out[0].cpu().numpy()


def sparse_flash_attention(q, k, v, scale: float, block_size: int, tile_starts: list, column_indices: list,
                           backend=None) -> np.ndarray:
    """kernels.py:38-70 with the b200 backend as the default implementation."""
    s_len = np.asarray(q).shape[0]
    n_rows = (s_len + block_size - 1) // block_size
    if len(tile_starts) != n_rows or len(column_indices) != n_rows:
        raise ValueError("need one tile list and one column list per query-block row")
    starts_flat, starts_off = _flatten(tile_starts, n_rows)
    cols_flat, cols_off = _flatten(column_indices, n_rows)
    impl = backend if backend is not None else _this_module()
    return impl.sparse_flash_rows(
        np.ascontiguousarray(q, dtype=np.float32), np.ascontiguousarray(k, dtype=np.float32),
        np.ascontiguousarray(v, dtype=np.float32), float(scale), int(block_size),
        starts_flat, starts_off, cols_flat, cols_off)


def _this_module():
    import sys

    return sys.modules[__name__]


def available_backends() -> dict:
    """kernels.py:73-82: importable kernel backends by name."""
    return {BACKEND_NAME: _this_module()}
