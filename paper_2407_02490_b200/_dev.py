"""Device plumbing for the ctypes boundary: torch owns memory and streams."""

from __future__ import annotations

import ctypes

import numpy as np
import torch


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_02490_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    major, minor = torch.cuda.get_device_capability(dev)
    if (major, minor) != (10, 0):
        raise RuntimeError(f"libspf is compiled for sm_100a only; device is sm_{major}{minor}")
    return dev


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


_ws_cache: dict = {}


def workspace(nbytes: int, device, stream=None) -> torch.Tensor | None:
    """Grow-only scratch buffer per (device, stream): work ordered on one stream reuses
    it in stream order, and two streams never share one (include/spf.h: the library is
    re-entrant per stream with caller-owned workspaces)."""
    if nbytes <= 0:
        return None
    dev = torch.device(device)
    s = torch.cuda.current_stream(dev) if stream is None else stream
    key = (dev.type, dev.index, int(s.cuda_stream))
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        with torch.cuda.stream(s):  # owned by (allocated on) the stream that uses it
            buf = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return buf


def to_device_i32(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int32).contiguous()
    arr = np.asarray(a, dtype=np.int64)
    if arr.size and (arr.max() > np.iinfo(np.int32).max or arr.min() < np.iinfo(np.int32).min):
        raise ValueError("layout entries exceed int32 range")
    return torch.from_numpy(np.ascontiguousarray(arr.astype(np.int32))).to(device)


def to_device_i64(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).to(device)
