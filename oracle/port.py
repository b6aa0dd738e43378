"""CPU restatement of the reference's sparse pre-fill path -- TEST INFRASTRUCTURE.

This module is the *checker* for the B200 implementation.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product package never does
(the product path fails loudly when its CUDA library is missing).

Every function restates the reference algorithm at the cited
``/root/reference/pkg/src/sparseprefill/<file>:<line>``; rounding points
(fp64 accumulation, fp32 storage) follow the reference exactly because the
index-set parity gate is bit-exact.  Parity of this port is pinned two ways:

* ``tests/golden/*.npz`` -- vectors produced by importing the reference
  package itself (``tests/golden/make_golden.py``), checked in
  ``tests/test_oracle_golden.py``;
* ``oracle/_ref/spf_ref_core*.so`` -- the reference's own Cython kernel
  compiled from /root/reference by ``oracle/Makefile``; when present the tests
  check this port's ``sparse_flash_rows`` against it bit-for-bit.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

STORAGE = np.float32
ACCUM = np.float64
MASK_SENTINEL = float(np.finfo(np.float32).min)  # tensor.py:18

_HERE = os.path.dirname(os.path.abspath(__file__))


# --------------------------------------------------------------------------
# tensor.py
# --------------------------------------------------------------------------
def seeded_gaussian(rows: int, cols: int, seed: int) -> np.ndarray:
    """tensor.py:81-90: PCG64 + ziggurat standard normal, stored fp32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((rows, cols)).astype(STORAGE)


def softmax_rows(scores) -> np.ndarray:
    """tensor.py:61-78: fp64 softmax, sentinel-masked cells -> exactly 0,
    fully-masked rows -> zeros, result rounded to fp32."""
    s = np.asarray(scores, dtype=ACCUM)
    masked = s <= MASK_SENTINEL
    s = np.where(masked, -np.inf, s)
    if s.shape[1]:
        mx = np.max(s, axis=1, keepdims=True)
    else:
        mx = np.zeros((s.shape[0], 1))
    mx = np.where(np.isfinite(mx), mx, 0.0)
    e = np.exp(s - mx)
    e[masked] = 0.0
    den = e.sum(axis=1, keepdims=True)
    out = np.divide(e, den, out=np.zeros_like(e), where=den > 0)
    return out.astype(STORAGE)


def mean_pool_rows(m, block: int) -> np.ndarray:
    """tensor.py:43-58: fp64 block sums (trailing block divided by its real
    length), rounded to fp32."""
    m = np.asarray(m)
    n = m.shape[0]
    starts = np.arange(0, n, block)
    sums = np.add.reduceat(m.astype(ACCUM), starts, axis=0)
    lens = np.minimum(starts + block, n) - starts
    return (sums / lens[:, None]).astype(STORAGE)


# --------------------------------------------------------------------------
# estimator.py
# --------------------------------------------------------------------------
def argtopk(values, k: int) -> np.ndarray:
    """estimator.py:59-67: stable descending order, ties -> lower index."""
    values = np.asarray(values)
    order = np.argsort(-values, kind="stable")
    return order[: min(k, values.size)].astype(np.int64)


def force_include(selected: np.ndarray, index: int) -> np.ndarray:
    """estimator.py:70-79: overwrite the weakest (last) pick when missing."""
    if index in selected:
        return selected
    out = selected.copy()
    out[-1] = index
    return out


def vs_scores(q, k, last_q: int):
    """estimator.py:99-110: fp32-rounded tail-row probabilities summed in
    fp64 per column (vertical) and per diagonal offset (slash)."""
    q = np.asarray(q)
    k = np.asarray(k)
    s_len, d = q.shape
    scale = 1.0 / math.sqrt(d)
    q_tail = q[s_len - last_q:].astype(ACCUM)
    scores = scale * (q_tail @ k.astype(ACCUM).T)
    abs_q = np.arange(s_len - last_q, s_len)
    keys = np.arange(s_len)
    scores[abs_q[:, None] < keys[None, :]] = MASK_SENTINEL
    est = softmax_rows(scores).astype(ACCUM)
    vertical = est.sum(axis=0)
    offsets = abs_q[:, None] - keys[None, :]
    causal = offsets >= 0
    slash = np.bincount(offsets[causal].ravel(), weights=est[causal].ravel(), minlength=s_len)
    return vertical, slash


def estimate_vertical_slash(q, k, k_v: int, k_s: int, last_q: int = 64):
    """estimator.py:82-114 -> (vertical ascending, slash descending) int64."""
    s_len = np.asarray(q).shape[0]
    if last_q > s_len:
        raise ValueError(f"last_q={last_q} exceeds seq_len={s_len}")
    kv = min(k_v, s_len)
    ks = min(k_s, s_len)
    vertical, slash = vs_scores(q, k, last_q)
    v = force_include(argtopk(vertical, kv), 0)
    s = force_include(argtopk(slash, ks), 0)
    return np.sort(v), -np.sort(-s)


def bs_probabilities(q, k, block: int) -> np.ndarray:
    """estimator.py:127-136: pooled fp64 scores, block-causal, fp32 softmax."""
    q = np.asarray(q)
    k = np.asarray(k)
    s_len, d = q.shape
    scale = 1.0 / math.sqrt(d)
    qp = mean_pool_rows(q, block).astype(ACCUM)
    kp = mean_pool_rows(k, block).astype(ACCUM)
    scores = scale * (qp @ kp.T)
    n = (s_len + block - 1) // block
    r = np.arange(n)
    scores[r[:, None] < r[None, :]] = MASK_SENTINEL
    return softmax_rows(scores).astype(ACCUM)


def estimate_block_sparse(q, k, k_b: int, block: int = 64):
    """estimator.py:117-143 -> tuple of ascending block-index tuples."""
    est = bs_probabilities(q, k, block)
    rows = []
    for r in range(est.shape[0]):
        k_eff = min(k_b, r + 1)
        sel = force_include(argtopk(est[r, : r + 1], k_eff), r)
        rows.append(tuple(sorted(int(x) for x in sel)))
    return tuple(rows)


# --------------------------------------------------------------------------
# vs_index.py  (pure-Python restatement + the C restatement in vs_merge.c)
# --------------------------------------------------------------------------
def build_vs_layout_with_stats(vertical, slash, seq_len: int, block: int):
    """vs_index.py:28-95.  Returns (tile_starts per row, cols per row, ops)."""
    if block < 1:
        raise ValueError("block_size must be >= 1")
    pts = [int(x) for x in np.asarray(vertical, dtype=np.int64)]
    sls = [int(x) for x in np.asarray(slash, dtype=np.int64)]
    if pts and (max(pts) >= seq_len or min(pts) < 0):
        raise ValueError("vertical index out of range")
    if sls and (max(sls) >= seq_len or min(sls) < 0):
        raise ValueError("slash offset out of range")
    b = block
    tiles_all, cols_all, ops_all = [], [], []
    for r in range((seq_len + b - 1) // b):
        q_start = r * b
        q_end = min(q_start + b, seq_len)
        tiles, cols = [], []
        state = {"jv": 0, "ops": 0}

        def cov(cs, ce):
            return cs + -(-(ce - cs) // b) * b

        def flush(cs, ce):
            ce_cov = cov(cs, ce)
            while state["jv"] < len(pts) and pts[state["jv"]] < ce_cov:
                if pts[state["jv"]] < cs:
                    cols.append(pts[state["jv"]])
                state["jv"] += 1
                state["ops"] += 1
            s = cs
            while s < ce:
                tiles.append(s)
                s += b
                state["ops"] += 1

        cur = None
        for o in sls:
            if o >= q_end:
                continue
            state["ops"] += 1
            rs, re = max(0, q_start - o), q_end - o
            if cur is None:
                cur = [rs, re]
            elif rs <= cur[1] or rs < cov(cur[0], cur[1]):
                cur[1] = max(cur[1], re)
            else:
                flush(cur[0], cur[1])
                cur = [rs, re]
        if cur is not None:
            flush(cur[0], cur[1])
        while state["jv"] < len(pts):
            if pts[state["jv"]] < q_end:
                cols.append(pts[state["jv"]])
            state["jv"] += 1
            state["ops"] += 1
        tiles_all.append(tiles)
        cols_all.append(cols)
        ops_all.append(state["ops"])
    return tiles_all, cols_all, ops_all


def _vs_lib():
    path = os.path.join(_HERE, "liboracle_vs.so")
    if not os.path.exists(path):
        import subprocess

        subprocess.run(["make", "-s", "-C", _HERE, "restate"], check=True)
    lib = ctypes.CDLL(path)
    p = ctypes.POINTER(ctypes.c_int64)
    i64 = ctypes.c_int64
    lib.oracle_vs_count.argtypes = [p, i64, p, i64, i64, i64, p, p, p]
    lib.oracle_vs_fill.argtypes = [p, i64, p, i64, i64, i64, p, p, p, p]
    return lib


def build_vs_csr(vertical, slash, seq_len: int, block: int):
    """Same algorithm through oracle/vs_merge.c; returns CSR int64 arrays
    (tile_starts, tile_offsets, col_indices, col_offsets)."""
    lib = _vs_lib()
    pts = np.ascontiguousarray(vertical, dtype=np.int64)
    sls = np.ascontiguousarray(slash, dtype=np.int64)
    n = (seq_len + block - 1) // block
    tc = np.zeros(n, np.int64)
    cc = np.zeros(n, np.int64)
    P = ctypes.POINTER(ctypes.c_int64)

    def ptr(a):
        return a.ctypes.data_as(P)

    lib.oracle_vs_count(ptr(pts), pts.size, ptr(sls), sls.size, seq_len, block, ptr(tc), ptr(cc), None)
    toff = np.zeros(n + 1, np.int64)
    coff = np.zeros(n + 1, np.int64)
    np.cumsum(tc, out=toff[1:])
    np.cumsum(cc, out=coff[1:])
    tiles = np.zeros(max(int(toff[-1]), 1), np.int64)
    cols = np.zeros(max(int(coff[-1]), 1), np.int64)
    lib.oracle_vs_fill(ptr(pts), pts.size, ptr(sls), sls.size, seq_len, block,
                       ptr(toff), ptr(coff), ptr(tiles), ptr(cols))
    return tiles[: toff[-1]], toff, cols[: coff[-1]], coff


# --------------------------------------------------------------------------
# patterns.py / sparse_attn.py layout builders + accounting
# --------------------------------------------------------------------------
def a_shape_layout(seq_len: int, global_tokens: int, local_window: int, block: int):
    """patterns.py:109-128 -> per-row sorted aligned tile starts."""
    out = []
    for r in range((seq_len + block - 1) // block):
        q_start, q_end = r * block, min((r + 1) * block, seq_len)
        starts = set(range(0, min(global_tokens, q_end), block))
        local_start = max(0, q_start - local_window) // block * block
        starts.update(range(local_start, q_end, block))
        out.append(sorted(starts))
    return out


def block_rows_to_tiles(rows, block: int):
    """sparse_attn.py:30-33: block index b -> tile start b*B."""
    return [[b * block for b in row] for row in rows]


def clipped_tile_cells(s, b, q_start, q_end, seq_len) -> int:
    """patterns.py:166-184."""
    lo, hi = max(s, 0), min(s + b, seq_len)
    if hi <= lo:
        return 0
    full_from = max(q_start, hi - 1)
    cells = max(0, q_end - full_from) * (hi - lo)
    ramp_lo, ramp_hi = max(q_start, lo), min(q_end, hi - 1)
    if ramp_hi > ramp_lo:
        n = ramp_hi - ramp_lo
        cells += n * ((ramp_lo + 1 - lo) + (ramp_hi - lo)) // 2
    return cells


def layout_area(seq_len, block, tiles, cols) -> int:
    """patterns.py:147-163."""
    total = 0
    for r in range(len(tiles)):
        q_start, q_end = r * block, min((r + 1) * block, seq_len)
        for s in tiles[r]:
            total += clipped_tile_cells(int(s), block, q_start, q_end, seq_len)
        total += ((len(cols[r]) + block - 1) // block) * block * (q_end - q_start)
    return total


def layout_to_mask(seq_len, block, tiles, cols) -> np.ndarray:
    """patterns.py:131-144."""
    m = np.zeros((seq_len, seq_len), dtype=bool)
    for r in range(len(tiles)):
        q0, q1 = r * block, min((r + 1) * block, seq_len)
        for s in tiles[r]:
            m[q0:q1, max(s, 0):min(s + block, seq_len)] = True
        for c in cols[r]:
            m[q0:q1, c] = True
    i = np.arange(seq_len)
    return m & (i[:, None] >= i[None, :])


# --------------------------------------------------------------------------
# attention_ref.py + the kernel contract (_core_py.py / _core.pyx)
# --------------------------------------------------------------------------
def masked_attention(q, k, v, scale, mask) -> np.ndarray:
    """attention_ref.py:78-86 (Eq. 1 with the sentinel mask), fp64 -> fp32."""
    s = scale * (np.asarray(q, ACCUM) @ np.asarray(k, ACCUM).T)
    s[~mask] = MASK_SENTINEL
    p = softmax_rows(s)
    return (p.astype(ACCUM) @ np.asarray(v, ACCUM)).astype(STORAGE)


def sparse_flash_rows(q, k, v, scale, block, tile_starts, tile_offsets, col_indices, col_offsets,
                      rows=None) -> np.ndarray:
    """_core_py.py:17-66 / _core.pyx:72-192: per query-block row, streaming
    softmax over the row's tiles (per-cell causal mask), then its residual
    columns in chips of B; fp64 state, fp32 output, zero rows when l == 0.

    ``rows`` optionally restricts the computation to a subset of row blocks
    (row-sampled parity at long S); other rows stay 0.
    """
    q64 = np.asarray(q, ACCUM)
    k64 = np.asarray(k, ACCUM)
    v64 = np.asarray(v, ACCUM)
    s_len, d = q64.shape
    b = block
    n = (s_len + b - 1) // b
    out = np.zeros((s_len, d), dtype=STORAGE)
    for r in (range(n) if rows is None else rows):
        q0, q1 = r * b, min(r * b + b, s_len)
        qs = q64[q0:q1]
        qi = np.arange(q0, q1)
        m = np.full(q1 - q0, -np.inf)
        l = np.zeros(q1 - q0)
        acc = np.zeros((q1 - q0, d))

        def update(keys, kk, vv):
            nonlocal m, l, acc
            sc = scale * (qs @ kk.T)
            sc[qi[:, None] < keys[None, :]] = -np.inf
            m_new = np.maximum(m, sc.max(axis=1))
            shift = np.where(np.isfinite(m_new), m_new, 0.0)
            p = np.exp(sc - shift[:, None])
            a = np.exp(m - shift)
            l = a * l + p.sum(axis=1)
            acc = a[:, None] * acc + p @ vv
            m = m_new

        for t in range(int(tile_offsets[r]), int(tile_offsets[r + 1])):
            s = int(tile_starts[t])
            ks, ke = max(s, 0), min(s + b, s_len)
            if ke <= ks:
                continue
            update(np.arange(ks, ke), k64[ks:ke], v64[ks:ke])
        cols = np.asarray(col_indices[int(col_offsets[r]): int(col_offsets[r + 1])], dtype=np.int64)
        for c0 in range(0, cols.size, b):
            chip = cols[c0: c0 + b]
            # _core.pyx:172-179: allowed prefix = leading columns <= query
            keys = np.maximum.accumulate(chip)
            update(keys, k64[chip], v64[chip])
        res = np.divide(acc, l[:, None], out=np.zeros_like(acc), where=l[:, None] > 0)
        out[q0:q1] = res.astype(STORAGE)
    return out


def flatten(per_row):
    """kernels.py:28-35: per-row lists -> (flat int64, offsets int64)."""
    off = np.zeros(len(per_row) + 1, np.int64)
    for r, row in enumerate(per_row):
        off[r + 1] = off[r] + len(row)
    flat = np.fromiter((int(x) for row in per_row for x in row), dtype=np.int64, count=int(off[-1]))
    return flat, off


# --------------------------------------------------------------------------
# the reference's own compiled kernel (oracle/_ref), when built
# --------------------------------------------------------------------------
def load_ref_core():
    """Import oracle/_ref/spf_ref_core (the reference _core.pyx built by
    oracle/Makefile).  Returns None when it was not built."""
    import importlib.machinery
    import importlib.util
    import sysconfig

    path = os.path.join(_HERE, "_ref", "spf_ref_core" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not os.path.exists(path):
        return None
    loader = importlib.machinery.ExtensionFileLoader("spf_ref_core", path)
    spec = importlib.util.spec_from_file_location("spf_ref_core", path, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


@dataclass
class LocalityInputs:
    """SURVEY.md section 8(d) 'G-local' generator (numpy twin of the GPU one)."""

    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
