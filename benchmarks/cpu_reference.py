"""The reference's CPU path, timed on the host cores (bench.py's cpu_baseline
and the ``--impl reference`` arm).  TEST/BENCH INFRASTRUCTURE: this is the
one place bench.py executes oracle/.

One work item = one (layer, head) of the benchmark config, run exactly as the
reference's ``run_head_timed`` does (sparse_attn.py:67-94):
  * with the reference package installed in baseline/_ref (pip --target, see
    DESIGN.md section 5): the reference's OWN code end to end -- its
    estimate_vertical_slash / estimate_block_sparse, build_vs_layout / a_shape_layout,
    and kernels.sparse_flash_attention on its compiled Cython kernel;
  * otherwise: oracle/port.py's restatement (estimator.py:82-143, Alg. 4 of
    vs_index.py:28-95, patterns.py:109-128) and the reference's compiled Cython
    kernel from oracle/_ref (else the port's kernel);
  * the kernel runs on a row sample (other rows' lists empty) and is extrapolated by
    tiles + column chips (kernel time is linear in them).
Items run in a process pool (one process per core; the Cython kernel holds the
GIL, so threads would not help) with OPENBLAS_NUM_THREADS=1; the step's
latency = sum(item seconds) / cores.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np


def g_local_np(s: int, d: int, seed: int):
    """numpy twin of benchmarks.workloads.g_local_qkv for one head (fp32, bf16-exact)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    q = (rng.standard_normal((s, d)) * 0.5).astype(np.float32)
    k = (rng.standard_normal((s, d)) * 0.5).astype(np.float32)
    v = rng.standard_normal((s, d)).astype(np.float32)
    j = np.arange(s)
    k[:, 0] = j % 256
    k[:, 1] = (j >> 8) % 256
    k[:, 2] = j >> 16
    a = 2.0 ** -3
    q[:, 0], q[:, 1], q[:, 2] = a, a * 256, a * 65536
    k[:4, 3] = 64.0
    q[:, 3] = 1.0

    def bf16(x):
        u = x.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32)

    return bf16(q), bf16(k), bf16(v)


def _timed(fn) -> float:
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def _ref_package():
    """The reference package from baseline/_ref (None when it is not installed)."""
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(repo, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "sparseprefill")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import sparseprefill  # noqa: F401
        from sparseprefill import estimator, kernels, patterns, sparse_attn, vs_index
    except ImportError:
        return None
    if kernels.BACKEND != "cython":
        return None
    return estimator, kernels, patterns, sparse_attn, vs_index


def _run_item_reference(pkg, kind, params, s, d, b, q, k, v, n_sample_rows):
    estimator, kernels, patterns, sparse_attn, vs_index = pkg
    t0 = time.perf_counter()
    if kind == "vertical_slash":
        idx = estimator.estimate_vertical_slash(q, k, patterns.VerticalSlash(*params))
        t1 = time.perf_counter()
        layout = vs_index.build_vs_layout(idx, s, b)
    elif kind == "a_shape":
        t1 = time.perf_counter()
        layout = patterns.a_shape_layout(s, patterns.AShape(*params), b)
    else:
        blocks = estimator.estimate_block_sparse(q, k, patterns.BlockSparse(params[0], b))
        t1 = time.perf_counter()
        layout = sparse_attn.block_indices_to_layout(blocks, s, b)
    t2 = time.perf_counter()
    tiles, cols = layout.block_starts, layout.column_indices
    n = len(tiles)
    units = np.array([len(tiles[r]) + (len(cols[r]) + b - 1) // b for r in range(n)], dtype=np.int64)
    sample = np.unique(np.linspace(0, n - 1, min(n_sample_rows, n)).round().astype(np.int64))
    chosen = set(sample.tolist())
    st = [list(tiles[r]) if r in chosen else [] for r in range(n)]
    sc = [list(cols[r]) if r in chosen else [] for r in range(n)]
    scale = 1.0 / math.sqrt(d)
    empty = [[] for _ in range(n)]
    # the first call in a process pays one-time allocation / first-touch costs: warm up, then
    # time the fixed per-call cost (every row empty) and the sampled rows (best of two each)
    kernels.sparse_flash_attention(q, k, v, scale, b, empty, empty)
    fixed = min(_timed(lambda: kernels.sparse_flash_attention(q, k, v, scale, b, empty, empty)) for _ in range(2))
    sampled = min(_timed(lambda: kernels.sparse_flash_attention(q, k, v, scale, b, st, sc)) for _ in range(2))
    t4, t5 = 0.0, sampled
    sampled_units = int(units[sample].sum())
    total_units = int(units.sum())
    kernel_s = fixed + max(0.0, (t5 - t4) - fixed) * total_units / max(1, sampled_units)
    return {"kind": kind, "t_est": t1 - t0, "t_index": t2 - t1, "t_kernel": kernel_s,
            "t_item": (t1 - t0) + (t2 - t1) + kernel_s, "units": total_units, "sampled_units": sampled_units,
            "ref_kernel": True, "impl": "reference package (baseline/_ref): estimator, vs_index, Cython kernel"}


def _run_item(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    kind, params, s, d, b, seed, n_sample_rows = args
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if repo not in sys.path:
        sys.path.insert(0, repo)
    from oracle import port

    q, k, v = g_local_np(s, d, seed)
    pkg = _ref_package()
    if pkg is not None:
        return _run_item_reference(pkg, kind, params, s, d, b, q, k, v, n_sample_rows)
    ref = port.load_ref_core()
    t0 = time.perf_counter()
    if kind == "vertical_slash":
        k_v, k_s, last_q = params
        vv, ss = port.estimate_vertical_slash(q, k, k_v, k_s, last_q)
        t1 = time.perf_counter()
        tiles, cols, _ = port.build_vs_layout_with_stats(vv, ss, s, b)
    elif kind == "a_shape":
        t1 = time.perf_counter()
        tiles = port.a_shape_layout(s, params[0], params[1], b)
        cols = [[] for _ in tiles]
    else:
        rows = port.estimate_block_sparse(q, k, params[0], b)
        t1 = time.perf_counter()
        tiles = port.block_rows_to_tiles(rows, b)
        cols = [[] for _ in tiles]
    t2 = time.perf_counter()
    n = len(tiles)
    units = np.array([len(tiles[r]) + (len(cols[r]) + b - 1) // b for r in range(n)], dtype=np.int64)
    sample = np.unique(np.linspace(0, n - 1, min(n_sample_rows, n)).round().astype(np.int64))
    chosen = set(sample.tolist())
    st = [tiles[r] if r in chosen else [] for r in range(n)]
    sc = [cols[r] if r in chosen else [] for r in range(n)]
    ts, to = port.flatten(st)
    cs, co = port.flatten(sc)
    scale = 1.0 / math.sqrt(d)
    # fixed per-call cost (fp64 copies of q/k/v, output allocation): one call
    # with every row empty; only the per-row work is extrapolated.
    e_t, e_to = port.flatten([[] for _ in range(n)])
    if ref is not None:
        ref.sparse_flash_rows(q, k, v, scale, b, e_t, e_to, e_t, e_to)  # warm-up (first-touch costs)
        fixed = min(_timed(lambda: ref.sparse_flash_rows(q, k, v, scale, b, e_t, e_to, e_t, e_to))
                    for _ in range(2))
        sampled = min(_timed(lambda: ref.sparse_flash_rows(q, k, v, scale, b, ts, to, cs, co)) for _ in range(2))
    else:
        fixed = 0.0
        sampled = _timed(lambda: port.sparse_flash_rows(q, k, v, scale, b, ts, to, cs, co, rows=sample))
    t4, t5 = 0.0, sampled
    sampled_units = int(units[sample].sum())
    total_units = int(units.sum())
    kernel_s = fixed + max(0.0, (t5 - t4) - fixed) * total_units / max(1, sampled_units)
    return {"kind": kind, "t_est": t1 - t0, "t_index": t2 - t1, "t_kernel": kernel_s,
            "t_item": (t1 - t0) + (t2 - t1) + kernel_s, "units": total_units, "sampled_units": sampled_units,
            "ref_kernel": ref is not None}


def pattern_of(cfg):
    name = type(cfg).__name__
    if name == "VerticalSlash":
        return "vertical_slash", (cfg.k_v, cfg.k_s, cfg.last_q)
    if name == "AShape":
        return "a_shape", (cfg.global_tokens, cfg.local_window)
    return "block_sparse", (cfg.k_b,)


def run_sample(layer_cfgs, s: int, d: int, b: int, cores: int, items_per_pattern: int, n_sample_rows: int,
               step_seed: int = 0):
    """One bounded sample: items_per_pattern (layer, head) items per pattern,
    run on `cores` processes.  Returns (extrapolated step seconds, details)."""
    import multiprocessing as mp

    by_pattern: dict = {}
    for layer, row in enumerate(layer_cfgs):
        for h, cfg in enumerate(row):
            kind, params = pattern_of(cfg)
            by_pattern.setdefault((kind, params), []).append((layer, h))
    rng = np.random.Generator(np.random.PCG64(1234 + step_seed))
    jobs = []
    for (kind, params), heads in by_pattern.items():
        pick = rng.choice(len(heads), size=min(items_per_pattern, len(heads)), replace=False)
        for i in pick:
            layer, h = heads[int(i)]
            jobs.append((kind, params, s, d, b, 1000 * layer + h, n_sample_rows))
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(processes=min(cores, len(jobs))) as pool:
        res = pool.map(_run_item, jobs)
    wall = time.perf_counter() - t0
    total = 0.0
    per = {}
    for (kind, params), heads in by_pattern.items():
        rs = [r for r, j in zip(res, jobs) if (j[0], j[1]) == (kind, params)]
        mean_item = float(np.mean([r["t_item"] for r in rs]))
        per[f"{kind}{list(params)}"] = {"heads": len(heads), "mean_item_s": mean_item,
                                        "mean_est_s": float(np.mean([r["t_est"] for r in rs])),
                                        "mean_index_s": float(np.mean([r["t_index"] for r in rs])),
                                        "mean_kernel_s": float(np.mean([r["t_kernel"] for r in rs]))}
        total += mean_item * len(heads)
    step_s = total / cores
    return step_s, {"items": len(jobs), "wall_s": wall, "patterns": per,
                    "ref_kernel": all(r["ref_kernel"] for r in res),
                    "impl": res[0].get("impl", "oracle port (estimation, merge) + oracle/_ref Cython kernel")}
