"""Parity of the sm_100a sparse FlashAttention kernel (libspf) against the
reference kernel contract (_core.pyx:72-192) restated in oracle/port.py and
against the reference's own outputs stored in tests/golden.

Tolerances (BASELINE.json north_star): fp32 I/O -> max-abs error <= 1e-3 x
max|ref| ("1e-3 relative", relative to the output's own scale, however small);
bf16 I/O -> max-abs <= 2e-2.
"""

import math

import numpy as np
import pytest
import torch

from conftest import bf16_round, gaussian_qkv
from oracle import port

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3
BF16_TOL = 2e-2


def rel_err(got, want):
    scale = float(np.max(np.abs(want)))
    err = float(np.max(np.abs(got.astype(np.float64) - want.astype(np.float64))))
    return err / scale if scale > 0 else err


def max_abs(got, want):
    return float(np.max(np.abs(got.astype(np.float64) - want.astype(np.float64))))


@pytest.fixture(scope="module")
def K():
    from paper_2407_02490_b200 import kernels

    return kernels


def _rows_of(blocks, s, b):
    return np.concatenate([np.arange(r * b, min(r * b + b, s)) for r in blocks])


@pytest.mark.parametrize("prefix", ["vs_", "bs_", "as_"])
def test_golden_layouts_fp32(golden, K, prefix):
    names = sorted({k.split("__")[0] for k in golden.files if k.startswith(prefix)})
    assert names
    for name in names:
        prm = golden[f"{name}__params"]
        if prefix == "vs_":
            s, d, _, _, _, seed, bf16, b = (int(x) for x in prm)
            cols, col_off = golden[f"{name}__cols"], golden[f"{name}__col_off"]
        elif prefix == "bs_":
            s, d, _, b, seed, bf16 = (int(x) for x in prm)
        else:
            s, d, _, _, b, seed, bf16 = (int(x) for x in prm)
        if prefix != "vs_":
            n = (s + b - 1) // b
            cols, col_off = np.zeros(0, np.int64), np.zeros(n + 1, np.int64)
        q, k, v = gaussian_qkv(s, d, seed, bool(bf16))
        got = K.sparse_flash_rows(q, k, v, 1.0 / math.sqrt(d), b, golden[f"{name}__tiles"],
                                  golden[f"{name}__tile_off"], cols, col_off)
        rows = _rows_of(golden[f"{name}__out_blocks"], s, b)
        err = rel_err(got[rows], golden[f"{name}__out"])
        assert err <= F32_TOL, (name, err)


def _random_layout(rng, s, b, n_tiles=3, n_cols=5, unaligned=True):
    n = (s + b - 1) // b
    tiles, cols = [], []
    for r in range(n):
        q_end = min((r + 1) * b, s)
        if unaligned:
            cand = np.sort(rng.choice(np.arange(-b // 2, q_end), size=min(n_tiles, q_end + b // 2), replace=False))
        else:
            cand = np.arange(0, q_end, b)
            cand = np.sort(rng.choice(cand, size=min(n_tiles, cand.size), replace=False))
        tiles.append([int(x) for x in cand])
        cc = np.sort(rng.choice(q_end, size=min(n_cols, q_end), replace=False))
        cols.append([int(x) for x in cc])
    return tiles, cols


@pytest.mark.parametrize("s,d,b", [(17, 16, 4), (64, 16, 16), (257, 64, 64), (300, 128, 64), (1000, 128, 64),
                                   (515, 32, 16), (200, 64, 100), (130, 128, 2), (777, 128, 128)])
def test_random_layouts_fp32(K, s, d, b):
    rng = np.random.Generator(np.random.PCG64(1000 * s + d + b))
    q, k, v = gaussian_qkv(s, d, s + d)
    tiles, cols = _random_layout(rng, s, b)
    ts, to = port.flatten(tiles)
    cs, co = port.flatten(cols)
    want = port.sparse_flash_rows(q, k, v, 1.0 / math.sqrt(d), b, ts, to, cs, co)
    got = K.sparse_flash_attention(q, k, v, 1.0 / math.sqrt(d), b, tiles, cols)
    assert rel_err(got, want) <= F32_TOL


def test_empty_rows_zero_and_full_equals_dense(K):
    # test_sparse_attn.py:58-85 of the reference
    q, k, v = gaussian_qkv(8, 4, 3)
    out = K.sparse_flash_attention(q, k, v, 0.5, 4, [[], [4]], [[], []])
    np.testing.assert_array_equal(out[:4], np.zeros((4, 4)))
    assert np.any(out[4:] != 0)
    q, k, v = gaussian_qkv(50, 8, 4)
    tiles, cols, _ = port.build_vs_layout_with_stats([0], list(range(49, -1, -1)), 50, 8)
    got = K.sparse_flash_attention(q, k, v, 1 / math.sqrt(8), 8, tiles, cols)
    mask = np.tril(np.ones((50, 50), bool))
    want = port.masked_attention(q, k, v, 1 / math.sqrt(8), mask)
    assert rel_err(got, want) <= F32_TOL


def test_row_count_mismatch_rejected(K):
    q, k, v = gaussian_qkv(16, 4, 0)
    with pytest.raises(ValueError):
        K.sparse_flash_attention(q, k, v, 0.5, 4, [[0]], [[]])


@pytest.mark.parametrize("s,hq,hkv,b", [(1000, 4, 2, 64), (4096, 8, 2, 64), (2048, 4, 4, 32)])
def test_multihead_bf16_gqa(K, s, hq, hkv, b):
    d = 128
    rng = np.random.Generator(np.random.PCG64(s + hq))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    v = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    n = (s + b - 1) // b
    tiles_all, cols_all = [], []
    for h in range(hq):
        t, c = _random_layout(rng, s, b, n_tiles=6, n_cols=40)
        tiles_all += t
        cols_all += c
    ts, to = port.flatten(tiles_all)
    cs, co = port.flatten(cols_all)
    dev = torch.device("cuda")
    out = K.sparse_flash_attention_gpu(
        torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
        torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
        torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
        torch.from_numpy(cs.astype(np.int32)).to(dev), torch.from_numpy(co).to(dev)).float().cpu().numpy()
    worst = 0.0
    for h in range(hq):
        kvh = h // (hq // hkv)
        sl = slice(h * n, (h + 1) * n + 1)
        want = port.sparse_flash_rows(q[h], k[kvh], v[kvh], 1 / math.sqrt(d), b, ts, to[sl], cs, co[sl])
        worst = max(worst, max_abs(out[h], want))
    assert worst <= BF16_TOL, worst


@pytest.mark.parametrize("s,kb,d,routing", [(1000, 3, 128, "mask"), (4097, 8, 128, "mask"), (63, 2, 64, "mask"),
                                            (3000, 1, 64, "mask"), (1000, 3, 128, "list"), (4097, 8, 64, "all")])
def test_paired_box_kernel_matches_oracle(K, s, kb, d, routing):
    """The paired-box kernel (Block-Sparse heads, pair_heads) on block-sparse layouts with
    an odd number of row blocks, rows shorter than k_b, k_b = 1 (diagonal only) and a
    sub-block sequence: every row equals the oracle kernel; unlisted heads in the same
    launch still run the union kernel.  Routing given as a uint8 mask, as an unordered
    int32 head list, or as every head (then the union kernel is not launched at all)."""
    hq, hkv, b = 4, 2, 64
    rng = np.random.Generator(np.random.PCG64(s + kb))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    v = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    n = (s + b - 1) // b
    tiles_all = []
    for h in range(hq):
        for r in range(n):
            m = min(kb, r + 1)
            blocks = sorted(set([r] + rng.choice(r + 1, size=m, replace=False).tolist()))[-m:]
            if r not in blocks:
                blocks[-1] = r
            tiles_all.append(sorted(x * b for x in blocks))
    ts, to = port.flatten(tiles_all)
    co = np.zeros(hq * n + 1, np.int64)
    dev = torch.device("cuda")
    pair = {"mask": torch.tensor([1, 0, 1, 1], dtype=torch.uint8, device=dev),
            "list": torch.tensor([3, 0, 2], dtype=torch.int32, device=dev),
            "all": torch.arange(hq, dtype=torch.int32, device=dev)}[routing]
    args = (torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
            torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
            torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
            torch.zeros(1, dtype=torch.int32, device=dev), torch.from_numpy(co).to(dev))
    got = K.sparse_flash_attention_gpu(*args, pair_heads=pair).float().cpu().numpy()
    union = K.sparse_flash_attention_gpu(*args).float().cpu().numpy()
    for h in range(hq):
        kvh = h // (hq // hkv)
        t0, t1 = h * n, (h + 1) * n
        tt, tto = port.flatten(tiles_all[t0:t1])
        want = port.sparse_flash_rows(q[h], k[kvh], v[kvh], 1 / math.sqrt(d), b, tt, tto,
                                      np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
        assert np.abs(got[h] - want).max() < BF16_TOL, (h, np.abs(got[h] - want).max())
        assert np.abs(got[h] - union[h]).max() < BF16_TOL


@pytest.mark.parametrize("s,kb,jump", [(1000, 5, 0.0), (4097, 8, 40.0), (2049, 64, 160.0), (200, 3, 160.0)])
def test_block_sparse_kernel_sink_and_lse(K, s, kb, jump):
    """Block-Sparse heads routed by pair_heads (paired-box kernel; also the parity test the
    transposed-step experiment, benchmarks/experiments/attn_bst.cu, passed) on layouts whose
    every row also takes block 0, with key 0 made a sink `jump` above the rest (20 and 81 in
    log2 units: the running maxima must be raised after the diagonal step, O and the row sums
    rescaled).  Rows with an odd tile count, a partial last block and kb beyond the row
    length.  Output and the per-row log-sum-exp equal the oracle's."""
    hq, hkv, b, d = 4, 2, 64, 128
    rng = np.random.Generator(np.random.PCG64(s + kb))
    q = rng.standard_normal((hq, s, d)).astype(np.float32)
    k = rng.standard_normal((hkv, s, d)).astype(np.float32)
    v = rng.standard_normal((hkv, s, d)).astype(np.float32)
    q[..., 0] = 4.0
    k[:, 0, 0] = jump
    q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    n = (s + b - 1) // b
    tiles_all = []
    for h in range(hq):
        for r in range(n):
            m = min(kb, r + 1)
            blocks = set(rng.choice(r + 1, size=m, replace=False).tolist()) | {0, r}
            tiles_all.append(sorted(x * b for x in blocks))
    ts, to = port.flatten(tiles_all)
    co = np.zeros(hq * n + 1, np.int64)
    dev = torch.device("cuda")
    args = (torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
            torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
            torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
            torch.zeros(1, dtype=torch.int32, device=dev), torch.from_numpy(co).to(dev))
    lse = torch.empty(hq, s, dtype=torch.float32, device=dev)
    got = K.sparse_flash_attention_gpu(*args, lse=lse, pair_heads=torch.arange(hq, dtype=torch.int32, device=dev))
    got = got.float().cpu().numpy()
    lse = lse.cpu().numpy()
    for h in range(hq):
        kvh = h // (hq // hkv)
        tt, tto = port.flatten(tiles_all[h * n:(h + 1) * n])
        want = port.sparse_flash_rows(q[h], k[kvh], v[kvh], 1 / math.sqrt(d), b, tt, tto,
                                      np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
        assert np.abs(got[h] - want).max() < BF16_TOL, (h, np.abs(got[h] - want).max())
        mask = port.layout_to_mask(s, b, tiles_all[h * n:(h + 1) * n], [[] for _ in range(n)])
        sc = (q[h].astype(np.float64) @ k[kvh].astype(np.float64).T) / math.sqrt(d)
        sc = np.where(mask, sc, -np.inf)
        mx = sc.max(axis=1)
        want_lse = mx + np.log(np.exp(sc - mx[:, None]).sum(axis=1))
        assert np.abs(lse[h] - want_lse).max() < 1e-2 * max(1.0, np.abs(want_lse).max()), h


def test_pair_heads_validation(K):
    dev = torch.device("cuda")
    q = torch.zeros(2, 128, 64, dtype=torch.bfloat16, device=dev)
    k = torch.zeros(1, 128, 64, dtype=torch.bfloat16, device=dev)
    to = torch.zeros(5, dtype=torch.int64, device=dev)
    args = (q, k, k, 0.125, 64, torch.zeros(0, dtype=torch.int32, device=dev), to,
            torch.zeros(0, dtype=torch.int32, device=dev), to)
    with pytest.raises(ValueError):
        K.sparse_flash_attention_gpu(*args, pair_heads=torch.ones(3, dtype=torch.uint8, device=dev))
    with pytest.raises(ValueError):
        K.sparse_flash_attention_gpu(*args, pair_heads=torch.zeros(3, dtype=torch.int32, device=dev))
    with pytest.raises(ValueError):
        K.sparse_flash_attention_gpu(*args, pair_heads=torch.zeros(2, dtype=torch.float32, device=dev))
    out = K.sparse_flash_attention_gpu(*args, pair_heads=torch.zeros(2, dtype=torch.uint8, device=dev))
    assert out.abs().max().item() == 0  # no coverage -> zero rows; empty list = union kernel only
    for bad in ([0, 0], [0, 5], [-1]):  # host id lists are validated: distinct, in range
        with pytest.raises(ValueError):
            K.sparse_flash_attention_gpu(*args, pair_heads=torch.tensor(bad, dtype=torch.int32))


def _bs_case(hq, hkv, s, d, kb, seed, b=64):
    rng = np.random.Generator(np.random.PCG64(seed))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    v = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    n = (s + b - 1) // b
    tiles_all = []
    for _h in range(hq):
        for r in range(n):
            m = min(kb, r + 1)
            blocks = sorted(set([r] + rng.choice(r + 1, size=m, replace=False).tolist()))[-m:]
            if r not in blocks:
                blocks[-1] = r
            tiles_all.append(sorted(x * b for x in blocks))
    return q, k, v, n, tiles_all, rng


def test_pair_device_list_duplicates_never_drop_a_head(K):
    """a device list [0, 0] (or with an out-of-range id) must not leave head 1
    unwritten -- the union kernel runs every head the paired-box kernel does not."""
    hq, hkv, s, d, b = 2, 1, 2048 + 77, 64, 64
    q, k, v, n, tiles_all, _ = _bs_case(hq, hkv, s, d, 6, 5)
    ts, to = port.flatten(tiles_all)
    co = np.zeros(hq * n + 1, np.int64)
    dev = torch.device("cuda")
    args = (torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
            torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
            torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
            torch.zeros(1, dtype=torch.int32, device=dev), torch.from_numpy(co).to(dev))
    for ids in ([0, 0], [0, 5], [7, -3]):
        out = torch.full((hq, s, d), float("nan"), dtype=torch.bfloat16, device=dev)
        got = K.sparse_flash_attention_gpu(*args, out=out,
                                           pair_heads=torch.tensor(ids, dtype=torch.int32, device=dev))
        got = got.float().cpu().numpy()
        for h in range(hq):
            tt, tto = port.flatten(tiles_all[h * n:(h + 1) * n])
            want = port.sparse_flash_rows(q[h], k[0], v[0], 1 / math.sqrt(d), b, tt, tto,
                                          np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
            assert np.isfinite(got[h]).all(), (ids, h)
            assert max_abs(got[h], want) < BF16_TOL, (ids, h)


def test_listed_head_with_columns_runs_union_kernel(K):
    """the paired-box kernel has no column-chip path; a listed head (here: every
    head listed, so no unlisted head forces a union launch) that has residual columns must
    still get them -- it is routed to the union kernel."""
    hq, hkv, s, d, b = 2, 1, 4096 + 13, 64, 64
    q, k, v, n, tiles_all, rng = _bs_case(hq, hkv, s, d, 5, 9)
    cols_all = []
    for h in range(hq):
        for r in range(n):
            covered = set()
            for t in tiles_all[h * n + r]:
                covered.update(range(t, min(t + b, s)))
            cand = [j for j in range(0, min(s, r * b + b)) if j not in covered]
            pick = sorted(rng.choice(cand, size=min(len(cand), 70 if h == 1 else 0), replace=False).tolist())
            cols_all.append(pick)
    ts, to = port.flatten(tiles_all)
    cs, co = port.flatten(cols_all)
    dev = torch.device("cuda")
    args = (torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
            torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
            torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
            torch.from_numpy(cs.astype(np.int32)).to(dev), torch.from_numpy(co).to(dev))
    got = K.sparse_flash_attention_gpu(*args, pair_heads=torch.arange(hq, dtype=torch.int32, device=dev))
    got = got.float().cpu().numpy()
    for h in range(hq):
        tt, tto = port.flatten(tiles_all[h * n:(h + 1) * n])
        cc, cco = port.flatten(cols_all[h * n:(h + 1) * n])
        want = port.sparse_flash_rows(q[h], k[0], v[0], 1 / math.sqrt(d), b, tt, tto, cc, cco)
        assert max_abs(got[h], want) < BF16_TOL, (h, max_abs(got[h], want))


def test_mixed_layer_routes_block_sparse_heads_by_overlap(K):
    """A mixed layer (one unlisted head): listed heads whose row blocks share most tiles (a
    locality band) stay on the union kernel, listed heads with scattered tiles run the
    paired-box kernel (pair_stats_kernel decides on device); every head equals the oracle."""
    hq, hkv, b, s, d = 4, 2, 64, 4096 + 64 * 7 + 9, 64
    rng = np.random.Generator(np.random.PCG64(11))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    v = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    n = (s + b - 1) // b
    kb = 24
    tiles_all = []
    for h in range(hq):
        for r in range(n):
            m = min(kb, r + 1)
            if h in (0, 3):  # locality band: consecutive row blocks share all but one block
                blocks = list(range(r - m + 1, r + 1))
            else:  # scattered, diagonal forced
                blocks = sorted(set([r] + rng.choice(r + 1, size=m, replace=False).tolist()))[-m:]
                if r not in blocks:
                    blocks[-1] = r
            tiles_all.append(sorted(x * b for x in blocks))
    ts, to = port.flatten(tiles_all)
    co = np.zeros(hq * n + 1, np.int64)
    dev = torch.device("cuda")
    args = (torch.from_numpy(q).to(dev, torch.bfloat16), torch.from_numpy(k).to(dev, torch.bfloat16),
            torch.from_numpy(v).to(dev, torch.bfloat16), 1 / math.sqrt(d), b,
            torch.from_numpy(ts.astype(np.int32)).to(dev), torch.from_numpy(to).to(dev),
            torch.zeros(1, dtype=torch.int32, device=dev), torch.from_numpy(co).to(dev))
    got = K.sparse_flash_attention_gpu(*args, pair_heads=torch.tensor([0, 1, 3], dtype=torch.int32, device=dev))
    got = got.float().cpu().numpy()
    for h in range(hq):
        kvh = h // (hq // hkv)
        tt, tto = port.flatten(tiles_all[h * n:(h + 1) * n])
        want = port.sparse_flash_rows(q[h], k[kvh], v[kvh], 1 / math.sqrt(d), b, tt, tto,
                                      np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
        assert np.abs(got[h] - want).max() < BF16_TOL, (h, np.abs(got[h] - want).max())
