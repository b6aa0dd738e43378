"""Parity at BASELINE.json's full sequence lengths (C3: 1M-token Vertical-Slash,
C5: 512K A-shape) through size-independent checks: the certified
tensor-core estimation equals the fp64 path, the GPU layout equals the C / NumPy
oracle layout bit for bit, and sampled row blocks of the attention output match
the oracle kernel (fp64) within the bf16 tolerance."""

import math

import numpy as np
import pytest
import torch

from oracle import port

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


@pytest.fixture(scope="module")
def P():
    import paper_2407_02490_b200 as P

    return P


def _sampled_rows(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return sorted(set([0, 1, 2, n // 3, n // 2, n - 2, n - 1] + rng.choice(n, 9, replace=False).tolist()))


def _check_rows(out, q, k, v, lay, s_len, b, rows):
    qn, kn, vn = (x[0].float().cpu().numpy() for x in (q, k, v))
    t = lay.tiles.cpu().numpy().astype(np.int64)
    to = lay.tile_offsets.cpu().numpy()
    c = lay.cols.cpu().numpy().astype(np.int64)
    co = lay.col_offsets.cpu().numpy()
    want = port.sparse_flash_rows(qn, kn, vn, 1 / math.sqrt(qn.shape[1]), b, t, to, c, co, rows=rows)
    got = out[0].float().cpu().numpy()
    for r in rows:
        sl = slice(r * b, min((r + 1) * b, s_len))
        err = float(np.abs(got[sl] - want[sl]).max())
        assert err < BF16_TOL, (r, err)


def test_c3_vs_1m_pipeline(P):
    from benchmarks.workloads import g_local_qkv

    from paper_2407_02490_b200 import kernels
    from paper_2407_02490_b200.estimator import vs_estimate_async

    s_len, d, b = 1 << 20, 128, 64
    q, k, v = g_local_qkv(1, 1, s_len, d, seed=11, device="cuda")
    cfg = P.VerticalSlash(1000, 6096, 64)
    vf, sf, _, _, _ = vs_estimate_async(q, k, cfg, mode="fast")
    ve, se, _, _, _ = vs_estimate_async(q, k, cfg, mode="exact")
    assert torch.equal(vf, ve) and torch.equal(sf, se)
    lay = P.build_layer_layout(q, k, [cfg], b)
    wt, wto, wc, wco = port.build_vs_csr(vf[0].cpu().numpy(), sf[0].cpu().numpy(), s_len, b)
    np.testing.assert_array_equal(lay.tile_offsets.cpu().numpy(), wto)
    np.testing.assert_array_equal(lay.tiles.cpu().numpy().astype(np.int64), wt)
    np.testing.assert_array_equal(lay.col_offsets.cpu().numpy(), wco)
    np.testing.assert_array_equal(lay.cols.cpu().numpy().astype(np.int64), wc)
    out = kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), b, lay.tiles, lay.tile_offsets, lay.cols,
                                             lay.col_offsets)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out).all())
    _check_rows(out, q, k, v, lay, s_len, b, _sampled_rows((s_len + b - 1) // b, 3))


def test_c5_ashape_512k(P):
    from benchmarks.workloads import g_iid_qkv

    from paper_2407_02490_b200 import kernels

    s_len, d, b = 1 << 19, 128, 64
    q, k, v = g_iid_qkv(1, 1, s_len, d, seed=5, device="cuda")
    cfg = P.AShape(128, 4096)
    lay = P.build_layer_layout(q, k, [cfg], b)
    want = port.a_shape_layout(s_len, 128, 4096, b)
    wt, wto = port.flatten(want)
    np.testing.assert_array_equal(lay.tile_offsets.cpu().numpy(), wto)
    np.testing.assert_array_equal(lay.tiles.cpu().numpy().astype(np.int64), wt)
    assert lay.n_cols == 0
    out = kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), b, lay.tiles, lay.tile_offsets, lay.cols,
                                             lay.col_offsets)
    _check_rows(out, q, k, v, lay, s_len, b, _sampled_rows((s_len + b - 1) // b, 4))


def test_c4_bs_256k(P):
    from benchmarks.workloads import g_iid_qkv

    from paper_2407_02490_b200 import kernels

    s_len, d, b = 1 << 18, 128, 64
    q, k, v = g_iid_qkv(1, 1, s_len, d, seed=9, device="cuda")
    cfg = P.BlockSparse(100)
    lay = P.build_layer_layout(q, k, [cfg], b)
    rows = port.estimate_block_sparse(q[0].float().cpu().numpy(), k[0].float().cpu().numpy(), 100, b)
    wt, wto = port.flatten(port.block_rows_to_tiles(rows, b))
    np.testing.assert_array_equal(lay.tile_offsets.cpu().numpy(), wto)
    np.testing.assert_array_equal(lay.tiles.cpu().numpy().astype(np.int64), wt)
    for pair in (None, torch.ones(1, dtype=torch.uint8, device="cuda")):  # union and paired-box kernels
        out = kernels.sparse_flash_attention_gpu(q, k, v, 1 / math.sqrt(d), b, lay.tiles, lay.tile_offsets, lay.cols,
                                                 lay.col_offsets, pair_heads=pair)
        _check_rows(out, q, k, v, lay, s_len, b, _sampled_rows((s_len + b - 1) // b, 6))
