"""End-to-end parity of the production layer pipeline (mixed per-head
patterns, GQA, bf16) and of the drop-in executors against the oracle."""

import math

import numpy as np
import pytest
import torch

from conftest import bf16_round, gaussian_qkv
from oracle import port

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
F32_TOL = 1e-3  # relative to the output's own scale (max |want|)


def _rel(got, want):
    scale = float(np.max(np.abs(want)))
    err = float(np.max(np.abs(np.asarray(got, np.float64) - np.asarray(want, np.float64))))
    return err / scale if scale > 0 else err


@pytest.fixture(scope="module")
def P():
    import paper_2407_02490_b200 as P

    return P


def _oracle_head(q, k, v, cfg, b, P):
    s = q.shape[0]
    if isinstance(cfg, P.VerticalSlash):
        vv, ss = port.estimate_vertical_slash(q, k, cfg.k_v, cfg.k_s, cfg.last_q)
        tiles, cols, _ = port.build_vs_layout_with_stats(vv, ss, s, b)
    elif isinstance(cfg, P.AShape):
        tiles = port.a_shape_layout(s, cfg.global_tokens, cfg.local_window, b)
        cols = [[] for _ in tiles]
    else:
        rows = port.estimate_block_sparse(q, k, cfg.k_b, b)
        tiles = port.block_rows_to_tiles(rows, b)
        cols = [[] for _ in tiles]
    return tiles, cols


@pytest.mark.parametrize("s", [1000, 4096])
def test_mixed_layer_matches_oracle(P, s):
    d, hq, hkv, b = 128, 8, 2, 64
    rng = np.random.Generator(np.random.PCG64(s))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    v = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    cfgs = [P.VerticalSlash(100, 300), P.VerticalSlash(100, 300), P.AShape(128, 512), P.BlockSparse(8),
            P.VerticalSlash(30, 60, 32), P.AShape(64, 1024), P.BlockSparse(8), P.VerticalSlash(100, 300)]
    dev = torch.device("cuda")
    out, lay = P.sparse_prefill_attention(torch.from_numpy(q).to(dev, torch.bfloat16),
                                          torch.from_numpy(k).to(dev, torch.bfloat16),
                                          torch.from_numpy(v).to(dev, torch.bfloat16), cfgs, b,
                                          return_layout=True)
    out = out.float().cpu().numpy()
    n = (s + b - 1) // b
    tiles = lay.tiles.cpu().numpy().astype(np.int64)
    cols = lay.cols.cpu().numpy().astype(np.int64)
    toff = lay.tile_offsets.cpu().numpy()
    coff = lay.col_offsets.cpu().numpy()
    for h, cfg in enumerate(cfgs):
        kvh = h // (hq // hkv)
        wt, wc = _oracle_head(q[h], k[kvh], v[kvh], cfg, b, P)
        gt = [tiles[toff[h * n + r]: toff[h * n + r + 1]].tolist() for r in range(n)]
        gc = [cols[coff[h * n + r]: coff[h * n + r + 1]].tolist() for r in range(n)]
        assert gt == wt, (h, cfg)
        assert gc == wc, (h, cfg)
        ts, to = port.flatten(wt)
        cs, co = port.flatten(wc)
        want = port.sparse_flash_rows(q[h], k[kvh], v[kvh], 1 / math.sqrt(d), b, ts, to, cs, co)
        err = float(np.max(np.abs(out[h] - want)))
        assert err <= BF16_TOL, (h, cfg, err)


@pytest.mark.parametrize("cfg_name", ["ashape", "vs", "bs"])
def test_run_head_matches_masked_oracle(P, cfg_name):
    # test_sparse_attn.py:109-118 of the reference
    cfg = {"ashape": P.AShape(8, 16), "vs": P.VerticalSlash(4, 4, 16), "bs": P.BlockSparse(3, 16)}[cfg_name]
    q, k, v = gaussian_qkv(95, 16, 8)
    inp = P.AttentionInputs(q, k, v)
    out, layout = P.run_head(inp, cfg, 16)
    want = port.masked_attention(q, k, v, inp.scale, P.layout_to_mask(layout))
    assert _rel(out, want) <= F32_TOL
    out2, lay2, t_est, t_sparse = P.run_head_timed(inp, cfg, 16)
    np.testing.assert_array_equal(out, out2)
    assert t_est >= 0 and t_sparse >= 0


def test_unknown_config_rejected(P):
    q, k, v = gaussian_qkv(8, 4, 0)
    with pytest.raises(TypeError):
        P.run_head(P.AttentionInputs(q, k, v), object(), 4)


def test_executors_acceptance_sweep(P):
    # criterion 1 of test_acceptance.py:59-94 (reduced): random VS/A-shape/BS
    rng = np.random.Generator(np.random.PCG64(2024))
    worst = 0.0
    for s in (17, 64, 257):
        for b in (4, 16, 64):
            q, k, v = gaussian_qkv(s, 32, 1000 * s + b)
            inp = P.AttentionInputs(q, k, v)
            vertical = np.sort(rng.choice(s, size=min(int(rng.integers(1, 9)), s), replace=False))
            slash = -np.sort(-rng.choice(s, size=min(int(rng.integers(1, 9)), s), replace=False))
            layout = P.build_vs_layout(P.VSIndices(vertical=vertical, slash=slash), s, b)
            got = P.vertical_slash_attention(inp, layout)
            want = port.masked_attention(q, k, v, inp.scale, P.layout_to_mask(layout))
            worst = max(worst, _rel(got, want))
            out, layout = P.run_head(inp, P.AShape(int(rng.integers(1, s + 1)), int(rng.integers(1, s + 1))), b)
            want = port.masked_attention(q, k, v, inp.scale, P.layout_to_mask(layout))
            worst = max(worst, _rel(out, want))
            blocks = P.estimate_block_sparse(q, k, P.BlockSparse(int(rng.integers(1, 6)), b))
            got = P.block_sparse_attention(inp, blocks, b)
            lay = P.block_indices_to_layout(blocks, s, b)
            want = port.masked_attention(q, k, v, inp.scale, P.layout_to_mask(lay))
            worst = max(worst, _rel(got, want))
    assert worst <= F32_TOL, worst


def test_layer_outputs_deterministic_across_runs(P):
    """Repeated launches give bit-identical outputs (guards against pipeline races
    between the softmax warps and the MMA warp, e.g. barrier phases completing early)."""
    s, d, hq, hkv, b = 4096, 128, 8, 2, 64
    rng = np.random.Generator(np.random.PCG64(s))
    q, k, v = (torch.from_numpy(bf16_round(rng.standard_normal((h, s, d)).astype(np.float32))).cuda()
               .to(torch.bfloat16) for h in (hq, hkv, hkv))
    cfgs = [P.VerticalSlash(100, 300), P.VerticalSlash(100, 300), P.AShape(128, 512), P.BlockSparse(8),
            P.VerticalSlash(30, 60, 32), P.AShape(64, 1024), P.BlockSparse(8), P.VerticalSlash(100, 300)]
    ref = P.sparse_prefill_attention(q, k, v, cfgs, b).clone()
    assert not torch.isnan(ref.float()).any()
    for it in range(30):
        out = torch.full_like(ref, float("nan"))
        P.sparse_prefill_attention(q, k, v, cfgs, b, out=out)
        assert torch.equal(out, ref), it
