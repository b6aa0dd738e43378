"""Index parity of the GPU estimators against the reference (golden vectors)
and the oracle port: index sets must be bit-exact (north_star), the fp64
score vectors equal to ~1 ulp."""

import numpy as np
import pytest
import torch

from conftest import bf16_round, gaussian_qkv
from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2407_02490_b200 as P

    return P


def _vs_names(golden):
    return sorted({k.split("__")[0] for k in golden.files if k.startswith("vs_")})


def test_vs_golden_numpy_api(golden, P):
    for name in _vs_names(golden):
        s, d, kv, ks, lq, seed, bf16, b = (int(x) for x in golden[f"{name}__params"])
        q, k, _ = gaussian_qkv(s, d, seed, bool(bf16))
        idx = P.estimate_vertical_slash(q, k, P.VerticalSlash(kv, ks, lq))
        np.testing.assert_array_equal(idx.vertical, golden[f"{name}__vertical"], err_msg=name)
        np.testing.assert_array_equal(idx.slash, golden[f"{name}__slash"], err_msg=name)


def test_vs_golden_scores_and_bf16_path(golden, P):
    for name in _vs_names(golden):
        s, d, kv, ks, lq, seed, bf16, b = (int(x) for x in golden[f"{name}__params"])
        if not bf16:
            continue
        q, k, _ = gaussian_qkv(s, d, seed, True)
        tq = torch.from_numpy(q).cuda().to(torch.bfloat16)[None]
        tk = torch.from_numpy(k).cuda().to(torch.bfloat16)[None]
        cfg = P.VerticalSlash(kv, ks, lq)
        # fp64 path: scores equal to the reference's to ~1 ulp
        vert, sl, vsc, ssc = P.estimate_vertical_slash_gpu(tq, tk, cfg, with_scores=True, mode="exact")
        np.testing.assert_array_equal(vert[0].cpu().numpy(), golden[f"{name}__vertical"], err_msg=name)
        np.testing.assert_array_equal(sl[0].cpu().numpy(), golden[f"{name}__slash"], err_msg=name)
        np.testing.assert_allclose(vsc[0].cpu().numpy(), golden[f"{name}__vscore"], rtol=1e-12, atol=0)
        np.testing.assert_allclose(ssc[0].cpu().numpy(), golden[f"{name}__sscore"], rtol=1e-12, atol=0)
        # production path (tensor cores + certification / exact re-run): same index sets
        vert, sl = P.estimate_vertical_slash_gpu(tq, tk, cfg, mode="fast")
        np.testing.assert_array_equal(vert[0].cpu().numpy(), golden[f"{name}__vertical"], err_msg=name)
        np.testing.assert_array_equal(sl[0].cpu().numpy(), golden[f"{name}__slash"], err_msg=name)


@pytest.mark.parametrize("s,seed,gen", [(8192, 0, "iid"), (8192, 3, "iid"), (32768, 1, "iid"), (5000, 2, "iid"),
                                        (16384, 0, "local"), (131072, 0, "local")])
def test_vs_tensor_core_error_model(P, s, seed, gen):
    """Measured error of the raw tensor-core vectors (mode "uncertified") against the
    fp64 path, next to the rigorous bound eta of estimate_vs_tc.cu: the bound holds with
    room to spare (it is a worst case, the measured error a typical one), and the
    production path ("fast") selects exactly the fp64 sets on all four heads."""
    from benchmarks.workloads import g_iid_qkv, g_local_qkv

    from test_headline_parity_gpu import _eta_bound

    gen_fn = g_iid_qkv if gen == "iid" else g_local_qkv
    q, k, _ = gen_fn(4, 1, s, 128, seed=seed, device="cuda")
    cfg = P.VerticalSlash(1000, 6096, 64)
    from paper_2407_02490_b200.estimator import vs_estimate_async

    _, _, vsr, ssr, _ = vs_estimate_async(q, k, cfg, mode="uncertified", with_scores=True)
    vf, sf, _, _, _ = vs_estimate_async(q, k, cfg, mode="fast")
    ve, se, vse, sse, _ = vs_estimate_async(q, k, cfg, mode="exact", with_scores=True)
    etas = _eta_bound(q, k, 4, 1)
    for h in range(4):
        for fast, exact in ((vsr[h], vse[h]), (ssr[h], sse[h])):
            fast, exact = fast.cpu().numpy(), exact.cpu().numpy()
            big = exact > 1e-30
            rel = np.abs(fast[big] - exact[big]) / exact[big]
            assert rel.max() <= etas[h], (gen, s, h, rel.max(), etas[h])
    assert torch.equal(vf, ve) and torch.equal(sf, se)


def test_vs_gqa_multihead_matches_port(P):
    s, d, hq, hkv = 2048, 128, 4, 2
    rng = np.random.Generator(np.random.PCG64(7))
    q = bf16_round(rng.standard_normal((hq, s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((hkv, s, d)).astype(np.float32))
    cfg = P.VerticalSlash(100, 500, 64)
    heads = torch.tensor([3, 0, 2], dtype=torch.int32, device="cuda")
    vert, sl = P.estimate_vertical_slash_gpu(torch.from_numpy(q).cuda().to(torch.bfloat16),
                                             torch.from_numpy(k).cuda().to(torch.bfloat16), cfg, heads)
    for i, h in enumerate([3, 0, 2]):
        wv, ws = port.estimate_vertical_slash(q[h], k[h // 2], 100, 500, 64)
        np.testing.assert_array_equal(vert[i].cpu().numpy(), wv)
        np.testing.assert_array_equal(sl[i].cpu().numpy(), ws)


@pytest.mark.parametrize("s,d,lq", [(300, 64, 100), (1000, 128, 130), (129, 32, 129), (64, 16, 1)])
def test_vs_last_q_variants(P, s, d, lq):
    q, k, _ = gaussian_qkv(s, d, 100 + s)
    idx = P.estimate_vertical_slash(q, k, P.VerticalSlash(20, 30, lq))
    wv, ws = port.estimate_vertical_slash(q, k, 20, 30, lq)
    np.testing.assert_array_equal(idx.vertical, wv)
    np.testing.assert_array_equal(idx.slash, ws)


def test_vs_rejects_last_q_over_seq_len(P):
    q, k, _ = gaussian_qkv(8, 4, 1)
    with pytest.raises(ValueError):
        P.estimate_vertical_slash(q, k, P.VerticalSlash(2, 2, 16))


def test_vs_clip_and_force_include(P):
    q, k, _ = gaussian_qkv(8, 4, 1)
    idx = P.estimate_vertical_slash(q, k, P.VerticalSlash(100, 100, 8))
    assert idx.vertical.size == 8 and idx.slash.size == 8
    q, k, _ = gaussian_qkv(64, 16, 0)
    idx = P.estimate_vertical_slash(q, k, P.VerticalSlash(4, 4, 16))
    assert 0 in idx.vertical and 0 in idx.slash


def test_bs_golden(golden, P):
    names = sorted({k.split("__")[0] for k in golden.files if k.startswith("bs_")})
    for name in names:
        s, d, kb, b, seed, bf16 = (int(x) for x in golden[f"{name}__params"])
        q, k, _ = gaussian_qkv(s, d, seed, bool(bf16))
        blocks = P.estimate_block_sparse(q, k, P.BlockSparse(kb, b))
        flat = np.array([x * b for row in blocks.rows for x in row], dtype=np.int64)
        np.testing.assert_array_equal(flat, golden[f"{name}__tiles"], err_msg=name)


def test_planted_golden(golden, P):
    q, k = golden["planted__q"], golden["planted__k"]
    idx = P.estimate_vertical_slash(q, k, P.VerticalSlash(4, 4, 64))
    np.testing.assert_array_equal(idx.vertical, golden["planted__vertical"])
    np.testing.assert_array_equal(idx.slash, golden["planted__slash"])
    assert 137 in idx.vertical and 33 in idx.slash
    blocks = P.estimate_block_sparse(q, k, P.BlockSparse(2, 64))
    flat = np.array([x * 64 for row in blocks.rows for x in row], dtype=np.int64)
    np.testing.assert_array_equal(flat, golden["planted__bs_tiles"])


@pytest.mark.parametrize("s,kb,b", [(256, 100, 64), (130, 2, 64), (777, 7, 16)])
def test_bs_vs_port(P, s, kb, b):
    q, k, _ = gaussian_qkv(s, 32, s + kb)
    blocks = P.estimate_block_sparse(q, k, P.BlockSparse(kb, b))
    assert blocks.rows == port.estimate_block_sparse(q, k, kb, b)


def test_argtopk_ties(P):
    np.testing.assert_array_equal(P.argtopk([1.0, 5.0, 3.0], 2), [1, 2])
    np.testing.assert_array_equal(P.argtopk([2.0, 2.0, 2.0], 2), [0, 1])
    assert P.argtopk([3.0, 1.0], 10).tolist() == [0, 1]
    with pytest.raises(ValueError):
        P.argtopk([1.0], 0)


@pytest.mark.parametrize("hq,hkv,ids", [(14, 2, None), (7, 1, [6, 0, 3, 5]), (12, 4, [11, 2, 7]), (8, 8, [1, 6])])
def test_vs_fast_gqa_grouping_matches_exact(P, hq, hkv, ids):
    """Groups of up to 4 q-heads per kv head (7 q-heads per kv head -> 2 groups), head
    subsets in arbitrary order: the production path equals the fp64 path head by head."""
    from benchmarks.workloads import g_local_qkv

    from paper_2407_02490_b200.estimator import vs_estimate_async

    s = 4096 + 64 * 3 + 17
    q, k, _ = g_local_qkv(hq, hkv, s, 128, seed=hq + hkv, device="cuda")
    cfg = P.VerticalSlash(300, 900, 64)
    head_ids = None if ids is None else torch.tensor(ids, dtype=torch.int32, device="cuda")
    vf, sf, _, _, _ = vs_estimate_async(q, k, cfg, head_ids, mode="fast")
    ve, se, _, _, _ = vs_estimate_async(q, k, cfg, head_ids, mode="exact")
    assert torch.equal(vf, ve) and torch.equal(sf, se)
    # and against the CPU oracle for two of the heads
    qn, kn = q.float().cpu().numpy(), k.float().cpu().numpy()
    for i, h in list(enumerate(ids if ids is not None else range(hq)))[:2]:
        wv, ws = port.estimate_vertical_slash(qn[h], kn[h // (hq // hkv)], 300, 900, 64)
        np.testing.assert_array_equal(vf[i].cpu().numpy(), wv)
        np.testing.assert_array_equal(sf[i].cpu().numpy(), ws)


def test_vs_ties_resolved_by_lowest_index(P):
    """Repeated identical keys make exactly tied vertical scores: the reference's
    stable order (ties to the lower index, estimator.py:66) must hold on both paths."""
    s, d = 2048, 64
    rng = np.random.Generator(np.random.PCG64(11))
    q = bf16_round(rng.standard_normal((s, d)).astype(np.float32))
    k = bf16_round(rng.standard_normal((s, d)).astype(np.float32))
    k[100:1700:4] = k[90]  # 400 identical columns (tied vertical sums)
    cfg = P.VerticalSlash(150, 200, 64)
    wv, ws = port.estimate_vertical_slash(q, k, 150, 200, 64)
    tq = torch.from_numpy(q).cuda().to(torch.bfloat16)[None]
    tk = torch.from_numpy(k).cuda().to(torch.bfloat16)[None]
    for mode in ("fast", "exact"):
        vert, sl = P.estimate_vertical_slash_gpu(tq, tk, cfg, mode=mode)
        np.testing.assert_array_equal(vert[0].cpu().numpy(), wv, err_msg=mode)
        np.testing.assert_array_equal(sl[0].cpu().numpy(), ws, err_msg=mode)


@pytest.mark.parametrize("s", [65536 + 100, 200000])
def test_vs_fast_dead_tile_skipping_matches_exact(P, s):
    """Long G-local sequences: most 128-key tiles lie > 2^127 below the row max and are
    skipped by both tensor-core passes (estimate_vs_tc.cu, kDeadExp); the index sets
    still equal the fp64 path's and the skipped tiles' vertical scores are exactly 0."""
    from benchmarks.workloads import g_local_qkv

    from paper_2407_02490_b200.estimator import vs_estimate_async

    q, k, _ = g_local_qkv(8, 2, s, 128, seed=7, device="cuda")
    cfg = P.VerticalSlash(1000, 6096, 64)
    ids = torch.tensor([5, 0, 2, 7, 3], dtype=torch.int32, device="cuda")
    vf, sf, vsf, ssf, _ = vs_estimate_async(q, k, cfg, ids, mode="fast", with_scores=True)
    ve, se, vse, sse, _ = vs_estimate_async(q, k, cfg, ids, mode="exact", with_scores=True)
    assert torch.equal(vf, ve) and torch.equal(sf, se)
    # far-from-diagonal keys: probabilities below fp32's range in both paths
    far = s // 4
    assert float(vsf[:, :far].abs().max()) == 0.0 and float(vse[:, :far].abs().max()) == 0.0


@pytest.mark.parametrize("n,k,kind", [(1, 1, "rand"), (10, 20, "rand"), (1000, 100, "ties"), (4097, 4097, "ties"),
                                      (100000, 6096, "rand"), (1 << 20, 16384, "ties"), (5000, 300, "zeros")])
def test_argtopk_matches_reference_rule(P, n, k, kind):
    """spf_argtopk == np.argsort(-x, kind="stable")[:k] (estimator.py:59-67): descending
    values, ties to the lower index, -0.0 equal to +0.0, k clipped to n."""
    rng = np.random.Generator(np.random.PCG64(n + k))
    if kind == "rand":
        x = rng.standard_normal(n)
    elif kind == "ties":
        x = rng.integers(0, 50, n).astype(np.float64) / 7.0
    else:
        x = np.where(rng.random(n) < 0.5, 0.0, -0.0) + np.where(rng.random(n) < 0.01, 1.0, 0.0)
    got = P.argtopk(x, k)
    np.testing.assert_array_equal(got, port.argtopk(x, k))
