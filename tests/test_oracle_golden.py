"""CPU: pin the oracle port to the reference's golden vectors (and, when built,
to the reference's own compiled kernel oracle/_ref/spf_ref_core)."""

import math

import numpy as np
import pytest

from conftest import gaussian_qkv
from oracle import port


def _names(golden, prefix):
    return sorted({k.split("__")[0] for k in golden.files if k.startswith(prefix)})


def _rows(blocks, s, b):
    return np.concatenate([np.arange(r * b, min(r * b + b, s)) for r in blocks])


def test_input_generator_pinned(golden):
    import hashlib

    for name in _names(golden, "vs_") + _names(golden, "bs_") + _names(golden, "as_"):
        prm = golden[f"{name}__params"]
        s, d = int(prm[0]), int(prm[1])
        seed = int(prm[5]) if name.startswith("vs_") else int(prm[4] if name.startswith("bs_") else prm[5])
        bf16 = bool(prm[6] if name.startswith("vs_") else prm[5] if name.startswith("bs_") else prm[6])
        q, k, v = gaussian_qkv(s, d, seed, bf16)
        h = hashlib.sha256()
        for a in (q, k, v):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(golden[f"{name}__digest"]), name


def test_vs_estimator_and_merge(golden):
    for name in _names(golden, "vs_"):
        s, d, kv, ks, lq, seed, bf16, b = (int(x) for x in golden[f"{name}__params"])
        if s > 4096:
            continue  # keep the CPU suite fast; the 8K cases are covered on GPU
        q, k, _ = gaussian_qkv(s, d, seed, bool(bf16))
        vv, ss = port.estimate_vertical_slash(q, k, kv, ks, lq)
        np.testing.assert_array_equal(vv, golden[f"{name}__vertical"])
        np.testing.assert_array_equal(ss, golden[f"{name}__slash"])
        tiles, cols, ops = port.build_vs_layout_with_stats(vv, ss, s, b)
        t, to = port.flatten(tiles)
        c, co = port.flatten(cols)
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"])
        np.testing.assert_array_equal(c, golden[f"{name}__cols"])
        np.testing.assert_array_equal(np.asarray(ops), golden[f"{name}__ops"])
        assert port.layout_area(s, b, tiles, cols) == int(golden[f"{name}__area"])


def test_c_merge_equals_python_merge(golden, rng):
    for name in _names(golden, "vs_"):
        s, d, kv, ks, lq, seed, bf16, b = (int(x) for x in golden[f"{name}__params"])
        t, to, c, co = port.build_vs_csr(golden[f"{name}__vertical"], golden[f"{name}__slash"], s, b)
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"])
        np.testing.assert_array_equal(to, golden[f"{name}__tile_off"])
        np.testing.assert_array_equal(c, golden[f"{name}__cols"])
        np.testing.assert_array_equal(co, golden[f"{name}__col_off"])
    for _ in range(200):
        s = int(rng.integers(4, 200))
        b = int(rng.choice([2, 4, 8, 64]))
        vv = np.sort(rng.choice(s, size=int(rng.integers(1, min(12, s) + 1)), replace=False))
        ss = -np.sort(-rng.choice(s, size=int(rng.integers(1, min(12, s) + 1)), replace=False))
        wt, wc, _ = port.build_vs_layout_with_stats(vv, ss, s, b)
        t, to, c, co = port.build_vs_csr(vv, ss, s, b)
        assert [t[to[r]:to[r + 1]].tolist() for r in range(to.size - 1)] == wt
        assert [c[co[r]:co[r + 1]].tolist() for r in range(co.size - 1)] == wc


def test_bs_and_ashape(golden):
    for name in _names(golden, "bs_"):
        s, d, kb, b, seed, bf16 = (int(x) for x in golden[f"{name}__params"])
        if s > 4096:
            continue
        q, k, _ = gaussian_qkv(s, d, seed, bool(bf16))
        rows = port.estimate_block_sparse(q, k, kb, b)
        t, _ = port.flatten(port.block_rows_to_tiles(rows, b))
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"])
    for name in _names(golden, "as_"):
        s, d, g, w, b, seed, bf16 = (int(x) for x in golden[f"{name}__params"])
        t, to = port.flatten(port.a_shape_layout(s, g, w, b))
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"])
        np.testing.assert_array_equal(to, golden[f"{name}__tile_off"])


def test_kernel_port_matches_reference_outputs(golden):
    for prefix in ("vs_", "bs_", "as_"):
        for name in _names(golden, prefix):
            prm = [int(x) for x in golden[f"{name}__params"]]
            if prefix == "vs_":
                s, d, seed, bf16, b = prm[0], prm[1], prm[5], prm[6], prm[7]
                cs, co = golden[f"{name}__cols"], golden[f"{name}__col_off"]
            elif prefix == "bs_":
                s, d, b, seed, bf16 = prm[0], prm[1], prm[3], prm[4], prm[5]
            else:
                s, d, b, seed, bf16 = prm[0], prm[1], prm[4], prm[5], prm[6]
            ts, to = golden[f"{name}__tiles"], golden[f"{name}__tile_off"]
            if prefix != "vs_":
                cs, co = np.zeros(0, np.int64), np.zeros(to.size, np.int64)
            q, k, v = gaussian_qkv(s, d, seed, bool(bf16))
            blocks = golden[f"{name}__out_blocks"]
            got = port.sparse_flash_rows(q, k, v, 1 / math.sqrt(d), b, ts, to, cs, co, rows=blocks)
            rows = _rows(blocks, s, b)
            np.testing.assert_allclose(got[rows], golden[f"{name}__out"], rtol=0, atol=2e-6, err_msg=name)


def test_ref_core_agrees_with_port():
    ref = port.load_ref_core()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    q, k, v = gaussian_qkv(130, 16, 7)
    tiles, cols, _ = port.build_vs_layout_with_stats([0, 7, 64, 100], [65, 9, 0], 130, 64)
    ts, to = port.flatten(tiles)
    cs, co = port.flatten(cols)
    a = ref.sparse_flash_rows(q, k, v, 0.25, 64, ts, to, cs, co)
    b = port.sparse_flash_rows(q, k, v, 0.25, 64, ts, to, cs, co)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-6)


def test_masked_oracle_equals_streaming_port():
    # criterion 2 flavour: dense layout through the streaming port == Eq. (1)
    q, k, v = gaussian_qkv(127, 16, 127)
    tiles = port.a_shape_layout(127, 127, 127, 16)
    ts, to = port.flatten(tiles)
    n = to.size - 1
    got = port.sparse_flash_rows(q, k, v, 0.25, 16, ts, to, np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
    want = port.masked_attention(q, k, v, 0.25, np.tril(np.ones((127, 127), bool)))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-5)
