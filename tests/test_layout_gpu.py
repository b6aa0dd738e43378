"""Bit-exact parity of the GPU index compaction (VS merge, A-shape, areas)
with the reference (golden) and the oracle restatements; the reference's own
hand traces (test_vs_index.py:19-57) are replayed verbatim."""

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2407_02490_b200 as P

    return P


def test_vs_golden_layouts(golden, P):
    names = sorted({k.split("__")[0] for k in golden.files if k.startswith("vs_")})
    for name in names:
        s, d, kv, ks, lq, seed, bf16, b = (int(x) for x in golden[f"{name}__params"])
        idx = P.VSIndices(vertical=golden[f"{name}__vertical"], slash=golden[f"{name}__slash"])
        layout, ops = P.build_vs_layout_with_stats(idx, s, b)
        t, to, c, co = layout.csr()
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"], err_msg=name)
        np.testing.assert_array_equal(to, golden[f"{name}__tile_off"], err_msg=name)
        np.testing.assert_array_equal(c, golden[f"{name}__cols"], err_msg=name)
        np.testing.assert_array_equal(co, golden[f"{name}__col_off"], err_msg=name)
        np.testing.assert_array_equal(np.asarray(ops), golden[f"{name}__ops"], err_msg=name)
        assert P.layout_area(layout) == int(golden[f"{name}__area"])


def test_hand_traces(P):
    V = P.VSIndices
    lay = P.build_vs_layout(V(vertical=[0], slash=[0]), 8, 4)
    assert lay.block_starts == [[0], [4]] and lay.column_indices == [[], [0]]
    lay = P.build_vs_layout(V(vertical=[7], slash=[4, 2]), 8, 4)
    assert lay.block_starts[1] == [0, 4] and lay.column_indices[1] == []
    lay = P.build_vs_layout(V(vertical=[6], slash=[12, 0]), 16, 4)
    assert lay.block_starts[3] == [0, 12] and lay.column_indices[3] == [6]
    lay = P.build_vs_layout(V(vertical=[1, 3], slash=[0]), 8, 4)
    assert lay.block_starts[0] == [0] and lay.column_indices[0] == []
    lay = P.build_vs_layout(V(vertical=[0], slash=[6]), 8, 4)
    assert lay.block_starts[0] == [] and lay.column_indices[0] == [0]
    lay = P.build_vs_layout(V(vertical=[0], slash=[3]), 8, 4)
    assert lay.block_starts[0] == [0]


def test_range_checks(P):
    with pytest.raises(ValueError):
        P.build_vs_layout(P.VSIndices(vertical=[8], slash=[0]), 8, 4)
    with pytest.raises(ValueError):
        P.build_vs_layout(P.VSIndices(vertical=[0], slash=[8]), 8, 4)
    with pytest.raises(ValueError):
        P.build_vs_layout(P.VSIndices(vertical=[0], slash=[0]), 8, 0)


def test_random_merges_match_oracle(P, rng):
    # test_vs_index.py:74-99 style: 500 random instances, exact CSR equality
    for trial in range(500):
        s_len = int(rng.integers(4, 300))
        b = int(rng.choice([2, 4, 8, 64]))
        kv = int(rng.integers(1, min(40, s_len) + 1))
        ks = int(rng.integers(1, min(40, s_len) + 1))
        vertical = np.sort(rng.choice(s_len, size=kv, replace=False))
        slash = -np.sort(-rng.choice(s_len, size=ks, replace=False))
        layout, ops = P.build_vs_layout_with_stats(P.VSIndices(vertical=vertical, slash=slash), s_len, b)
        wt, wc, wops = port.build_vs_layout_with_stats(vertical, slash, s_len, b)
        assert layout.block_starts == wt, trial
        assert layout.column_indices == wc, trial
        assert ops == wops, trial


def test_large_merge_matches_c_oracle(P, rng):
    s_len, b = 131072, 64
    vertical = np.sort(rng.choice(s_len, size=1000, replace=False))
    slash = -np.sort(-rng.choice(s_len, size=6096, replace=False))
    layout = P.build_vs_layout(P.VSIndices(vertical=vertical, slash=slash), s_len, b)
    t, to, c, co = layout.csr()
    wt, wto, wc, wco = port.build_vs_csr(vertical, slash, s_len, b)
    np.testing.assert_array_equal(to, wto)
    np.testing.assert_array_equal(t, wt)
    np.testing.assert_array_equal(co, wco)
    np.testing.assert_array_equal(c, wc)


@pytest.mark.parametrize("kind", ["band", "spaced_b", "spaced_b1", "clustered", "dense_v", "unstaged"])
def test_structured_merges_match_c_oracle(P, rng, kind):
    """Slash patterns that stress the coalescing rule of the warp-parallel
    merge: one contiguous band (G-local), offsets exactly B and B+1 apart
    (every range a gap candidate, half of them coalesced by the cover rule),
    and clustered offsets; dense verticals (groups absorbing and rows emitting
    hundreds of points: the warp-wide partition searches) with the lists staged
    in shared memory and, past its capacity, read from global memory."""
    s_len, b = 65536 + 37, 64
    if kind == "band":
        slash = np.arange(6095, -1, -1)
    elif kind == "spaced_b":
        slash = np.arange(0, 64 * 900, 64)[::-1]
    elif kind == "spaced_b1":
        slash = np.arange(0, 65 * 900, 65)[::-1]
    elif kind == "clustered":
        centers = rng.choice(s_len - 200, size=60, replace=False)
        slash = np.unique((centers[:, None] + rng.integers(0, 150, size=(60, 40))).ravel())[::-1]
    elif kind == "dense_v":
        slash = np.arange(6095, -1, -1)
    else:  # unstaged: n_v + 2 n_s above the shared-memory capacity (24K indices)
        slash = np.sort(rng.choice(s_len, size=8000, replace=False))[::-1]
    slash = slash[slash < s_len]
    n_v = {"dense_v": 6000, "unstaged": 10000}.get(kind, 1000)
    vertical = np.sort(rng.choice(s_len, size=n_v, replace=False))
    layout = P.build_vs_layout(P.VSIndices(vertical=vertical, slash=slash), s_len, b)
    t, to, c, co = layout.csr()
    wt, wto, wc, wco = port.build_vs_csr(vertical, slash, s_len, b)
    np.testing.assert_array_equal(to, wto)
    np.testing.assert_array_equal(t, wt)
    np.testing.assert_array_equal(co, wco)
    np.testing.assert_array_equal(c, wc)


def test_ashape_golden_and_random(golden, P, rng):
    names = sorted({k.split("__")[0] for k in golden.files if k.startswith("as_")})
    for name in names:
        s, d, g, w, b, seed, bf16 = (int(x) for x in golden[f"{name}__params"])
        lay = P.a_shape_layout(s, P.AShape(g, w), b)
        t, to, _, _ = lay.csr()
        np.testing.assert_array_equal(t, golden[f"{name}__tiles"], err_msg=name)
        np.testing.assert_array_equal(to, golden[f"{name}__tile_off"], err_msg=name)
        assert P.layout_area(lay) == int(golden[f"{name}__area"])
    for _ in range(200):
        s = int(rng.integers(1, 700))
        b = int(rng.choice([3, 4, 16, 64]))
        g, w = int(rng.integers(1, s + 50)), int(rng.integers(1, s + 50))
        lay = P.a_shape_layout(s, P.AShape(g, w), b)
        assert lay.block_starts == port.a_shape_layout(s, g, w, b)


def test_bs_golden_area(golden, P):
    names = sorted({k.split("__")[0] for k in golden.files if k.startswith("bs_")})
    for name in names:
        s, d, kb, b, seed, bf16 = (int(x) for x in golden[f"{name}__params"])
        t, to = golden[f"{name}__tiles"], golden[f"{name}__tile_off"]
        n = to.size - 1
        lay = P.SparseLayout.from_csr(s, b, t, to, np.zeros(0, np.int64), np.zeros(n + 1, np.int64))
        assert P.layout_area(lay) == int(golden[f"{name}__area"])


def test_area_matches_mask_popcount(P):
    # test_patterns.py:97-112: tile-only layouts, area == masked cell count
    for seed in range(10):
        rng = np.random.Generator(np.random.PCG64(seed))
        s_len = int(rng.integers(5, 80))
        b = int(rng.choice([2, 4, 8]))
        lay = P.SparseLayout(s_len, b, [], [])
        for r in range((s_len + b - 1) // b):
            q_end = min((r + 1) * b, s_len)
            choices = np.arange(0, q_end, b)
            take = rng.random(choices.size) < 0.5
            lay.block_starts.append([int(x) for x in choices[take]])
            lay.column_indices.append([])
        lay.validate()
        assert P.layout_area(lay) == int(P.layout_to_mask(lay).sum())
