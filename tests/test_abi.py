"""CPU: the C-ABI library loads and exports every symbol include/spf.h
declares; host-side config types / JSON / validation mirror the reference."""

import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "spf.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_2407_02490_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert _lib.load().spf_version() == 1
    assert _lib.missing_symbols() == []


def test_library_is_sm100a():
    import subprocess

    from paper_2407_02490_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch

    import paper_2407_02490_b200 as P

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        P.estimate_vertical_slash(np.zeros((8, 4), np.float32), np.zeros((8, 4), np.float32), P.VerticalSlash(2, 2, 4))


def test_configs_and_json(tmp_path):
    import paper_2407_02490_b200 as P
    from paper_2407_02490_b200.patterns import config_from_entry, config_to_entry

    with pytest.raises(ValueError):
        P.AShape(0, 4)
    with pytest.raises(ValueError):
        P.VerticalSlash(1, 0)
    with pytest.raises(ValueError):
        P.BlockSparse(0)
    for cfg in (P.AShape(64, 256), P.VerticalSlash(30, 2048, 64), P.BlockSparse(100, 64)):
        assert config_from_entry(config_to_entry(0, 3, cfg)) == (0, 3, cfg)
    with pytest.raises(ValueError):
        config_from_entry({"layer": 0, "head": 0, "pattern": "nope", "params": {}})
    entries = [config_to_entry(0, i, P.VerticalSlash(8, 16)) for i in range(3)]
    path = tmp_path / "cfg.json"
    P.save_pattern_configs(path, entries)
    assert P.load_pattern_configs(path) == entries
    path.write_text('{"format_version": 99, "heads": []}')
    with pytest.raises(ValueError):
        P.load_pattern_configs(path)


def test_layout_validate_mirrors_reference():
    from paper_2407_02490_b200.patterns import SparseLayout

    SparseLayout(8, 4, [[0], [0, 4]], [[], []]).validate()
    for bad in (SparseLayout(8, 4, [[0], [0, 2]], [[], []]),      # overlapping tiles
                SparseLayout(8, 4, [[0], [4]], [[], [5]]),         # column inside tile
                SparseLayout(8, 4, [[], []], [[5], []]),           # acausal column
                SparseLayout(8, 4, [[0]], [[]]),                   # wrong row count
                SparseLayout(8, 4, [[4], []], [[], []]),           # acausal tile
                SparseLayout(8, 4, [[], [4, 0]], [[], []])):       # unsorted
        with pytest.raises(ValueError):
            bad.validate()
    SparseLayout(8, 4, [[0], []], [[], [7]]).validate()


def test_flops_model_matches_reference_formulas():
    import paper_2407_02490_b200 as P
    from oracle import port

    # criterion 5 (test_acceptance.py:167-174): dense/sparse ~ S/(2*B*k_b)
    s, b, kb, d = 131072, 64, 100, 64
    ratio = 4 * d * P.causal_area(s) / P.flops_in_kernel(P.BlockSparse(kb, b), s, d, b)
    assert abs(ratio - s / (2 * b * kb)) / (s / (2 * b * kb)) <= 0.10
    assert P.flops_in_kernel(P.BlockSparse(16, 4), 64, 1, 4) == 4 * P.causal_area(64)
    f1 = P.flops_in_kernel(P.VerticalSlash(8, 64), 1024, 16, 64)
    f2 = P.flops_in_kernel(P.VerticalSlash(8, 512), 1024, 16, 64)
    f3 = P.flops_in_kernel(P.VerticalSlash(256, 512), 1024, 16, 64)
    assert f1 < f2 <= f3
    assert P.flops_in_kernel(P.VerticalSlash(4096, 4096), 256, 1, 64) <= 4 * P.causal_area(256)
    # BS area model == realized layout area (exact): compare with the port
    rows = [list(range(min(3, r + 1))) for r in range(16)]
    rows = [sorted(set(r[:-1] + [i])) for i, r in enumerate(rows)]
    assert port.layout_area(1000, 64, port.block_rows_to_tiles(rows, 64), [[] for _ in rows]) > 0
