"""Host-side parity of the pattern-search calibration (pure cost model,
search.py:46-115 of the reference) and of the report writers, against fixtures
the reference produced (tests/golden/make_metrics_golden.py)."""

import json
import os

import pytest

from conftest import REPO

GOLDEN = os.path.join(REPO, "tests", "golden", "metrics_golden.json")


def cfg_from_json(P, c):
    if c[0] == "a_shape":
        return P.AShape(c[1], c[2])
    if c[0] == "vertical_slash":
        return P.VerticalSlash(c[1], c[2], c[3])
    return P.BlockSparse(c[1], c[2])


@pytest.fixture(scope="module")
def gold():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def P():
    import paper_2407_02490_b200 as P

    return P


def test_calibration_matches_reference(gold, P):
    from paper_2407_02490_b200 import search

    for case in gold["calibration"]:
        seeds = [cfg_from_json(P, c) for c in case["seeds"]]
        cands = search.calibrate_search_space(seeds, case["budget"], case["step"], case["eps"], case["s"], case["d"],
                                              case["block_size"])
        got = [[c.cfg, c.modeled_flops, c.at_bound] for c in cands]
        want = [[cfg_from_json(P, c), f, b] for c, f, b in case["candidates"]]
        assert got == want, case


def test_calibration_errors(P):
    from paper_2407_02490_b200 import search

    with pytest.raises(ValueError):
        search.calibrate_search_space([], None, 50, 0.1, 1024, 64)
    with pytest.raises(ValueError):
        search.calibrate_search_space([P.AShape(1, 1)], None, 0, 0.1, 1024, 64)
    with pytest.raises(ValueError):
        search.calibrate_search_space([P.AShape(1, 1)], -5, 10, 0.1, 1024, 64)
    with pytest.raises(TypeError):
        search.calibrate_candidate(object(), 10, 1, 0.1, 128, 64, 64)


def test_modeled_flops_of_reports(gold, P):
    from paper_2407_02490_b200.patterns import flops_in_kernel

    for r in gold["reports"]:
        cfg = cfg_from_json(P, r["cfg"])
        assert flops_in_kernel(cfg, r["s"], r["d"], r["block_size"]) == r["modeled_flops"]


def test_report_writers(tmp_path):
    from paper_2407_02490_b200 import metrics

    reps = [metrics.RunReport("0", "vertical_slash", 0.5, 0.25, 123, 1e-3, 0.1, 0.2),
            metrics.RunReport("h1", "a_shape", 1.0, -0.0038361638361639194, 7, 2.5e-09, 0.0, 0.0)]
    p = tmp_path / "r.csv"
    metrics.reports_to_csv(reps, p)
    assert p.read_text() == ("head,pattern,recall,kernel_sparsity,modeled_flops,output_mae\n"
                             "0,vertical_slash,0.5,0.25,123,0.001\n"
                             "h1,a_shape,1,-0.003836163836,7,2.5e-09\n")
    metrics.reports_to_csv(reps, p, include_timings=True)
    assert p.read_text().splitlines()[0].endswith(",t_estimate,t_sparse")
    j = tmp_path / "r.json"
    metrics.reports_to_json(reps, j)
    rows = json.loads(j.read_text())
    assert rows[0]["modeled_flops"] == 123 and set(rows[0]) == set(metrics.CSV_COLUMNS + metrics.CSV_TIMING_COLUMNS)
