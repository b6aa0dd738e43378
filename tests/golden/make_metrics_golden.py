"""Golden fixtures for the GPU report and pattern-search modules, produced by the
REFERENCE package itself (metrics.report_head, attention_ref.attention_recall,
search.calibrate_search_space / search_optimal_pattern).

Run in the build container (where /root/reference exists):

    make -C oracle
    python tests/golden/make_metrics_golden.py

Inputs are regenerated from seeds by ``oracle.port.seeded_gaussian`` (the
reference's tensor.py:81-90 generator); only the reference's outputs are stored
(tests/golden/metrics_golden.json).
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import port  # noqa: E402

ref_core = port.load_ref_core()
if ref_core is not None:
    sys.modules["sparseprefill._core"] = ref_core

from sparseprefill import metrics, search  # noqa: E402
from sparseprefill.attention_ref import AttentionInputs, attention_recall  # noqa: E402
from sparseprefill.patterns import AShape, BlockSparse, VerticalSlash, layout_to_mask  # noqa: E402
from sparseprefill.sparse_attn import run_head  # noqa: E402


def cfg_to_json(cfg):
    if isinstance(cfg, AShape):
        return ["a_shape", cfg.global_tokens, cfg.local_window]
    if isinstance(cfg, VerticalSlash):
        return ["vertical_slash", cfg.k_v, cfg.k_s, cfg.last_q]
    return ["block_sparse", cfg.k_b, cfg.block_size]


def inputs(s, d, seed):
    return AttentionInputs(port.seeded_gaussian(s, d, seed), port.seeded_gaussian(s, d, seed + 1),
                           port.seeded_gaussian(s, d, seed + 2))


def main():
    out = {"backend": __import__("sparseprefill").kernels.BACKEND, "reports": [], "recall": [], "calibration": [],
           "search": []}
    # per-head reports (metrics.py:54-70)
    for s, d, seed, cfg, b in [(512, 64, 7, VerticalSlash(40, 120), 64), (700, 64, 11, AShape(64, 256), 64),
                               (640, 32, 13, BlockSparse(3, 32), 64), (1000, 128, 17, VerticalSlash(100, 300), 64),
                               (333, 16, 19, VerticalSlash(8, 20, 16), 32)]:
        rep = metrics.report_head(inputs(s, d, seed), cfg, head=f"h{seed}", block_size=b)
        out["reports"].append({"s": s, "d": d, "seed": seed, "cfg": cfg_to_json(cfg), "block_size": b,
                               "head": rep.head, "pattern": rep.pattern, "recall": rep.recall,
                               "kernel_sparsity": rep.kernel_sparsity, "modeled_flops": rep.modeled_flops,
                               "output_mae": rep.output_mae})
    # recall of a planted-free Gaussian head under several layouts (attention_ref.py:128-139)
    for s, d, seed, cfg, b in [(256, 32, 23, VerticalSlash(10, 30), 16), (300, 64, 29, AShape(32, 64), 64),
                               (400, 64, 31, BlockSparse(2), 64)]:
        x = inputs(s, d, seed)
        _, layout = run_head(x, cfg, b)
        out["recall"].append({"s": s, "d": d, "seed": seed, "cfg": cfg_to_json(cfg), "block_size": b,
                              "recall": attention_recall(layout_to_mask(layout), x)})
    # calibration (search.py:62-115): pure cost model
    seeds = [VerticalSlash(1000, 6096), VerticalSlash(100, 500), BlockSparse(100), BlockSparse(4, 32),
             AShape(128, 4096), AShape(64, 64)]
    for s, d, b, budget, step, eps in [(131072, 128, 64, None, 50, 0.1), (8192, 128, 64, None, 50, 0.1),
                                       (4096, 64, 64, 3 * 10 ** 9, 7, 0.05), (1000, 64, 32, 10 ** 8, 1, 0.01)]:
        cands = search.calibrate_search_space(seeds, budget, step, eps, s, d, b)
        out["calibration"].append({"s": s, "d": d, "block_size": b, "budget": budget, "step": step, "eps": eps,
                                   "seeds": [cfg_to_json(c) for c in seeds],
                                   "candidates": [[cfg_to_json(c.cfg), c.modeled_flops, c.at_bound]
                                                  for c in cands]})
    # search on a validation head (search.py:118-138)
    for s, d, seed, budget in [(768, 64, 37, 6 * 10 ** 7), (1024, 128, 41, None)]:
        cands = search.calibrate_search_space([VerticalSlash(30, 100), BlockSparse(4), AShape(64, 128)], budget, 10,
                                              0.1, s, d, 64)
        res = search.search_optimal_pattern(inputs(s, d, seed), cands, 64)
        out["search"].append({"s": s, "d": d, "seed": seed, "budget": budget,
                              "candidates": [[cfg_to_json(c.cfg), c.modeled_flops, c.at_bound, c.fidelity_error]
                                             for c in res.candidates],
                              "chosen": cfg_to_json(res.chosen.cfg)})
    path = os.path.join(HERE, "metrics_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
