"""How many Vertical-Slash heads the tensor-core estimation cannot certify, and how close
the selection boundary is, on C2-shaped layers (32 q / 8 kv heads, 128K, G-local,
VS(1000, 6096)).

    python benchmarks/probe_vs_certify.py [--layers 4]

Per layer: the number of heads re-estimated on the fp64 path (flags of spf_vs_estimate)
and, for the first such head, the k-th / (k+1)-th slash and vertical scores.
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    args = ap.parse_args()
    import torch

    import paper_2407_02490_b200 as P
    from benchmarks.workloads import g_local_qkv
    from paper_2407_02490_b200.estimator import vs_estimate_async

    cfg = P.VerticalSlash(1000, 6096)
    for layer in range(args.layers):
        q, k, _ = g_local_qkv(32, 8, 131072, 128, seed=1000 * layer, device="cuda")
        _, _, vsc, ssc, flags = vs_estimate_async(q, k, cfg, with_scores=True)
        torch.cuda.synchronize()
        f = flags.cpu().tolist()
        msg = ""
        for h, u in enumerate(f):
            if u:
                s = torch.sort(ssc[h], descending=True).values
                v = torch.sort(vsc[h], descending=True).values
                msg = (f"head {h}: slash k-th {s[cfg.k_s - 1].item():.4e} next {s[cfg.k_s].item():.4e}; "
                       f"vertical k-th {v[cfg.k_v - 1].item():.4e} next {v[cfg.k_v].item():.4e}")
                break
        print(f"layer {layer}: uncertain {sum(f)} of {len(f)} | {msg}")


if __name__ == "__main__":
    main()
