"""Synthetic workloads for the benchmark configs of BASELINE.json.

* G-iid   : Q, K, V ~ N(0, 1), bf16.
* G-local : "linear-locality" inputs, exact in bf16: noise sigma = 0.5 on all
            dims, key digit columns K[:,0..2] = (j mod 256, (j>>8) mod 256, j>>16),
            query columns Q[:,0..2] = alpha * (1, 256, 65536) with alpha = 2^-3
            so q.k contains alpha*j exactly; sink K[0:4, 3] = 64, Q[:, 3] = 1.
            With VS(1000, 6096) the reference selects the slash band 0..k_s-1
            and the layouts are ~0.82 (64K) .. ~0.99 (1M) sparse.
* C2 head configs: the reference ships no per-head config for LLaMA-3-8B-1M
  (SURVEY.md section 5), so a documented deterministic mix following
  PAPER.md:938 is used: VS(1000, 6096) everywhere except AShape(1024, 4096)
  on heads h % 16 == 3 of layers 8..15 and BlockSparse(100) on heads
  h % 16 == 7 of layers 16..23 (992 VS / 16 A-shape / 16 BS heads, 96.9 % VS).
  ``configs/llama3_8b_1m_c2.json`` is this mix in the config JSON v1 format.
"""

from __future__ import annotations

import os

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C2_CONFIG = os.path.join(REPO, "configs", "llama3_8b_1m_c2.json")


def g_local_qkv(hq: int, hkv: int, s: int, d: int, seed: int, device="cuda"):
    g = torch.Generator(device=device).manual_seed(seed)
    q = torch.randn((hq, s, d), generator=g, device=device) * 0.5
    k = torch.randn((hkv, s, d), generator=g, device=device) * 0.5
    v = torch.randn((hkv, s, d), generator=g, device=device)
    j = torch.arange(s, device=device)
    k[:, :, 0] = (j % 256).float()
    k[:, :, 1] = ((j >> 8) % 256).float()
    k[:, :, 2] = (j >> 16).float()
    alpha = 2.0 ** -3
    q[:, :, 0] = alpha
    q[:, :, 1] = alpha * 256
    q[:, :, 2] = alpha * 65536
    k[:, :4, 3] = 64.0
    q[:, :, 3] = 1.0
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)


def g_iid_qkv(hq: int, hkv: int, s: int, d: int, seed: int, device="cuda"):
    g = torch.Generator(device=device).manual_seed(seed)
    q = torch.randn((hq, s, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    k = torch.randn((hkv, s, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    v = torch.randn((hkv, s, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    return q, k, v


def c2_head_configs(n_layers: int = 32, n_heads: int = 32):
    from paper_2407_02490_b200.patterns import AShape, BlockSparse, VerticalSlash

    layers = []
    for layer in range(n_layers):
        row = []
        for h in range(n_heads):
            if 8 <= layer < 16 and h % 16 == 3:
                row.append(AShape(1024, 4096))
            elif 16 <= layer < 24 and h % 16 == 7:
                row.append(BlockSparse(100))
            else:
                row.append(VerticalSlash(1000, 6096))
        layers.append(row)
    return layers


def load_layer_configs(path: str = C2_CONFIG):
    """Config JSON v1 (patterns.py:236-266) -> per-layer lists of configs."""
    from paper_2407_02490_b200.patterns import config_from_entry, load_pattern_configs

    entries = [config_from_entry(e) for e in load_pattern_configs(path)]
    n_layers = 1 + max(e[0] for e in entries)
    n_heads = 1 + max(e[1] for e in entries)
    layers = [[None] * n_heads for _ in range(n_layers)]
    for layer, head, cfg in entries:
        layers[layer][head] = cfg
    return layers


def write_c2_config(path: str = C2_CONFIG):
    from paper_2407_02490_b200.patterns import config_to_entry, save_pattern_configs

    entries = [config_to_entry(layer, h, cfg) for layer, row in enumerate(c2_head_configs()) for h, cfg in enumerate(row)]
    save_pattern_configs(path, entries)


if __name__ == "__main__":
    write_c2_config()
    print("wrote", C2_CONFIG)
