"""Time to first token of a LLaMA-3-8B-shaped model (random bf16 weights) with dense
attention (torch SDPA) vs the sparse pre-fill hook (paper_2407_02490_b200.hf) driven by
the C2 per-head pattern table -- the end-to-end view of SURVEY.md 8(f)4.

    python benchmarks/ttft_llama.py [--seq 131072] [--layers 32] [--reps 2]

Pre-fill of one sequence, logits of the last token only; CUDA-event timing after a
warm-up.  The model is LLaMA-3-8B's shape (hidden 4096, 32 q / 8 kv heads, head_dim 128,
MLP 14336, vocab 128256) with random weights: the timing does not depend on the
weights, the pattern table is the benchmark's synthetic C2 mix.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--patterns", default="c2", choices=["c2", "ashape"],
                    help="c2: the data-dependent C2 mix (with random weights Q/K have no locality, so the "
                         "estimated Vertical-Slash layouts come out nearly dense); ashape: static "
                         "A-shape(1024, 4096) on every head (sparse whatever the weights)")
    args = ap.parse_args()
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    from benchmarks.workloads import load_layer_configs
    from paper_2407_02490_b200 import hf
    from paper_2407_02490_b200.driver import PatternTable

    cfg = LlamaConfig(vocab_size=128256, hidden_size=4096, intermediate_size=14336, num_hidden_layers=args.layers,
                      num_attention_heads=32, num_key_value_heads=8, head_dim=128,
                      max_position_embeddings=max(args.seq, 8192), rope_theta=500000.0)
    torch.manual_seed(0)
    torch.set_default_dtype(torch.bfloat16)
    with torch.device("cuda"):
        model = LlamaForCausalLM(cfg).eval()
    torch.set_default_dtype(torch.float32)
    ids = torch.randint(0, cfg.vocab_size, (1, args.seq), device="cuda")
    from paper_2407_02490_b200.patterns import AShape

    table = PatternTable(load_layer_configs()[: args.layers] if args.patterns == "c2"
                         else [[AShape(1024, 4096)] * 32] * args.layers)
    sparse_impl = hf.register(table)

    def ttft(impl):
        model.set_attn_implementation(impl)
        times = []
        with torch.no_grad():
            for r in range(args.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                logits = model(ids, logits_to_keep=1, use_cache=False).logits
                e1.record()
                torch.cuda.synchronize()
                if r > 0:
                    times.append(e0.elapsed_time(e1))
        return min(times), logits.float()

    dense_ms, dense_logits = ttft("sdpa")
    sparse_ms, sparse_logits = ttft(sparse_impl)
    res = {"model": "LLaMA-3-8B shape, random bf16 weights", "layers": args.layers, "seq_len": args.seq,
           "ttft_dense_sdpa_ms": round(dense_ms, 1), "ttft_sparse_ms": round(sparse_ms, 1),
           "speedup": round(dense_ms / sparse_ms, 2),
           "patterns": args.patterns, "pattern_counts": table.pattern_counts(),
           "last_token_logit_max_abs_diff": round((dense_logits - sparse_logits).abs().max().item(), 4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
