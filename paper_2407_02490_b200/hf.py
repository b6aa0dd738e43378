"""Hugging Face transformers integration: the dynamic sparse pre-fill
as an attention implementation for LLaMA-family models.

    from paper_2407_02490_b200 import hf
    hf.register(table)      # driver.PatternTable ([layer][head] configs), a list of
                            # per-head configs, or one config for every head
    model = AutoModelForCausalLM.from_config(cfg, attn_implementation=hf.ATTN_IMPLEMENTATION)

A pre-fill call (query length == key length, no KV-cache prefix) runs
``prefill.sparse_prefill_attention`` for the layer's heads -- estimation, index
compaction and the sparse kernel on the GPU, GQA kept -- with the layer's per-head
patterns (``module.layer_idx`` selects the table row).  Decode steps (one query
against a cached prefix) are outside the pre-fill path: MInference keeps them dense,
and so does this hook (torch SDPA on the GPU).  Padded batches are not supported on
the sparse path (causal, unpadded sequences only), as in the reference.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from .driver import PatternTable
from .patterns import AShape, BlockSparse, VerticalSlash
from .prefill import sparse_prefill_attention

ATTN_IMPLEMENTATION = "minference_b200"

_table = None  # PatternTable | list | config


def _layer_cfgs(layer_idx: int, n_heads: int):
    t = _table
    if isinstance(t, PatternTable):
        row = t.layer(layer_idx if layer_idx is not None else 0)
    elif isinstance(t, (list, tuple)):
        row = list(t)
    elif isinstance(t, (AShape, VerticalSlash, BlockSparse)):
        row = [t] * n_heads
    else:
        raise RuntimeError("paper_2407_02490_b200.hf: call hf.register(...) with the pattern configs first")
    if len(row) != n_heads:
        raise ValueError(f"layer {layer_idx}: {len(row)} pattern configs for {n_heads} heads")
    return row


def _is_unpadded_causal(mask: torch.Tensor) -> bool:
    """A causal mask without padding lets the last query see every key: check that row
    (bool masks: True = attend; additive masks: 0 = attend)."""
    last = mask[..., -1, :]
    if mask.dtype == torch.bool:
        return bool(last.all())
    return bool((last == 0).all())


def sparse_prefill_attention_forward(module, query, key, value, attention_mask, scaling=None, dropout=0.0,
                                     **kwargs):
    """transformers AttentionInterface signature: query [B, Hq, Sq, d], key/value
    [B, Hkv, Sk, d] -> (attn_output [B, Sq, Hq, d], None)."""
    if dropout and module.training:
        raise ValueError("the sparse pre-fill path is inference-only (dropout > 0 in training mode)")
    b, hq, sq, d = query.shape
    sk = key.shape[2]
    scale = scaling if scaling is not None else d ** -0.5
    if sq != sk:  # decode / chunked continuation: dense, like MInference
        out = F.scaled_dot_product_attention(query, key, value, attn_mask=attention_mask, scale=scale,
                                             enable_gqa=hq != key.shape[1])
        return out.transpose(1, 2).contiguous(), None
    if attention_mask is not None and not _is_unpadded_causal(attention_mask):
        raise ValueError("the sparse pre-fill path supports unpadded causal batches only "
                         "(the attention mask hides keys from the last query: padding)")
    cfgs = _layer_cfgs(getattr(module, "layer_idx", 0), hq)
    bs = next((c.block_size for c in cfgs if isinstance(c, BlockSparse)), 64)
    outs = []
    for i in range(b):
        q = query[i].to(torch.bfloat16).contiguous()
        k = key[i].to(torch.bfloat16).contiguous()
        v = value[i].to(torch.bfloat16).contiguous()
        outs.append(sparse_prefill_attention(q, k, v, cfgs, bs, scale=scale))
    out = torch.stack(outs).to(query.dtype)  # [B, Hq, S, d]
    return out.transpose(1, 2).contiguous(), None


def register(table) -> str:
    """Install the per-layer/per-head patterns and register the attention implementation
    with transformers; returns its name (``ATTN_IMPLEMENTATION``)."""
    global _table
    _table = table
    from transformers import AttentionInterface

    AttentionInterface.register(ATTN_IMPLEMENTATION, sparse_prefill_attention_forward)
    try:  # transformers >= 4.53: the mask builder is looked up by the same name
        from transformers.masking_utils import ALL_MASK_ATTENTION_FUNCTIONS, sdpa_mask

        ALL_MASK_ATTENTION_FUNCTIONS.register(ATTN_IMPLEMENTATION, sdpa_mask)
    except ImportError:
        pass
    return ATTN_IMPLEMENTATION
