"""The union kernel on a dense causal layout (A-shape with a window covering S) against torch
SDPA (cuDNN / flash) on the same tensors: S = 32K, 32 q / 8 kv heads, d = 128, bf16."""
import os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch
import torch.nn.functional as F
import paper_2407_02490_b200 as P
from paper_2407_02490_b200 import kernels
from benchmarks.workloads import g_iid_qkv

S = int(os.environ.get("S", "32768")); HQ, HKV, D, B = 32, 8, 128, 64
q, k, v = g_iid_qkv(HQ, HKV, S, D, seed=0, device="cuda")
lay = P.build_layer_layout(q, k, [P.AShape(64, S)] * HQ, B)
out = torch.empty_like(q)
run = lambda: kernels.sparse_flash_attention_gpu(q, k, v, D ** -0.5, B, lay.tiles, lay.tile_offsets, lay.cols,
                                                 lay.col_offsets, out=out)
rep = HQ // HKV
kk, vv = k.repeat_interleave(rep, 0)[None], v.repeat_interleave(rep, 0)[None]
sdpa = lambda: F.scaled_dot_product_attention(q[None], kk, vv, is_causal=True)
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
flops_causal = 4 * D * HQ * S * S / 2
t_ours, t_sdpa = timed(run), timed(sdpa)
err = (out.float() - sdpa().float()).abs().max().item()
print(f"S={S} dense causal: union kernel {t_ours:.3f} ms ({flops_causal / t_ours / 1e9:.0f} TF/s), "
      f"SDPA {t_sdpa:.3f} ms ({flops_causal / t_sdpa / 1e9:.0f} TF/s), max|diff| {err:.2e}")
