"""Cycle trace of the paired-box kernel's union-pairing softmax (build with -DSPF_PAIR_UNION=1
-DSPF_PAIR_TRACE=1 [-DSPF_PAIR_DB=1 [-DSPF_PAIR_HALVES=2]] and load it via SPF_LIB_OVERRIDE):
median cycles per segment of softmax warp 2 over the first 300 CTAs, steps 5..29, on a
C2-shaped A-shape(128, 4096) layer with every head listed for the paired-box kernel."""
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_02490_b200 as P
from paper_2407_02490_b200 import _lib, kernels
from benchmarks.workloads import g_local_qkv
q, k, v = g_local_qkv(32, 8, 131072, 128, seed=0)
lay = P.build_layer_layout(q, k, [P.AShape(128, 4096)] * 32, 64)
out = torch.empty_like(q)
lib = _lib.load()
n_ctas = 300
buf = torch.zeros(n_ctas * 64 * 8, dtype=torch.int64, device="cuda")
lib.spf_debug_pair_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
pl = torch.arange(32, dtype=torch.int32, device="cuda")
run = lambda: kernels.sparse_flash_attention_gpu(q, k, v, 128 ** -0.5, 64, lay.tiles, lay.tile_offsets, lay.cols, lay.col_offsets, out=out, pair_heads=pl)
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
lib.spf_debug_pair_trace(ctypes.c_void_p(buf.data_ptr()), n_ctas)
run(); torch.cuda.synchronize()
tr = buf.cpu().numpy().reshape(n_ctas, 64, 8).astype(np.float64)[:, 5:30, :]
ok = tr[:, -1, 0] > 0
tr = tr[ok]
seg = lambda a, b: np.median(tr[:, :, b] - tr[:, :, a])
print(os.environ.get("SPF_LIB_OVERRIDE"), "layer ms %.2f" % e0.elapsed_time(e1), "ctas", ok.sum(),
      "| period %.0f" % np.median(np.diff(tr[:, :, 0], axis=1)),
      "top->S %.0f  S->ld %.0f  ld->max %.0f  max->exps %.0f  exps->Pst %.0f" % (seg(0, 1), seg(1, 2), seg(2, 3), seg(3, 4), seg(4, 6)))
