"""A/B timing of two libspf builds on the same inputs, interleaved (attention only).

    python benchmarks/ab_attention.py A/libspf.so B/libspf.so     # AB_CFG=vs|bs|as AB_SEQ=131072 AB_REPS=12
    AB_HQ=56 AB_GEN=iid AB_PAIR=1 AB_CFG=bs AB_SEQ=262144 ...       # the C4 layer through the paired-box kernel

Both libraries are loaded side by side with ctypes and launched alternately on one
C2-shaped layer (32 q-heads, 8 kv, d=128, G-local), so clock and power drift hit
both builds alike; prints the median times and their ratio.
"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_02490_b200 as P
from benchmarks.workloads import g_iid_qkv, g_local_qkv
libs = [ctypes.CDLL(os.path.abspath(p)) for p in sys.argv[1:3]]
seq = int(os.environ.get("AB_SEQ", "131072"))
hq = int(os.environ.get("AB_HQ", "32"))
gen = g_iid_qkv if os.environ.get("AB_GEN", "local") == "iid" else g_local_qkv
q, k, v = gen(hq, 8, seq, 128, seed=0, device="cuda")
cfg = os.environ.get("AB_CFG", "vs")
cfgs = {"vs": [P.VerticalSlash(1000, 6096)] * hq, "bs": [P.BlockSparse(100)] * hq, "as": [P.AShape(128, 4096)] * hq,
        "tiny": [P.AShape(1, 64)] * hq, "small": [P.AShape(64, 640)] * hq,
        # C2's mixed Block-Sparse layers: BS(100) on heads 7 and 23, VS elsewhere
        "mix": [P.BlockSparse(100) if h % 16 == 7 else P.VerticalSlash(1000, 6096) for h in range(hq)]}[cfg]
# AB_PAIR=1: every head through the paired-box kernel; AB_CFG=mix lists its Block-Sparse heads
pair_ids = [h for h in range(hq) if h % 16 == 7] if cfg == "mix" else list(range(hq))
pair = torch.tensor(pair_ids, dtype=torch.int32, device="cuda")
n_pairs = [len(pair_ids) if os.environ.get(f"AB_PAIR_{x}", os.environ.get("AB_PAIR", "0")) == "1" else 0 for x in "AB"]
lay = P.build_layer_layout(q, k, cfgs, 64)
out = torch.empty_like(q)
vp = ctypes.c_void_p
for lib in libs:
    lib.spf_sparse_flash_workspace_size.restype = ctypes.c_size_t
ws_bytes = max(int(lib.spf_sparse_flash_workspace_size(0, hq, 8, seq, 128)) for lib in libs)
ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
def run(lib, n_pair):
    lib.spf_sparse_flash_rows_ex.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_float, ctypes.c_int, vp, vp, vp, vp, vp,
                                             ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp]
    rc = lib.spf_sparse_flash_rows_ex(0, vp(q.data_ptr()), vp(k.data_ptr()), vp(v.data_ptr()), hq, 8, seq, 128,
                                      ctypes.c_float(128 ** -0.5), 64, vp(lay.tiles.data_ptr()),
                                      vp(lay.tile_offsets.data_ptr()), vp(lay.cols.data_ptr() if lay.cols.numel() else 0),
                                      vp(lay.col_offsets.data_ptr()), vp(pair.data_ptr()), n_pair, vp(out.data_ptr()), None,
                                      vp(ws.data_ptr()), ws_bytes, vp(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
ts = [[], []]
for r in range(int(os.environ.get("AB_REPS", "12"))):
    for i, lib in enumerate(libs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(lib, n_pairs[i]); e1.record(); torch.cuda.synchronize()
        if r >= 2:
            ts[i].append(e0.elapsed_time(e1))
print(cfg, "A %.3f ms  B %.3f ms  (B/A %.3f)" % (statistics.median(ts[0]), statistics.median(ts[1]),
                                             statistics.median(ts[1]) / statistics.median(ts[0])))
