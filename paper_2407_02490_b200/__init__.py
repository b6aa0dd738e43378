"""B200-native (sm_100a) dynamic sparse pre-fill attention (MInference, arXiv 2407.02490).

Drop-in for the hot path of the reference ``sparseprefill`` package:
online estimation -> index compaction -> sparse FlashAttention for A-shape,
Vertical-Slash and Block-Sparse heads.  The public names mirror the
reference's (``sparseprefill/__init__.py:9-40``) for that path; compute runs
in ``libspf.so`` (hand-written CUDA for sm_100a, see include/spf.h).
"""

from .estimator import (
    BlockIndices,
    VSIndices,
    argtopk,
    estimate_block_sparse,
    estimate_block_sparse_gpu,
    estimate_vertical_slash,
    estimate_vertical_slash_gpu,
)
from .kernels import BACKEND, available_backends, sparse_flash_attention, sparse_flash_attention_gpu
from .metrics import (
    RunReport,
    attention_recall_gpu,
    dense_layout,
    kernel_sparsity,
    modeled_kernel_sparsity,
    report_head,
    report_layer,
    reports_to_csv,
    reports_to_json,
)
from .patterns import (
    AShape,
    BlockSparse,
    SparseLayout,
    VerticalSlash,
    a_shape_layout,
    causal_area,
    config_from_entry,
    config_to_entry,
    flops_in_kernel,
    layout_area,
    layout_to_mask,
    load_pattern_configs,
    save_pattern_configs,
)
from .prefill import LayerLayout, build_layer_layout, sparse_prefill_attention
from .search import (
    SearchCandidate,
    SearchResult,
    calibrate_candidate,
    calibrate_search_space,
    candidate_errors_gpu,
    default_budget,
    search_optimal_pattern,
)
from .sparse_attn import (
    AttentionInputs,
    block_indices_to_layout,
    block_sparse_attention,
    run_head,
    run_head_timed,
    vertical_slash_attention,
)
from .vs_index import build_vs_layout, build_vs_layout_with_stats

__version__ = "0.1.0"
