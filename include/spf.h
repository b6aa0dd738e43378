/*
 * spf.h -- C ABI of libspf.so, the B200 (sm_100a) implementation of the
 * MInference dynamic sparse pre-fill path (online estimation -> index
 * compaction -> sparse FlashAttention).
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; every tensor pointer is a DEVICE pointer
 *     unless the parameter name ends in `_host`;
 *   - tensors are dense row-major: Q [n_q_heads][seq_len][head_dim],
 *     K/V [n_kv_heads][seq_len][head_dim]; q-head h reads kv-head
 *     h / (n_q_heads / n_kv_heads) (GQA);
 *   - per-(head, query-block-row) layouts are CSR: row index = h*n_rows + r,
 *     n_rows = ceil(seq_len / block_size), offsets are int64 [n_q_heads*n_rows + 1],
 *     entries int32 (tile starts / column indices, as in kernels.py:28-35 but
 *     with 32-bit entries);
 *   - work is enqueued on `stream` (a cudaStream_t; NULL = legacy default);
 *     functions return 0 on success, a non-zero SPF_ERR_* code otherwise,
 *     and spf_last_error() describes the failure (thread-local string);
 *   - nothing here allocates device memory: callers pass workspaces sized by
 *     the matching *_workspace_size() query.
 *
 * The reference interface each entry point replaces is cited inline
 * (paths relative to /root/reference/pkg/src/sparseprefill/).
 */
#ifndef SPF_H_
#define SPF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPF_OK 0
#define SPF_ERR_CUDA 1
#define SPF_ERR_INVALID 2
#define SPF_ERR_CAPACITY 3

#define SPF_DTYPE_BF16 0
#define SPF_DTYPE_F32 1

/* Library identification / error reporting. */
int spf_version(void);
const char* spf_last_error(void);
/* Number of CUDA kernels this library has launched in the process (for the
 * benchmark's gpu_launches accounting). */
unsigned long long spf_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * Sparse FlashAttention forward.
 * Replaces the kernel plugin call kernels.py:60-70 -> _core.sparse_flash_rows
 * (_core.pyx:72-192): streaming softmax over each query-block row's tiles
 * (keys [max(s,0), min(s+B,S)), per-cell causal) and then its residual
 * columns in chips of B (allowed = leading columns <= query); rows with no
 * coverage produce zeros.  Batched over heads with a GQA head map.
 *   dtype   : SPF_DTYPE_BF16 (bf16 in/out, the production path) or
 *             SPF_DTYPE_F32 (fp32 in/out via bf16x2 split, the drop-in path)
 *   out     : [n_q_heads][seq_len][head_dim] of the same dtype
 *   head_dim: <= 128 (padded internally to 64/128 through the workspace)
 * The workspace holds staged operand copies (fp32 split / padded head_dim; none for
 * bf16 at head_dim 64 or 128) followed by 16 bytes per q-head of routing statistics
 * used by spf_sparse_flash_rows_ex; a smaller workspace that still covers the copies
 * is accepted (the statistics are then skipped).
 * ------------------------------------------------------------------------- */
size_t spf_sparse_flash_workspace_size(int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim);
int spf_sparse_flash_rows(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                          int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                          const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                          void* out, void* workspace, size_t workspace_bytes, void* stream);
/* Same, and (lse_out != NULL) the per-row log-sum-exp of the cells the layout
 * covers: lse_out[h][i] = ln sum_{j in cells(i)} exp(scale * q_i.k_j), -inf for a
 * row with no cell (fp32 [n_q_heads][seq_len]).  With a dense causal layout this is
 * the softmax normaliser, so exp(lse_sparse - lse_dense) is the attention mass the
 * layout keeps: the streaming form of attention_ref.attention_recall
 * (attention_ref.py:128-139) without the S x S probability matrix. */
int spf_sparse_flash_rows_lse(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                              int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                              const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                              void* out, float* lse_out, void* workspace, size_t workspace_bytes, void* stream);
/* Same, with a per-head routing hint: pair_heads (device int32 [n_pair_heads], distinct
 * q-head ids in [0, n_q_heads); NULL when n_pair_heads == 0) lists heads whose 64-row
 * blocks have no residual columns and rarely share tiles -- the Block-Sparse heads of
 * estimator.estimate_block_sparse (estimator.py:117-143) -- which then run the
 * paired-box kernel: one step pairs the next tile of each of a CTA's two row blocks
 * (bf16, block_size 64, head_dim <= 128; otherwise the hint is ignored).  The count is
 * a host value, so a layer whose heads are all listed launches only that kernel; in a
 * mixed layer a listed head whose row blocks mostly share tiles (measured on the device
 * from the CSR) stays on the union kernel.  Results follow the same contract. */
int spf_sparse_flash_rows_ex(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                             int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                             const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                             const int32_t* pair_heads, int n_pair_heads, void* out, float* lse_out,
                             void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * argtopk (estimator.py:59-67): indices of the k largest values in descending-value
 * order, ties toward the lower index (np.argsort(-x, kind="stable")[:k]; -0.0 == 0.0).
 * values: device fp64 [n]; out: device int32 [min(k, n)]; k <= 16384.
 * ------------------------------------------------------------------------- */
size_t spf_argtopk_workspace_size(int64_t n);
int spf_argtopk(const double* values, int64_t n, int k, int32_t* out, void* workspace, size_t workspace_bytes,
                void* stream);

/* Heads selection: the estimation and layout entry points below work on a
 * subset of q-heads given by `head_ids` (device int32 [n_heads]; NULL means
 * heads 0..n_heads-1) so a layer whose heads use different patterns fills
 * one CSR over all n_q_heads (rows of other heads are left untouched).
 */

/* ---------------------------------------------------------------------------
 * Vertical-Slash online estimation.
 * Replaces estimator.py:82-114 (estimate_vertical_slash): probabilities of
 * the last `last_q` query rows against all keys (scale 1/sqrt(head_dim),
 * causal), rounded to fp32 (tensor.py:78), summed per column (vertical) and
 * per diagonal offset (slash), then top-k with ties to the lower index and
 * index 0 force-included (estimator.py:59-79).
 *   mode SPF_VS_EXACT : scores in fp64 from the bf16/fp32 inputs, sums in
 *                       fp64 in the reference's order (any shape);
 *   mode SPF_VS_FAST  : production path.  Scores on the tensor cores (tcgen05,
 *                       fp32 accumulate) for bf16 inputs with head_dim 64/128
 *                       and last_q 64 (other shapes run the exact path).  A
 *                       rigorous bound on the score error (gamma_d * sum_c
 *                       |q_c| max_j |k_jc|, estimate_vs_tc.cu) gives every
 *                       score-vector entry an interval; a head whose top-k
 *                       boundary is not separated by those intervals -- or
 *                       whose bound is too loose to try -- is re-estimated on
 *                       the fp64 path inside this call (same stream, no host
 *                       sync), skipping only keys whose probabilities provably
 *                       round to 0 in fp32.  The sets equal SPF_VS_EXACT's.
 *                       uncertain_out[i] = 1 marks the heads that were re-run.
 *   mode SPF_VS_FAST_UNCERTIFIED : test hook -- the tensor-core path alone
 *                       (no re-estimation; uncertain_out still reports the
 *                       heads the certification rejects).  Not exact.
 *   vertical_out : [n_heads][min(k_v, S)] int32, ascending
 *   slash_out    : [n_heads][min(k_s, S)] int32, descending
 *   vscore_out / sscore_out : optional [n_heads][seq_len] fp64 score vectors
 *                  (may be NULL; used for parity tests)
 *   uncertain_out: optional [n_heads] int32 (always 0 for SPF_VS_EXACT)
 * ------------------------------------------------------------------------- */
#define SPF_VS_EXACT 0
#define SPF_VS_FAST 1
#define SPF_VS_FAST_UNCERTIFIED 2
size_t spf_vs_estimate_workspace_size(int mode, int dtype, int n_q_heads, int n_kv_heads, int n_heads, int seq_len,
                                      int head_dim, int last_q);
int spf_vs_estimate(int mode, int dtype, const void* q, const void* k, int n_q_heads, int n_kv_heads, int seq_len,
                    int head_dim, const int32_t* head_ids, int n_heads, int last_q, int k_v, int k_s,
                    int32_t* vertical_out, int32_t* slash_out, double* vscore_out, double* sscore_out,
                    int32_t* uncertain_out, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Block-Sparse online estimation.
 * Replaces estimator.py:117-143 (estimate_block_sparse) with tensor.py:43-58
 * pooling: fp64 block means rounded to fp32, fp64 pooled scores,
 * block-causal softmax rounded to fp32, per row top-min(k_b, r+1) with the
 * diagonal forced, ascending.  The result is written straight into the CSR
 * tile layout of sparse_attn.py:30-33 (tile start = block * block_size) at
 * rows head_ids[i]*n_rows + r, using tile_offsets produced by
 * spf_bs_layout_count + spf_csr_offsets.
 * ------------------------------------------------------------------------- */
size_t spf_bs_estimate_workspace_size(int n_q_heads, int n_kv_heads, int seq_len, int head_dim, int block_size);
int spf_bs_estimate(int dtype, const void* q, const void* k, int n_q_heads, int n_kv_heads, int seq_len,
                    int head_dim, const int32_t* head_ids, int n_heads, int k_b, int block_size,
                    const int64_t* tile_offsets, int32_t* tile_starts, void* workspace, size_t workspace_bytes,
                    void* stream);

/* ---------------------------------------------------------------------------
 * Index compaction.  Three steps: per-row counts (per pattern, into
 * int64 [n_q_heads*n_rows] count arrays), one scan (spf_csr_offsets), then
 * per-pattern fills.
 * ------------------------------------------------------------------------- */
size_t spf_scan_workspace_size(int64_t n);
/* offsets[0] = 0, offsets[i+1] = sum(counts[0..i]); the total is copied to
 * *total_host (synchronising `stream`) when total_host != NULL. */
int spf_csr_offsets(const int64_t* counts, int64_t n, int64_t* offsets, int64_t* total_host, void* workspace,
                    size_t workspace_bytes, void* stream);
/* Speculative sizing without a host read-back: if tile_offsets[n] > cap_tiles or
 * col_offsets[n] > cap_cols, both offset arrays are zeroed (every row empty: the
 * fills write nothing and the attention produces zero rows, so no buffer of the
 * given capacities is overrun) and *overflow = 1; totals[0..1] receive the two
 * true totals either way.  The caller reads the flag later and redoes the layer
 * with an exact size.  Stream-ordered, no host sync.  (Replaces the size
 * read-back that kernels.py:28-35's host-side flattening implies.) */
int spf_csr_guard(int64_t* tile_offsets, int64_t* col_offsets, int64_t n, int64_t cap_tiles, int64_t cap_cols,
                  int32_t* overflow, int64_t* totals, void* stream);

/* Vertical-Slash point-range merge, vs_index.py:28-95 (Alg. 4), bit-exact.
 * vertical [n_heads][n_v] ascending, slash [n_heads][n_s] descending. */
int spf_vs_layout_count(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                        int n_heads, int seq_len, int block_size, int64_t* tile_counts, int64_t* col_counts,
                        void* stream);
int spf_vs_layout_fill(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                       int n_heads, int seq_len, int block_size, const int64_t* tile_offsets,
                       const int64_t* col_offsets, int32_t* tile_starts, int32_t* col_indices, void* stream);

/* A-shape static layout, patterns.py:109-128 (sink tiles + aligned local
 * window per row, no columns). */
int spf_ashape_layout_count(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int global_tokens,
                            int local_window, int64_t* tile_counts, void* stream);
int spf_ashape_layout_fill(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int global_tokens,
                           int local_window, const int64_t* tile_offsets, int32_t* tile_starts, void* stream);

/* Block-Sparse row counts min(k_b, r+1) (estimator.py:139-142). */
int spf_bs_layout_count(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int k_b,
                        int64_t* tile_counts, void* stream);

/* Computed cells at kernel granularity (patterns.py:147-184, layout_area)
 * for every head of a CSR layout: area_out[n_heads] int64.  Used for
 * kernel_sparsity (metrics.py:43-45) and FLOP accounting. */
int spf_layout_area(int n_heads, int seq_len, int block_size, const int32_t* tile_starts,
                    const int64_t* tile_offsets, const int64_t* col_offsets, int64_t* area_out, void* stream);

/* Round/convert helper for callers holding fp32 data that want the bf16
 * production path: dst[i] = bf16_rn(src[i]). */
int spf_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPF_H_ */
