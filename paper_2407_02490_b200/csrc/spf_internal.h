// spf_internal.h -- host-side declarations shared by the CUDA translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace spf {

// Sets the thread-local last-error string and returns the status code.
int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);

// Counts kernel launches issued by this library (spf_kernel_launches()).
void note_launches(int n);

// Encodes a 3-D [dim2][dim1][dim0] bf16 tensor map with a (64 x rows x 1) box
// and 128-byte swizzle; used for every Q/K/V operand.
int make_tmap_bf16_3d(CUtensorMap* map, const void* base, int dim0, int dim1, int dim2, int box_rows);

struct AttnArgs {
  int S, Hq, Hkv, B, d_out;
  float scale;
  const int32_t* tile_starts;
  const int64_t* tile_offsets;
  const int32_t* col_indices;
  const int64_t* col_offsets;
  // bf16 operands, padded to kD (64 or 128); *_lo are the split residuals (fp32 I/O path)
  const void *q_hi, *k_hi, *v_hi, *q_lo, *k_lo, *v_lo;
  void* out;
  bool out_f32;
  int kD;
  bool split;
  const int32_t* work_order;  // optional: CTA -> work-item list (nullptr = all items, heavy rows first)
  int n_work;                 // number of entries in work_order
  float* lse;                 // optional [Hq][S]: natural-log sum of exp(scale * q.k) over the row's cells
  const int32_t* pair_heads;  // optional device list of q-heads run by the paired-box kernel (attn_bs.cu)
  int n_pair;
  // [n_pair][kPairStatWords]: per listed head, union steps, paired steps and residual columns
  // summed over its CTAs (pair_stats_kernel); every listed head is routed by them.
  const unsigned long long* pair_stats;
};

constexpr int kPairStatWords = 3;

// The paired-box kernel pays ~1.6x a union step per step (N128 QK + K128 PV): it wins when the
// CTAs' union steps exceed 1.6x their paired steps (measured: Block-Sparse on i.i.d. inputs,
// union ~2x paired, pair 0.87x the union kernel's time; on locality inputs, union ~1.01x paired,
// pair 1.49x).  It has no column-chip path, so a head with residual columns never goes there.
// The union kernel runs every head the paired-box kernel does not (its CTAs of the others
// exit at once), so coverage never depends on the list: duplicate or out-of-range ids
// cannot leave a head unwritten.
__host__ __device__ inline bool pair_preferred(const unsigned long long* stats, int i) {
  const unsigned long long* s = stats + kPairStatWords * i;
  return s[2] == 0 && 5ull * s[0] > 8ull * s[1];
}

int launch_sparse_attn(const AttnArgs& a, cudaStream_t stream);
// Paired-box kernel for heads whose row blocks rarely share tiles (attn_bs.cu).
bool attn_pair_supported(const AttnArgs& a);
int launch_sparse_attn_pairs(const AttnArgs& a, cudaStream_t stream);
int launch_pair_stats(const AttnArgs& a, unsigned long long* stats, cudaStream_t stream);

// fp64 Vertical-Slash estimation (estimate_vs_exact.cu): all heads (gate == nullptr) or the
// flagged ones; tile_max / row_mc / row_marg (from the tensor-core pass, last_q 64: its scores,
// row maxima and per-row score-error margins) enable exact item skipping.
size_t vs_exact_workspace_size(int n_heads, int seq_len, int last_q);
int vs_exact_run(int dtype, const void* q, const void* k, int Hq, int Hkv, int S, int d, const int32_t* head_ids,
                 int n_heads, int L, int k_v, int k_s, int32_t* vout, int32_t* sout, double* vscore, double* sscore,
                 const int32_t* gate, const float* tile_max, const float* row_mc, const float* row_marg,
                 void* workspace, cudaStream_t st);

// Tensor-core Vertical-Slash estimation (estimate_vs_tc.cu), mode SPF_VS_FAST.
bool vs_fast_supported(int dtype, int head_dim, int seq_len, int last_q);
size_t vs_fast_workspace_size(int n_q_heads, int n_kv_heads, int n_heads, int seq_len);
int vs_estimate_fast(const void* q, const void* k, int Hq, int Hkv, int S, int d, const int32_t* head_ids,
                     int n_heads, int k_v, int k_s, int32_t* vout, int32_t* sout, double* vscore, double* sscore,
                     int32_t* uncertain, bool uncertified, void* workspace, cudaStream_t st);

}  // namespace spf
