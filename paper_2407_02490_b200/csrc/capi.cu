// capi.cu -- extern "C" boundary of libspf.so (see include/spf.h), error
// plumbing, TMA descriptor encoding and operand preparation for the attention
// kernel.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdio.h>

#include "spf.h"
#include "spf_internal.h"
#include "spf_ptx.cuh"

namespace spf {

static thread_local char g_err[1024] = "";
static unsigned long long g_launches = 0;

void note_launches(int n) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SPF_OK;
  return set_error(SPF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

int make_tmap_bf16_3d(CUtensorMap* map, const void* base, int dim0, int dim1, int dim2, int box_rows) {
  auto fn = encode_fn();
  if (fn == nullptr) return set_error(SPF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0) return set_error(SPF_ERR_INVALID, "operand not 16-byte aligned");
  cuuint64_t dims[3] = {(cuuint64_t)dim0, (cuuint64_t)dim1, (cuuint64_t)dim2};
  cuuint64_t strides[2] = {(cuuint64_t)dim0 * 2, (cuuint64_t)dim0 * 2 * (cuuint64_t)dim1};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SPF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SPF_OK;
}

// dst_hi/dst_lo [rows][kD] <- src [rows][d] (zero padded), optional hi/lo split of fp32.
template <typename Tin, bool kSplit>
__global__ void prep_operand_kernel(const Tin* __restrict__ src, __nv_bfloat16* __restrict__ hi,
                                    __nv_bfloat16* __restrict__ lo, int64_t rows, int d, int kD) {
  const int64_t n = rows * kD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / kD;
    const int c = (int)(i - r * kD);
    float x = 0.f;
    if (c < d) x = static_cast<float>(src[r * d + c]);
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[i] = h;
    if (kSplit) lo[i] = __float2bfloat16_rn(x - __bfloat162float(h));
  }
}

template <typename Tin, bool kSplit>
static int prep_operand(const void* src, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t rows, int d, int kD,
                        cudaStream_t st) {
  const int64_t n = rows * kD;
  if (n == 0) return SPF_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
  note_launches(1);
  prep_operand_kernel<Tin, kSplit><<<(unsigned)blocks, threads, 0, st>>>(reinterpret_cast<const Tin*>(src), hi, lo,
                                                                         rows, d, kD);
  return check_cuda(cudaGetLastError(), "prep_operand");
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace spf

using namespace spf;

extern "C" {

int spf_version(void) { return 1; }

const char* spf_last_error(void) { return spf::g_err; }

unsigned long long spf_kernel_launches(void) { return __atomic_load_n(&spf::g_launches, __ATOMIC_RELAXED); }

static int padded_dim(int d) { return d <= 64 ? 64 : 128; }

}  // extern "C"

namespace {
// staged (split / padded) operand copies: 0 for bf16 inputs at head_dim 64 or 128
size_t operand_bytes(int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim) {
  const int kD = padded_dim(head_dim);
  const bool split = dtype == SPF_DTYPE_F32;
  if (!split && head_dim == kD) return 0;
  const size_t copies = split ? 2 : 1;
  const size_t per_head = (size_t)seq_len * kD * 2;
  return copies * (align256(per_head * n_q_heads) + 2 * align256(per_head * n_kv_heads));
}
}  // namespace

extern "C" {

// operand copies + the pair-routing statistics (kPairStatWords uint64 per q-head) after them
size_t spf_sparse_flash_workspace_size(int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim) {
  return operand_bytes(dtype, n_q_heads, n_kv_heads, seq_len, head_dim) +
         align256((size_t)(n_q_heads > 0 ? n_q_heads : 0) * kPairStatWords * sizeof(unsigned long long));
}

int spf_sparse_flash_rows(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                          int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                          const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                          void* out, void* workspace, size_t workspace_bytes, void* stream) {
  return spf_sparse_flash_rows_lse(dtype, q, k, v, n_q_heads, n_kv_heads, seq_len, head_dim, scale, block_size,
                                   tile_starts, tile_offsets, col_indices, col_offsets, out, nullptr, workspace,
                                   workspace_bytes, stream);
}

int spf_sparse_flash_rows_lse(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                              int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                              const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                              void* out, float* lse_out, void* workspace, size_t workspace_bytes, void* stream) {
  return spf_sparse_flash_rows_ex(dtype, q, k, v, n_q_heads, n_kv_heads, seq_len, head_dim, scale, block_size,
                                  tile_starts, tile_offsets, col_indices, col_offsets, nullptr, 0, out, lse_out,
                                  workspace, workspace_bytes, stream);
}

int spf_sparse_flash_rows_ex(int dtype, const void* q, const void* k, const void* v, int n_q_heads, int n_kv_heads,
                             int seq_len, int head_dim, float scale, int block_size, const int32_t* tile_starts,
                             const int64_t* tile_offsets, const int32_t* col_indices, const int64_t* col_offsets,
                             const int32_t* pair_heads, int n_pair_heads, void* out, float* lse_out,
                             void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype != SPF_DTYPE_BF16 && dtype != SPF_DTYPE_F32) return set_error(SPF_ERR_INVALID, "unknown dtype %d", dtype);
  if (seq_len < 1 || head_dim < 1 || n_q_heads < 1 || n_kv_heads < 1)
    return set_error(SPF_ERR_INVALID, "need seq_len, head_dim, heads >= 1");
  if (head_dim > 128) return set_error(SPF_ERR_INVALID, "head_dim %d > 128 is not supported", head_dim);
  if (n_q_heads % n_kv_heads != 0) return set_error(SPF_ERR_INVALID, "n_q_heads must be a multiple of n_kv_heads");
  if (block_size < 2) return set_error(SPF_ERR_INVALID, "block_size must be >= 2 (got %d)", block_size);
  if (!q || !k || !v || !out || !tile_offsets || !col_offsets)
    return set_error(SPF_ERR_INVALID, "null tensor pointer");
  const int kD = padded_dim(head_dim);
  const bool split = dtype == SPF_DTYPE_F32;
  AttnArgs a{};
  a.S = seq_len;
  a.Hq = n_q_heads;
  a.Hkv = n_kv_heads;
  a.B = block_size;
  a.d_out = head_dim;
  a.scale = scale;
  a.tile_starts = tile_starts;
  a.tile_offsets = tile_offsets;
  a.col_indices = col_indices;
  a.col_offsets = col_offsets;
  a.out = out;
  a.out_f32 = split;
  a.kD = kD;
  a.split = split;
  a.work_order = nullptr;
  a.n_work = 0;
  a.lse = lse_out;
  a.pair_heads = nullptr;
  a.n_pair = 0;
  if (n_pair_heads < 0 || n_pair_heads > n_q_heads || (n_pair_heads > 0 && pair_heads == nullptr))
    return set_error(SPF_ERR_INVALID, "bad pair head list (%d heads)", n_pair_heads);
  const size_t need = operand_bytes(dtype, n_q_heads, n_kv_heads, seq_len, head_dim);
  if (need == 0) {
    a.q_hi = q;
    a.k_hi = k;
    a.v_hi = v;
  } else {
    if (workspace == nullptr || workspace_bytes < need)
      return set_error(SPF_ERR_INVALID, "workspace too small (%zu < %zu bytes)", workspace_bytes, need);
    uint8_t* w = reinterpret_cast<uint8_t*>(workspace);
    const size_t per_head = (size_t)seq_len * kD * 2;
    auto take = [&](size_t bytes) {
      void* ptr = w;
      w += align256(bytes);
      return reinterpret_cast<__nv_bfloat16*>(ptr);
    };
    __nv_bfloat16* qh = take(per_head * n_q_heads);
    __nv_bfloat16* kh = take(per_head * n_kv_heads);
    __nv_bfloat16* vh = take(per_head * n_kv_heads);
    __nv_bfloat16 *ql = nullptr, *kl = nullptr, *vl = nullptr;
    if (split) {
      ql = take(per_head * n_q_heads);
      kl = take(per_head * n_kv_heads);
      vl = take(per_head * n_kv_heads);
    }
    const int64_t qrows = (int64_t)n_q_heads * seq_len, kvrows = (int64_t)n_kv_heads * seq_len;
    int rc;
    if (split) {
      if ((rc = prep_operand<float, true>(q, qh, ql, qrows, head_dim, kD, st))) return rc;
      if ((rc = prep_operand<float, true>(k, kh, kl, kvrows, head_dim, kD, st))) return rc;
      if ((rc = prep_operand<float, true>(v, vh, vl, kvrows, head_dim, kD, st))) return rc;
    } else {
      if ((rc = prep_operand<__nv_bfloat16, false>(q, qh, nullptr, qrows, head_dim, kD, st))) return rc;
      if ((rc = prep_operand<__nv_bfloat16, false>(k, kh, nullptr, kvrows, head_dim, kD, st))) return rc;
      if ((rc = prep_operand<__nv_bfloat16, false>(v, vh, nullptr, kvrows, head_dim, kD, st))) return rc;
    }
    a.q_hi = qh;
    a.k_hi = kh;
    a.v_hi = vh;
    a.q_lo = ql;
    a.k_lo = kl;
    a.v_lo = vl;
  }
  if (n_pair_heads > 0 && attn_pair_supported(a)) {
    // every listed head is routed by its measured statistics (pair_stats_kernel, in the
    // caller's workspace after the operand copies); the union kernel runs all other heads
    const size_t stats_bytes = (size_t)n_pair_heads * kPairStatWords * sizeof(unsigned long long);
    if (workspace == nullptr || workspace_bytes < need + stats_bytes)
      return set_error(SPF_ERR_INVALID, "workspace too small for the pair-routing statistics (%zu < %zu bytes)",
                       workspace_bytes, need + stats_bytes);
    unsigned long long* stats = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(workspace) + need);
    a.pair_heads = pair_heads;
    a.n_pair = n_pair_heads;
    a.pair_stats = stats;
    int rc = launch_pair_stats(a, stats, st);
    if (rc) return rc;
    if ((rc = launch_sparse_attn(a, st))) return rc;
    return launch_sparse_attn_pairs(a, st);
  }
  return launch_sparse_attn(a, st);
}

int spf_f32_to_bf16(const float* src, void* dst, int64_t n, void* stream) {
  if (n <= 0) return SPF_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
  note_launches(1);
  f32_to_bf16_kernel<<<(unsigned)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      src, reinterpret_cast<__nv_bfloat16*>(dst), n);
  return check_cuda(cudaGetLastError(), "f32_to_bf16");
}

}  // extern "C"
