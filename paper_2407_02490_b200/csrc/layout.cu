// layout.cu -- index compaction on the GPU: per-(head, query-block-row) CSR
// layouts for the three patterns, plus the CSR scan and the layout-area
// accounting.  Integer work, bit-exact with the reference.
//
//  * Vertical-Slash point-range merge (Alg. 4), vs_index.py:28-95: one thread
//    per query-block row walks the head's slash offsets (descending) as ranges
//    and its verticals (ascending) as points; count pass -> scan -> fill pass.
//  * A-shape, patterns.py:109-128: aligned sink tiles below the local window
//    start, then the aligned local window.
//  * Block-Sparse row counts min(k_b, r+1) (estimator.py:139-142); the tile
//    entries themselves are written by the BS estimator (estimate_bs.cu).
//  * layout_area, patterns.py:147-184 (diagonal tile clipped to its lower
//    triangle, column chips rounded up to B).
#include <cub/device/device_scan.cuh>

#include "spf.h"
#include "spf_internal.h"

namespace spf {
namespace {

constexpr int kThreads = 128;
constexpr int kSmemIdx = 11 * 1024;  // ints staged in smem when the head's lists fit (44 KB)

__device__ __forceinline__ int head_of(const int32_t* head_ids, int i) { return head_ids ? head_ids[i] : i; }

// One row of the VS merge.  kFill=false: counts only.
template <bool kFill>
__device__ void vs_merge_row(const int32_t* __restrict__ pts, int np, const int32_t* __restrict__ sl, int ns, int r,
                             int S, int B, int32_t* __restrict__ tiles, int32_t* __restrict__ cols, int64_t& nt,
                             int64_t& nc) {
  const int q_start = r * B;
  const int q_end = min(q_start + B, S);
  int jv = 0;
  int64_t t = 0, c = 0;
  bool have = false;
  int cs = 0, ce = 0;
  auto flush = [&](int fs, int fe) {
    const int cover = fs + ((fe - fs + B - 1) / B) * B;
    while (jv < np && pts[jv] < cover) {
      const int x = pts[jv];
      if (x < fs) {
        if (kFill) cols[c] = x;
        ++c;
      }
      ++jv;
    }
    for (int s = fs; s < fe; s += B) {
      if (kFill) tiles[t] = s;
      ++t;
    }
  };
  for (int i = 0; i < ns; ++i) {
    const int o = sl[i];
    if (o >= q_end) continue;  // diagonal left of key 0 for this row (vs_index.py:71-72)
    const int rs = max(0, q_start - o);
    const int re = q_end - o;
    if (!have) {
      cs = rs;
      ce = re;
      have = true;
    } else if (rs <= ce || rs < cs + ((ce - cs + B - 1) / B) * B) {
      ce = max(ce, re);
    } else {
      flush(cs, ce);
      cs = rs;
      ce = re;
    }
  }
  if (have) flush(cs, ce);
  for (; jv < np; ++jv) {  // trailing points right of every range (vs_index.py:85-90)
    const int x = pts[jv];
    if (x < q_end) {
      if (kFill) cols[c] = x;
      ++c;
    }
  }
  nt = t;
  nc = c;
}

template <bool kFill>
__global__ void __launch_bounds__(kThreads) vs_merge_kernel(const int32_t* __restrict__ vertical, int n_v,
                                                            const int32_t* __restrict__ slash, int n_s,
                                                            const int32_t* __restrict__ head_ids, int S, int B,
                                                            int64_t* __restrict__ tile_cnt,
                                                            int64_t* __restrict__ col_cnt,
                                                            const int64_t* __restrict__ tile_off,
                                                            const int64_t* __restrict__ col_off,
                                                            int32_t* __restrict__ tiles, int32_t* __restrict__ cols) {
  extern __shared__ int32_t s_idx[];
  const int i = blockIdx.y;
  const int h = head_of(head_ids, i);
  const int n_rows = (S + B - 1) / B;
  const int32_t* pts = vertical + (int64_t)i * n_v;
  const int32_t* sl = slash + (int64_t)i * n_s;
  if (n_v + n_s <= kSmemIdx) {
    for (int j = threadIdx.x; j < n_v; j += blockDim.x) s_idx[j] = pts[j];
    for (int j = threadIdx.x; j < n_s; j += blockDim.x) s_idx[n_v + j] = sl[j];
    __syncthreads();
    pts = s_idx;
    sl = s_idx + n_v;
  }
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t row = (int64_t)h * n_rows + r;
  int64_t nt, nc;
  if (kFill) {
    vs_merge_row<true>(pts, n_v, sl, n_s, r, S, B, tiles + tile_off[row], cols + col_off[row], nt, nc);
  } else {
    vs_merge_row<false>(pts, n_v, sl, n_s, r, S, B, nullptr, nullptr, nt, nc);
    tile_cnt[row] = nt;
    col_cnt[row] = nc;
  }
}

__device__ __forceinline__ void ashape_row(int r, int S, int B, int g, int w, int& sink_n, int& local_start,
                                           int& local_n) {
  const int q_start = r * B;
  const int q_end = min(q_start + B, S);
  const int sink_end = min(g, q_end);
  local_start = max(0, q_start - w) / B * B;
  local_n = (q_end - local_start + B - 1) / B;
  // sink starts 0, B, ... < sink_end that are not already local starts (< local_start)
  const int lim = min(sink_end, local_start);
  sink_n = lim > 0 ? (lim + B - 1) / B : 0;
}

__global__ void ashape_kernel(const int32_t* __restrict__ head_ids, int S, int B, int g, int w,
                              int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
                              int32_t* __restrict__ tiles) {
  const int h = head_of(head_ids, blockIdx.y);
  const int n_rows = (S + B - 1) / B;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t row = (int64_t)h * n_rows + r;
  int sink_n, local_start, local_n;
  ashape_row(r, S, B, g, w, sink_n, local_start, local_n);
  if (tiles == nullptr) {
    cnt[row] = sink_n + local_n;
    return;
  }
  int32_t* out = tiles + off[row];
  for (int j = 0; j < sink_n; ++j) out[j] = j * B;
  for (int j = 0; j < local_n; ++j) out[sink_n + j] = local_start + j * B;
}

__global__ void bs_count_kernel(const int32_t* __restrict__ head_ids, int S, int B, int k_b,
                                int64_t* __restrict__ cnt) {
  const int h = head_of(head_ids, blockIdx.y);
  const int n_rows = (S + B - 1) / B;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  cnt[(int64_t)h * n_rows + r] = min(k_b, r + 1);
}

// patterns.py:166-184
__device__ __forceinline__ int64_t clipped_tile_cells(int64_t s, int64_t b, int64_t q_start, int64_t q_end,
                                                      int64_t S) {
  const int64_t lo = max(s, (int64_t)0), hi = min(s + b, S);
  if (hi <= lo) return 0;
  const int64_t full_from = max(q_start, hi - 1);
  int64_t cells = max((int64_t)0, q_end - full_from) * (hi - lo);
  const int64_t ramp_lo = max(q_start, lo), ramp_hi = min(q_end, hi - 1);
  if (ramp_hi > ramp_lo) {
    const int64_t n = ramp_hi - ramp_lo;
    cells += n * ((ramp_lo + 1 - lo) + (ramp_hi - lo)) / 2;
  }
  return cells;
}

__global__ void area_kernel(int S, int B, const int32_t* __restrict__ tiles, const int64_t* __restrict__ tile_off,
                            const int64_t* __restrict__ col_off, unsigned long long* __restrict__ area) {
  const int h = blockIdx.y;
  const int n_rows = (S + B - 1) / B;
  int64_t acc = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    const int64_t row = (int64_t)h * n_rows + r;
    const int64_t q_start = (int64_t)r * B, q_end = min(q_start + B, (int64_t)S);
    for (int64_t t = tile_off[row]; t < tile_off[row + 1]; ++t) acc += clipped_tile_cells(tiles[t], B, q_start, q_end, S);
    const int64_t nc = col_off[row + 1] - col_off[row];
    acc += ((nc + B - 1) / B) * B * (q_end - q_start);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(area + h, (unsigned long long)acc);
}

dim3 row_grid(int S, int B, int n_heads) { return dim3((unsigned)(((S + B - 1) / B + kThreads - 1) / kThreads), (unsigned)n_heads); }

}  // namespace
}  // namespace spf

using namespace spf;

extern "C" {

size_t spf_scan_workspace_size(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
  return bytes + 256;
}

int spf_csr_offsets(const int64_t* counts, int64_t n, int64_t* offsets, int64_t* total_host, void* workspace,
                    size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if ((rc = check_cuda(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st), "csr offsets memset"))) return rc;
  if (n > 0) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, counts, offsets + 1, n);
    if (workspace == nullptr || workspace_bytes < bytes)
      return set_error(SPF_ERR_INVALID, "scan workspace too small (%zu < %zu)", workspace_bytes, bytes);
    note_launches(2);
    if ((rc = check_cuda(cub::DeviceScan::InclusiveSum(workspace, bytes, counts, offsets + 1, n, st), "csr scan")))
      return rc;
  }
  if (total_host != nullptr) {
    if ((rc = check_cuda(cudaMemcpyAsync(total_host, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                         "csr total")))
      return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "csr total sync"))) return rc;
  }
  return SPF_OK;
}

int spf_vs_layout_count(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                        int n_heads, int seq_len, int block_size, int64_t* tile_counts, int64_t* col_counts,
                        void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  const size_t smem = (n_v + n_s <= kSmemIdx) ? (size_t)(n_v + n_s) * 4 : 0;
  note_launches(1);
  vs_merge_kernel<false><<<row_grid(seq_len, block_size, n_heads), kThreads, smem,
                           reinterpret_cast<cudaStream_t>(stream)>>>(vertical, n_v, slash, n_s, head_ids, seq_len,
                                                                     block_size, tile_counts, col_counts, nullptr,
                                                                     nullptr, nullptr, nullptr);
  return check_cuda(cudaGetLastError(), "vs_layout_count");
}

int spf_vs_layout_fill(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                       int n_heads, int seq_len, int block_size, const int64_t* tile_offsets,
                       const int64_t* col_offsets, int32_t* tile_starts, int32_t* col_indices, void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  const size_t smem = (n_v + n_s <= kSmemIdx) ? (size_t)(n_v + n_s) * 4 : 0;
  note_launches(1);
  vs_merge_kernel<true><<<row_grid(seq_len, block_size, n_heads), kThreads, smem,
                          reinterpret_cast<cudaStream_t>(stream)>>>(vertical, n_v, slash, n_s, head_ids, seq_len,
                                                                    block_size, nullptr, nullptr, tile_offsets,
                                                                    col_offsets, tile_starts, col_indices);
  return check_cuda(cudaGetLastError(), "vs_layout_fill");
}

int spf_ashape_layout_count(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int global_tokens,
                            int local_window, int64_t* tile_counts, void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (global_tokens < 1 || local_window < 1) return set_error(SPF_ERR_INVALID, "A-shape counts must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  note_launches(1);
  ashape_kernel<<<row_grid(seq_len, block_size, n_heads), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      head_ids, seq_len, block_size, global_tokens, local_window, tile_counts, nullptr, nullptr);
  return check_cuda(cudaGetLastError(), "ashape_layout_count");
}

int spf_ashape_layout_fill(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int global_tokens,
                           int local_window, const int64_t* tile_offsets, int32_t* tile_starts, void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  note_launches(1);
  ashape_kernel<<<row_grid(seq_len, block_size, n_heads), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      head_ids, seq_len, block_size, global_tokens, local_window, nullptr, tile_offsets, tile_starts);
  return check_cuda(cudaGetLastError(), "ashape_layout_fill");
}

int spf_bs_layout_count(const int32_t* head_ids, int n_heads, int seq_len, int block_size, int k_b,
                        int64_t* tile_counts, void* stream) {
  if (block_size < 1 || k_b < 1) return set_error(SPF_ERR_INVALID, "Block-Sparse counts must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  note_launches(1);
  bs_count_kernel<<<row_grid(seq_len, block_size, n_heads), kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      head_ids, seq_len, block_size, k_b, tile_counts);
  return check_cuda(cudaGetLastError(), "bs_layout_count");
}

int spf_layout_area(int n_heads, int seq_len, int block_size, const int32_t* tile_starts,
                    const int64_t* tile_offsets, const int64_t* col_offsets, int64_t* area_out, void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if ((rc = check_cuda(cudaMemsetAsync(area_out, 0, sizeof(int64_t) * n_heads, st), "area memset"))) return rc;
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  const int n_rows = (seq_len + block_size - 1) / block_size;
  const unsigned gx = (unsigned)min(64, (n_rows + 255) / 256);
  note_launches(1);
  area_kernel<<<dim3(gx, (unsigned)n_heads), 256, 0, st>>>(seq_len, block_size, tile_starts, tile_offsets,
                                                           col_offsets, reinterpret_cast<unsigned long long*>(area_out));
  return check_cuda(cudaGetLastError(), "layout_area");
}

}  // extern "C"
