// layout.cu -- index compaction on the GPU: per-(head, query-block-row) CSR
// layouts for the three patterns, plus the CSR scan and the layout-area
// accounting.  Integer work, bit-exact with the reference.
//
//  * Vertical-Slash point-range merge (Alg. 4), vs_index.py:28-95: one warp per
//    query-block row walks the head's slash offsets (descending) as ranges and its
//    verticals (ascending) as points; count pass -> scan -> fill pass.
//  * A-shape, patterns.py:109-128: aligned sink tiles below the local window
//    start, then the aligned local window.
//  * Block-Sparse row counts min(k_b, r+1) (estimator.py:139-142); the tile
//    entries themselves are written by the BS estimator (estimate.cu).
//  * layout_area, patterns.py:147-184 (diagonal tile clipped to its lower
//    triangle, column chips rounded up to B).
#include <cub/block/block_scan.cuh>

#include "spf.h"
#include "spf_internal.h"

namespace spf {
namespace {

constexpr int kThreads = 128;
constexpr int kSmemIdx = 24 * 1024;  // ints staged in smem when the head's lists + gap list fit (96 KB)

__device__ __forceinline__ int head_of(const int32_t* head_ids, int i) { return head_ids ? head_ids[i] : i; }

// Vertical-Slash point-range merge (Alg. 4, vs_index.py:44-94), one warp per
// query-block row, bit-exact with the reference's sequential loop.  The slash
// ranges of a row have non-decreasing starts and increasing ends, so a range
// can only end the current group where it starts past the previous range's
// end (a "gap"); gap lanes of each 32-range batch are resolved in order with
// the exact coalescing rule of vs_index.py:78, all other ranges merge.  The
// vertical points consumed by a flush are classified (column if < group
// start, else absorbed) 32 at a time with ballots.
constexpr int kMergeWarps = 8;

// Warp-wide partition point: the number of leading indices of [lo, hi) for which `pred` holds
// (pred true on a prefix), in ceil(log32(hi - lo)) rounds of 32 probes instead of a binary
// search's dependent loads.
template <class Pred>
__device__ __forceinline__ int warp_partition_point(int lo, int hi, int lane, Pred pred) {
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const int c = __popc(__ballot_sync(0xffffffffu, p < hi && pred(p)));
    if (c == 0) return lo;
    const int nhi = min(hi, lo + c * step);  // probe c (if inside) failed
    lo += (c - 1) * step + 1;                // probe c - 1 held
    hi = nhi;
  }
  const int p = lo + lane;
  return lo + __popc(__ballot_sync(0xffffffffu, p < hi && pred(p)));
}

template <bool kFill>
__global__ void __launch_bounds__(kMergeWarps * 32) vs_merge_warp_kernel(
    const int32_t* __restrict__ vertical, int n_v, const int32_t* __restrict__ slash, int n_s,
    const int32_t* __restrict__ head_ids, int S, int B, int rows_per_cta, int64_t* __restrict__ tile_cnt,
    int64_t* __restrict__ col_cnt, const int64_t* __restrict__ tile_off, const int64_t* __restrict__ col_off,
    int32_t* __restrict__ tiles, int32_t* __restrict__ cols) {
  extern __shared__ int32_t s_idx[];
  __shared__ int s_ngap;
  const int i = blockIdx.y;
  const int h = head_of(head_ids, i);
  const int n_rows = (S + B - 1) / B;
  const int32_t* pts = vertical + (int64_t)i * n_v;
  const int32_t* sl = slash + (int64_t)i * n_s;
  const bool staged = n_v + 2 * n_s <= kSmemIdx;
  int32_t* gaps = s_idx + n_v + n_s;
  __shared__ int s_wgap[kMergeWarps];
  if (staged) {
#pragma unroll 4
    for (int j = threadIdx.x; j < n_v; j += blockDim.x) s_idx[j] = pts[j];
#pragma unroll 4
    for (int j = threadIdx.x; j < n_s; j += blockDim.x) s_idx[n_v + j] = sl[j];
    __syncthreads();
    pts = s_idx;
    sl = s_idx + n_v;
    // gap list: slash indices j whose range starts past the previous range's end in every
    // full row (o[j-1] - o[j] > B); only these can end a coalesced group.  Each warp lists a
    // contiguous chunk of [1, n_s) (count, block prefix, write), in ascending order.
    const int wg = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const int chunk = (((n_s - 1 + kMergeWarps - 1) / kMergeWarps) + 31) & ~31;
    const int j0 = 1 + wg * chunk, j1 = min(n_s, j0 + chunk);
    int n = 0;
    for (int b0 = j0; b0 < j1; b0 += 32) {
      const int j = b0 + ln;
      n += __popc(__ballot_sync(0xffffffffu, j < j1 && sl[j - 1] - sl[j] > B));
    }
    if (ln == 0) s_wgap[wg] = n;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wg; ++w) base += s_wgap[w];
    for (int b0 = j0; b0 < j1; b0 += 32) {
      const int j = b0 + ln;
      const bool g = j < j1 && sl[j - 1] - sl[j] > B;
      const unsigned m = __ballot_sync(0xffffffffu, g);
      if (g) gaps[base + __popc(m & ((1u << ln) - 1u))] = j;
      base += __popc(m);
    }
    if (wg == kMergeWarps - 1 && ln == 0) s_ngap = base;
    __syncthreads();
  }
  const int n_gap = staged ? s_ngap : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // ceil(x / B) for x > -B without an integer division when B is a power of two (B = 64)
  const int bsh = (B & (B - 1)) == 0 ? __ffs(B) - 1 : -1;
  auto ceil_div = [=](int x) { return bsh >= 0 && x >= 0 ? (x + B - 1) >> bsh : (x + B - 1) / B; };
  const int r_end = min(n_rows, (blockIdx.x + 1) * rows_per_cta);
  for (int r = blockIdx.x * rows_per_cta + warp; r < r_end; r += kMergeWarps) {
    const int64_t row = (int64_t)h * n_rows + r;
    const int q_start = r * B, q_end = min(q_start + B, S);
    // a row emptied by spf_csr_guard (both counts 0) receives nothing (warp-uniform)
    if (kFill && tile_off[row + 1] == tile_off[row] && col_off[row + 1] == col_off[row]) continue;
    int32_t* tout = kFill ? tiles + tile_off[row] : nullptr;
    int32_t* cout = kFill ? cols + col_off[row] : nullptr;
    int64_t nt = 0, nc = 0;
    int jv = 0;
    // flush a group [fs, fe): points < its cover end are consumed (columns if < fs), then its tiles
    auto flush = [&](int fs, int fe, bool with_tiles) {
      const int cover = with_tiles ? fs + ceil_div(fe - fs) * B : fe;
      // the next 32 points (the common case: few points per group) ...
      const int idx = jv + lane;
      const int x = idx < n_v ? pts[idx] : INT_MAX;
      const bool in = x < cover;  // ascending points: a lane prefix
      const unsigned m_in = __ballot_sync(0xffffffffu, in);
      const bool is_col = in && x < fs;
      const unsigned m_col = __ballot_sync(0xffffffffu, is_col);
      if (kFill && is_col) cout[nc + __popc(m_col & lt)] = x;
      nc += __popc(m_col);
      jv += __popc(m_in);
      if (m_in == 0xffffffffu) {
        // ... then a long run: columns = the points < fs, the rest up to cover is absorbed
        const int jc = warp_partition_point(jv, n_v, lane, [=](int p) { return pts[p] < fs; });
        if (kFill)
          for (int t = jv + lane; t < jc; t += 32) cout[nc + (t - jv)] = pts[t];
        nc += jc - jv;
        jv = warp_partition_point(jc, n_v, lane, [=](int p) { return pts[p] < cover; });
      }
      if (with_tiles) {
        const int ntile = ceil_div(fe - fs);
        if (kFill)
          for (int t = lane; t < ntile; t += 32) tout[nt + t] = fs + t * B;
        nt += ntile;
      }
    };
    // slashes are descending: skip the prefix with o >= q_end (vs_index.py:71-72)
    const int lo = warp_partition_point(0, n_s, lane, [=](int j) { return sl[j] >= q_end; });
    if (lo < n_s && staged && q_end - q_start == B) {
      // full row: visit only the gap candidates after lo (the other ranges always coalesce)
      int cs = max(0, q_start - sl[lo]);
      const int g0 = warp_partition_point(0, n_gap, lane, [=](int m) { return gaps[m] <= lo; });
      for (int base = g0; base < n_gap; base += 32) {
        const int idx = base + lane;
        const bool valid = idx < n_gap;
        const int j = valid ? gaps[idx] : 1;
        const int rs = max(0, q_start - sl[j]);
        const int pre = q_end - sl[j - 1];
        unsigned cand = __ballot_sync(0xffffffffu, valid && rs > pre);
        while (cand) {
          const int l = __ffs(cand) - 1;
          cand &= cand - 1;
          const int rs_l = __shfl_sync(0xffffffffu, rs, l);
          const int pre_l = __shfl_sync(0xffffffffu, pre, l);
          if (rs_l >= cs + ceil_div(pre_l - cs) * B) {
            flush(cs, pre_l, true);
            cs = rs_l;
          }
        }
      }
      flush(cs, q_end - sl[n_s - 1], true);
    } else if (lo < n_s) {
      int cs = max(0, q_start - sl[lo]);
      int ce = q_end - sl[lo];
      for (int base = lo + 1; base < n_s; base += 32) {
        const int idx = base + lane;
        const bool valid = idx < n_s;
        const int o = valid ? sl[idx] : 0;
        const int rs = max(0, q_start - o), re = q_end - o;
        int prev_re = __shfl_up_sync(0xffffffffu, re, 1);
        if (lane == 0) prev_re = ce;
        unsigned cand = __ballot_sync(0xffffffffu, valid && rs > prev_re);
        while (cand) {
          const int l = __ffs(cand) - 1;
          cand &= cand - 1;
          const int rs_l = __shfl_sync(0xffffffffu, rs, l);
          const int pre = __shfl_sync(0xffffffffu, prev_re, l);  // current group end
          if (rs_l >= cs + ceil_div(pre - cs) * B) {  // not coalesced (vs_index.py:78)
            flush(cs, pre, true);
            cs = rs_l;
          }
        }
        ce = __shfl_sync(0xffffffffu, re, min(31, n_s - 1 - base));
      }
      flush(cs, ce, true);
    }
    flush(q_end, q_end, false);  // trailing points < q_end become columns (vs_index.py:85-90)
    if (!kFill && lane == 0) {
      tile_cnt[row] = nt;
      col_cnt[row] = nc;
    }
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
  if (off[row + 1] - off[row] < sink_n + local_n) return;  // row emptied by spf_csr_guard
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

// rows per CTA for the warp-per-row merge: about 4 CTAs per SM over all heads, >= 8 rows
int merge_rows_per_cta(int S, int B, int n_heads) {
  const int n_rows = (S + B - 1) / B;
  const int ctas_per_head = max(1, (148 * 4) / max(1, n_heads));
  return max(kMergeWarps, (n_rows + ctas_per_head - 1) / ctas_per_head);
}
dim3 merge_grid(int S, int B, int n_heads, int rpc) {
  const int n_rows = (S + B - 1) / B;
  return dim3((unsigned)((n_rows + rpc - 1) / rpc), (unsigned)n_heads);
}

// CSR offsets: a two-level inclusive scan of the int64 row counts (tiles of kScanTile rows:
// per-tile sums, one CTA scanning the tile sums, per-tile scans plus the tile's prefix).
constexpr int kScanThreads = 1024, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
using ScanBlock = cub::BlockScan<int64_t, kScanThreads>;

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int64_t* __restrict__ counts, int64_t n,
                                                                   int64_t* __restrict__ block_sums) {
  __shared__ typename ScanBlock::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t x = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) x += base + i < n ? counts[base + i] : 0;
  int64_t incl, total;
  ScanBlock(tmp).InclusiveSum(x, incl, total);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_blocks_kernel(int64_t* __restrict__ block_sums, int64_t nb) {
  __shared__ typename ScanBlock::TempStorage tmp;
  int64_t x[kScanItems];
  const int64_t base = (int64_t)threadIdx.x * kScanItems;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) x[i] = base + i < nb ? block_sums[base + i] : 0;
  ScanBlock(tmp).ExclusiveSum(x, x);  // block_sums[b] <- prefix of the tiles before b
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < nb) block_sums[base + i] = x[i];
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const int64_t* __restrict__ counts, int64_t n,
                                                                  const int64_t* __restrict__ block_prefix,
                                                                  int64_t* __restrict__ out) {
  __shared__ typename ScanBlock::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t x[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) x[i] = base + i < n ? counts[base + i] : 0;
  ScanBlock(tmp).InclusiveSum(x, x);
  const int64_t pre = block_prefix[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) out[base + i] = x[i] + pre;
}

// spf_csr_guard: one CTA; thread 0 compares the totals with the capacities, then on overflow
// every thread helps zero the two offset arrays.
__global__ void __launch_bounds__(1024) csr_guard_kernel(int64_t* __restrict__ toff, int64_t* __restrict__ coff,
                                                         int64_t n, int64_t cap_t, int64_t cap_c,
                                                         int32_t* __restrict__ overflow, int64_t* __restrict__ totals) {
  __shared__ int over;
  if (threadIdx.x == 0) {
    const int64_t t = toff[n], c = coff[n];
    totals[0] = t;
    totals[1] = c;
    over = (t > cap_t || c > cap_c) ? 1 : 0;
    if (over) *overflow = 1;
  }
  __syncthreads();
  if (!over) return;
  for (int64_t i = threadIdx.x; i <= n; i += blockDim.x) {
    toff[i] = 0;
    coff[i] = 0;
  }
}

dim3 row_grid(int S, int B, int n_heads) { return dim3((unsigned)(((S + B - 1) / B + kThreads - 1) / kThreads), (unsigned)n_heads); }

}  // namespace
}  // namespace spf

using namespace spf;

extern "C" {

size_t spf_scan_workspace_size(int64_t n) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  return (size_t)(nb + 1) * sizeof(int64_t) + 256;
}

int spf_csr_offsets(const int64_t* counts, int64_t n, int64_t* offsets, int64_t* total_host, void* workspace,
                    size_t workspace_bytes, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if ((rc = check_cuda(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st), "csr offsets memset"))) return rc;
  if (n > 0) {
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb > kScanTile) return set_error(SPF_ERR_INVALID, "scan of %lld rows exceeds the two-level limit", (long long)n);
    if (workspace == nullptr || workspace_bytes < spf_scan_workspace_size(n))
      return set_error(SPF_ERR_INVALID, "scan workspace too small (%zu < %zu)", workspace_bytes,
                       spf_scan_workspace_size(n));
    int64_t* block_sums = reinterpret_cast<int64_t*>(workspace);
    note_launches(3);
    scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(counts, n, block_sums);
    scan_blocks_kernel<<<1, kScanThreads, 0, st>>>(block_sums, nb);
    scan_apply_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(counts, n, block_sums, offsets + 1);
    if ((rc = check_cuda(cudaGetLastError(), "csr scan"))) return rc;
  }
  if (total_host != nullptr) {
    if ((rc = check_cuda(cudaMemcpyAsync(total_host, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                         "csr total")))
      return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "csr total sync"))) return rc;
  }
  return SPF_OK;
}

int spf_csr_guard(int64_t* tile_offsets, int64_t* col_offsets, int64_t n, int64_t cap_tiles, int64_t cap_cols,
                  int32_t* overflow, int64_t* totals, void* stream) {
  if (n < 0 || cap_tiles < 0 || cap_cols < 0) return set_error(SPF_ERR_INVALID, "negative size or capacity");
  if (!tile_offsets || !col_offsets || !overflow || !totals) return set_error(SPF_ERR_INVALID, "null pointer");
  note_launches(1);
  csr_guard_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(tile_offsets, col_offsets, n, cap_tiles,
                                                                           cap_cols, overflow, totals);
  return check_cuda(cudaGetLastError(), "csr guard");
}

int spf_vs_layout_count(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                        int n_heads, int seq_len, int block_size, int64_t* tile_counts, int64_t* col_counts,
                        void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  const size_t smem = (n_v + 2 * n_s <= kSmemIdx) ? (size_t)(n_v + 2 * n_s) * 4 : 0;
  const int rpc = merge_rows_per_cta(seq_len, block_size, n_heads);
  int rc;
  if ((rc = check_cuda(cudaFuncSetAttribute(vs_merge_warp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kSmemIdx * 4), "merge smem attr")))
    return rc;
  note_launches(1);
  vs_merge_warp_kernel<false><<<merge_grid(seq_len, block_size, n_heads, rpc), kMergeWarps * 32, smem,
                                reinterpret_cast<cudaStream_t>(stream)>>>(vertical, n_v, slash, n_s, head_ids, seq_len,
                                                                          block_size, rpc, tile_counts, col_counts,
                                                                          nullptr, nullptr, nullptr, nullptr);
  return check_cuda(cudaGetLastError(), "vs_layout_count");
}

int spf_vs_layout_fill(const int32_t* vertical, int n_v, const int32_t* slash, int n_s, const int32_t* head_ids,
                       int n_heads, int seq_len, int block_size, const int64_t* tile_offsets,
                       const int64_t* col_offsets, int32_t* tile_starts, int32_t* col_indices, void* stream) {
  if (block_size < 1) return set_error(SPF_ERR_INVALID, "block_size must be >= 1");
  if (n_heads <= 0 || seq_len <= 0) return SPF_OK;
  const size_t smem = (n_v + 2 * n_s <= kSmemIdx) ? (size_t)(n_v + 2 * n_s) * 4 : 0;
  const int rpc = merge_rows_per_cta(seq_len, block_size, n_heads);
  int rc;
  if ((rc = check_cuda(cudaFuncSetAttribute(vs_merge_warp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kSmemIdx * 4), "merge smem attr")))
    return rc;
  note_launches(1);
  vs_merge_warp_kernel<true><<<merge_grid(seq_len, block_size, n_heads, rpc), kMergeWarps * 32, smem,
                               reinterpret_cast<cudaStream_t>(stream)>>>(vertical, n_v, slash, n_s, head_ids, seq_len,
                                                                         block_size, rpc, nullptr, nullptr,
                                                                         tile_offsets, col_offsets, tile_starts,
                                                                         col_indices);
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
