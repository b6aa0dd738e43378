// estimate_vs_exact.cu -- Vertical-Slash estimation with fp64 scores (mode
// SPF_VS_EXACT, and the in-stream fallback of SPF_VS_FAST for the heads whose
// tensor-core selection could not be certified).
//
// Follows estimator.py:82-114 with the rounding points of tensor.py:61-78:
//   s   = scale * (q_tail[i] . k[j])            fp64 FMA chain over d
//   m_i = max_j s, l_i = sum_j exp(s - m_i)     fp64 (deterministic order)
//   p   = fp32(exp(s - m_i) / l_i)              the reference's fp32 rounding
//   vertical[j] = sum_i p (i ascending, fp64)   est.sum(axis=0)
//   slash[o]    = sum_i p[i][abs_i - o] (fp64)  np.bincount over the row-major order
//
// Streaming design (no [rows x S] score matrix): the key axis is cut into
// items of KB keys (KB = 64, or the multiple of 64 >= last_q - 1 so a
// diagonal spans at most two items).  Pass A computes per-(row, item) partial
// (max, sum exp); a combine fixes (m_i, l_i); pass B recomputes the scores,
// forms p, sums columns in-CTA in row order and diagonals in-CTA, and adds
// each diagonal's (at most two) item partials with fp64 atomics into a
// zeroed vector -- two-term sums are order-free, so the result is
// deterministic.
//
// Fallback mode: `gate` restricts the work to flagged heads (device-side, no
// host sync) and `tile_max` (per row and 128-key tile, from the tensor-core
// pass) lets an item be skipped when every score in it is below the row max
// by more than 151 + row_marg in log2 units: row_marg is twice the rigorous bound
// on the tensor-core score error (estimate_vs_tc.cu, vs_tc_combine_kernel), so
// the exact scores are > 150 below the exact row max, such p are < 2^-150 and
// round to exactly 0 in fp32 (l_i >= 1): the skip is exact, not an approximation.
#include <algorithm>
#include <cuda_bf16.h>

#include "spf.h"
#include "spf_internal.h"
#include "cluster_topk.cuh"

namespace spf {
namespace {

constexpr int kThreads = 256;
constexpr int kRowT = 64;    // rows per register tile
constexpr int kKeyT = 64;    // keys per register tile
constexpr int kDc = 32;      // d chunk staged in shared memory
constexpr int kLd = 68;      // padded leading dimension (doubles) of the staged chunks
constexpr int kMaxL = 2048;  // last_q supported by this path

struct ExArgs {
  int S, d, L, KB, n_kblk, n_heads, hpk;
  const int32_t* head_ids;
  const int32_t* gate;     // nullable
  const float* tile_max;   // nullable: [n_heads][ceil(S/128)][64] raw fp32 scores
  const float* row_mc;     // [n_heads][64]: fp32(max raw score * c)
  const float* row_marg;   // [n_heads][64]: 2 x score-error bound of the tensor-core scores (log2 units)
  float c;                 // scale * log2(e)
  double scale;
  double2* stats;          // [n_heads][L][n_kblk]
  double2* row_ml;         // [n_heads][L]
  double* vscore;          // [n_heads][S]
  double* sscore;          // [n_heads][S]
  // fallback (tile_max given, L = KB = 64): per flagged head the significant 64-key items,
  // list[h * n_kblk + i] = kb for i < head_count[h] (any order)
  int32_t* list;
  int32_t* head_count;     // [n_heads]
  uint8_t* sig;            // [n_heads][n_kblk]: item significant (prep), compacted in kb order by the list kernel
  double* cache;           // pass A's scaled scores of the listed items, [virtual item][64][64]
  int cache_items;         // items the cache holds (virtual items >= this are rescored in pass B)
};

constexpr int kCacheItems = 8192;  // 256 MB: the significant items of 32 G-local heads at 128K-1M

template <typename T>
__device__ __forceinline__ double ld_f64(const T* p) {
  return static_cast<double>(static_cast<float>(*p));
}
template <>
__device__ __forceinline__ double ld_f64<__nv_bfloat16>(const __nv_bfloat16* p) {
  return static_cast<double>(__bfloat162float(*p));
}

struct ExSmem {
  double At[kDc * kLd];
  double Bt[kDc * kLd];
  float P[kRowT][kKeyT + 1];
};

// acc[a][b] = q_tail row (r0 + 4 tr + a) . key (k0 + tk + 16 b), fp64, d ascending.
// Keys are strided by 16 across a thread's four columns so one warp-wide LDS.64
// of the key chunk reads 16 consecutive doubles (one wavefront, no conflicts);
// the row operand is a 2-address broadcast.
template <typename T>
__device__ void score_tile(ExSmem& sm, const T* qh, const T* kh, int r0, int n_rows_valid, int k0, int S, int d,
                           double (&acc)[4][4]) {
  const int tid = threadIdx.x, tr = tid >> 4, tk = tid & 15;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  const bool vec = (d % 8) == 0 && sizeof(T) == 2;  // 16-byte loads of 8 bf16
  for (int c0 = 0; c0 < d; c0 += kDc) {
    __syncthreads();
    if (vec) {
      // one 16-byte load per thread per operand: row r = tid / 4, dims c0 + 8 (tid % 4) .. + 7
      const int r = tid >> 2, cc = (tid & 3) * 8;
      if (cc < kDc) {
        int4 qa = make_int4(0, 0, 0, 0), kbv = make_int4(0, 0, 0, 0);
        if (c0 + cc < d && r < n_rows_valid) qa = *reinterpret_cast<const int4*>(qh + (int64_t)(r0 + r) * d + c0 + cc);
        if (c0 + cc < d && k0 + r < S) kbv = *reinterpret_cast<const int4*>(kh + (int64_t)(k0 + r) * d + c0 + cc);
        const __nv_bfloat16* qv = reinterpret_cast<const __nv_bfloat16*>(&qa);
        const __nv_bfloat16* kv = reinterpret_cast<const __nv_bfloat16*>(&kbv);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sm.At[(cc + u) * kLd + r] = (double)__bfloat162float(qv[u]);
          sm.Bt[(cc + u) * kLd + r] = (double)__bfloat162float(kv[u]);
        }
      }
    } else {
      for (int e = tid; e < kRowT * kDc; e += kThreads) {
        const int r = e / kDc, c = e % kDc;
        const bool okc = c0 + c < d;
        sm.At[c * kLd + r] = (okc && r < n_rows_valid) ? ld_f64(qh + (int64_t)(r0 + r) * d + c0 + c) : 0.0;
        sm.Bt[c * kLd + r] = (okc && k0 + r < S) ? ld_f64(kh + (int64_t)(k0 + r) * d + c0 + c) : 0.0;
      }
    }
    __syncthreads();
    const int cn = min(kDc, d - c0);
#pragma unroll 4
    for (int c = 0; c < cn; ++c) {
      const double2 qa = *reinterpret_cast<const double2*>(sm.At + c * kLd + 4 * tr);
      const double2 qb = *reinterpret_cast<const double2*>(sm.At + c * kLd + 4 * tr + 2);
      const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
      double kv[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) kv[b] = sm.Bt[c * kLd + tk + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(qv[a], kv[b], acc[a][b]);
    }
  }
}

// Is any score of item (h, kb) within 151 + margin (log2 units) of its row max?  Exact-skip test.
__device__ bool item_significant(const ExArgs& a, int h, int k0) {
  if (a.tile_max == nullptr) return true;
  const int n_t = (a.S + 127) / 128;
  const int t = k0 / 128;
  int sig = 0;
  if (threadIdx.x < 64) {
    const float tm = a.tile_max[((int64_t)h * n_t + t) * 64 + threadIdx.x];
    const float mc = a.row_mc[(int64_t)h * 64 + threadIdx.x];
    const float mg = a.row_marg[(int64_t)h * 64 + threadIdx.x];
    sig = !(tm * a.c - mc < -151.f - mg);  // NaN-safe: anything unexpected counts as significant
  }
  return __syncthreads_or(sig) != 0;
}

// Fallback preparation (tile_max given): one warp per (flagged head, 64-key item).
// Zeroes the item's slash entries, writes the vertical scores of items whose
// probabilities are all exactly 0 in fp32 and flags the others.
__global__ void vs_exact_prep_kernel(const ExArgs a) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)a.n_heads * a.n_kblk) return;
  const int h = (int)(w / a.n_kblk), kb = (int)(w % a.n_kblk);
  if (a.gate != nullptr && a.gate[h] == 0) return;
  const int S = a.S, k0 = kb * a.KB;
  const int n_t = (S + 127) / 128, t = k0 / 128;
  int sig = 0;
  for (int i = lane; i < 64; i += 32) {
    const float tm = a.tile_max[((int64_t)h * n_t + t) * 64 + i];
    const float mc = a.row_mc[(int64_t)h * 64 + i];
    const float mg = a.row_marg[(int64_t)h * 64 + i];
    sig |= !(tm * a.c - mc < -151.f - mg);
  }
  sig = __any_sync(0xffffffffu, sig);
  for (int o = k0 + lane; o < min(k0 + a.KB, S); o += 32) a.sscore[(int64_t)h * S + o] = 0.0;
  if (lane == 0) a.sig[w] = (uint8_t)(sig ? 1 : 0);
  if (!sig)
    for (int j = k0 + lane; j < min(k0 + a.KB, S); j += 32) a.vscore[(int64_t)h * S + j] = 0.0;
}

// Per flagged head: the significant items in ascending kb order (a block scan of the
// flags), so pass A's per-item statistics are combined in a fixed order.
constexpr int kListThreads = 1024;
__global__ void __launch_bounds__(kListThreads) vs_exact_list_kernel(const ExArgs a) {
  using Scan = cub::BlockScan<int, kListThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int h = blockIdx.x;
  if (a.gate != nullptr && a.gate[h] == 0) return;
  int base = 0;
  for (int c0 = 0; c0 < a.n_kblk; c0 += kListThreads) {
    const int kb = c0 + threadIdx.x;
    const int f = kb < a.n_kblk ? a.sig[(int64_t)h * a.n_kblk + kb] : 0;
    int pos, tot;
    Scan(tmp).ExclusiveSum(f, pos, tot);
    if (f) a.list[(int64_t)h * a.n_kblk + base + pos] = kb;
    base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.head_count[h] = base;
}

template <typename T, int kPass>
__global__ void __launch_bounds__(kThreads, 2) vs_exact_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                            const ExArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  ExSmem& sm = *reinterpret_cast<ExSmem*>(smraw);
  double* colsum = reinterpret_cast<double*>(smraw + sizeof(ExSmem));   // [KB]
  double* diagsum = colsum + a.KB;                                      // [KB + L - 1]
  const int tid = threadIdx.x, tr = tid >> 4, tk = tid & 15;
  const int S = a.S, L = a.L, KB = a.KB, d = a.d;
  const int n_rt = (L + kRowT - 1) / kRowT;
  // items (head, key block) interleaved head-fastest, so the significant blocks of every
  // head (often a narrow band of keys) spread over all CTAs
  const int64_t n_items = (int64_t)a.n_heads * a.n_kblk;
  for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const int h = (int)(w % a.n_heads);
    const int kb = (int)(w / a.n_heads);
    if (a.gate != nullptr && a.gate[h] == 0) continue;
    const int qh_id = a.head_ids ? a.head_ids[h] : h;
    const T* qh = q + ((int64_t)qh_id * S + (S - L)) * d;
    const T* kh = k + (int64_t)(qh_id / a.hpk) * S * d;
    {
      const int k0 = kb * KB;
      if (kPass == 1) {  // zero this item's share of the slash vector (pass 2 accumulates into it)
        for (int o = k0 + tid; o < min(k0 + KB, S); o += kThreads) a.sscore[(int64_t)h * S + o] = 0.0;
      }
      const bool sig = item_significant(a, h, k0);
      if (!sig) {
        if (kPass == 1) {
          for (int i = tid; i < L; i += kThreads)
            a.stats[((int64_t)h * L + i) * a.n_kblk + kb] = make_double2(-INFINITY, 0.0);
        } else {
          for (int j = k0 + tid; j < min(k0 + KB, S); j += kThreads) a.vscore[(int64_t)h * S + j] = 0.0;
        }
        continue;
      }
      if (kPass == 2) {
        for (int x = tid; x < KB + L - 1; x += kThreads) diagsum[x] = 0.0;
        for (int x = tid; x < KB; x += kThreads) colsum[x] = 0.0;
      }
      for (int rt = 0; rt < n_rt; ++rt) {
        const int r0 = rt * kRowT;
        const int nrv = min(kRowT, L - r0);
        double m_run[4], l_run[4];
        double mrow[4], ilrow[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          m_run[x] = -INFINITY;
          l_run[x] = 0.0;
          const int i = r0 + 4 * tr + x;
          if (kPass == 2 && i < L) {
            const double2 ml = a.row_ml[(int64_t)h * L + i];
            mrow[x] = ml.x;
            ilrow[x] = ml.y;
          } else {
            mrow[x] = 0.0;
            ilrow[x] = 0.0;
          }
        }
        for (int sb = 0; sb < KB / kKeyT; ++sb) {
          const int kk0 = k0 + sb * kKeyT;
          double acc[4][4];
          score_tile(sm, qh, kh, r0, nrv, kk0, S, d, acc);
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int i = r0 + 4 * tr + x;
            const int abs_i = S - L + i;
            double s[4];
            double mx = -INFINITY;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              const int j = kk0 + tk + 16 * y;
              const bool valid = i < L && j <= abs_i;  // abs_i < S
              s[y] = valid ? a.scale * acc[x][y] : -INFINITY;
              mx = fmax(mx, s[y]);
            }
            if (kPass == 1) {
#pragma unroll
              for (int o = 1; o < 16; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              double l = 0.0;
              if (mx != -INFINITY) {
#pragma unroll
                for (int y = 0; y < 4; ++y)
                  if (s[y] != -INFINITY) l += exp(s[y] - mx);
              }
#pragma unroll
              for (int o = 1; o < 16; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
              if (mx != -INFINITY) {
                if (mx > m_run[x]) {
                  l_run[x] = (m_run[x] == -INFINITY ? 0.0 : l_run[x] * exp(m_run[x] - mx)) + l;
                  m_run[x] = mx;
                } else {
                  l_run[x] += l * exp(mx - m_run[x]);
                }
              }
            } else {
#pragma unroll
              for (int y = 0; y < 4; ++y) {
                const float p = (s[y] == -INFINITY) ? 0.f : __double2float_rn(exp(s[y] - mrow[x]) / ilrow[x]);
                sm.P[4 * tr + x][tk + 16 * y] = p;
              }
            }
          }
          if (kPass == 2) {
            __syncthreads();
            // columns: rows ascending (est.sum(axis=0) order)
            if (tid < kKeyT) {
              double cs = colsum[sb * kKeyT + tid];
              for (int ii = 0; ii < nrv; ++ii) cs += (double)sm.P[ii][tid];
              colsum[sb * kKeyT + tid] = cs;
            }
            // diagonals of this (row tile, key tile): local key jj - row ii = cl in [-63, 63]
            for (int cl = tid - 63; cl <= 63; cl += kThreads) {
              const int ii0 = max(0, -cl), ii1 = min(nrv, kKeyT - cl);
              if (ii0 >= ii1) continue;
              const int x = sb * kKeyT - r0 + cl + (L - 1);  // diagsum index of (key - k0) - row
              double ds = diagsum[x];
              for (int ii = ii0; ii < ii1; ++ii) ds += (double)sm.P[ii][ii + cl];
              diagsum[x] = ds;
            }
            __syncthreads();
          }
        }
        if (kPass == 1 && tk == 0) {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int i = r0 + 4 * tr + x;
            if (i < L) a.stats[((int64_t)h * L + i) * a.n_kblk + kb] = make_double2(m_run[x], l_run[x]);
          }
        }
      }
      if (kPass == 2) {
        __syncthreads();
        for (int x = tid; x < KB; x += kThreads)
          if (k0 + x < S) a.vscore[(int64_t)h * S + k0 + x] = colsum[x];
        // diagonal (key - k0) - row = x - (L - 1); offset o = (S - L + row) - key
        for (int x = tid; x < KB + L - 1; x += kThreads) {
          const int o = S - L - k0 - (x - (L - 1));
          if (o >= 0 && o < S && diagsum[x] != 0.0) atomicAdd(a.sscore + (int64_t)h * S + o, diagsum[x]);
        }
        __syncthreads();
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Fallback fp64 scoring on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64: 37 TF/s on this
// B200 vs 30-34 for DFMA, benchmarks/mb_dmma.cu), for the flagged heads' listed items
// (L = KB = 64, bf16 inputs, head_dim 64 / 128).  The work is the concatenation of the
// heads' item lists ("virtual items"); CTA b takes a contiguous range of it, so the 64 tail
// rows of Q (fp64 in shared memory) are staged once per head, and the next item's K rows
// are fetched into registers while the current item is scored.  Per item the 64 x 64 fp64
// scores are exact products of bf16 values summed in fp64 (DMMA, fixed order: bit-identical
// across runs).  Pass A caches the scaled scores and writes per-(row, item) (max, sum exp);
// pass B reads them back (or rescores items past the cache) and forms p, column and
// diagonal sums exactly as vs_exact_kernel does.
constexpr int kFbThreads = 256;

template <int kD>
struct FbSmem {
  // Q and K rows staged as bf16 (converted to fp64 at fragment load): 17 KB each, so two
  // CTAs fit per SM.  The 8-element pad puts the 8 rows a fragment load touches on
  // distinct banks.
  static constexpr int kLd = kD + 8;                // bf16 per staged row
  static constexpr int kOffQ = 0;                   // bf16 [64][kLd]
  static constexpr int kOffK = kOffQ + 64 * kLd * 2;
  static constexpr int kOffP = kOffK + 64 * kLd * 2;  // float [64][65] (pass B)
  static constexpr int kOffCol = kOffP + 64 * 65 * 4;  // double [64]
  static constexpr int kOffDiag = kOffCol + 64 * 8;    // double [127]
  static constexpr int kOffRed = kOffDiag + 128 * 8;   // double [2][64] (cross-warp row reductions)
  static constexpr int kOffOff = kOffRed + 2 * 64 * 8;  // int [kMaxFbHeads + 1]
  static constexpr int kBytes = kOffOff + (1024 + 1) * 4;
};
constexpr int kMaxFbHeads = 1024;

__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// 64 rows x kD bf16 -> fp64 rows of the staged matrix (rows past `valid` are zero)
template <int kD>
__device__ __forceinline__ void fb_fetch(const __nv_bfloat16* src, int valid, int4 (&r)[kD / 32]) {
  // 64 rows x kD bf16 = 64 * kD / 8 16-byte chunks; thread t takes chunks t, t + 256, ...
#pragma unroll
  for (int u = 0; u < kD / 32; ++u) {
    const int ch = threadIdx.x + u * kFbThreads;
    const int row = ch / (kD / 8), c8 = ch % (kD / 8);
    r[u] = row < valid ? *reinterpret_cast<const int4*>(src + (int64_t)row * kD + c8 * 8) : make_int4(0, 0, 0, 0);
  }
}
template <int kD>
__device__ __forceinline__ void fb_store(__nv_bfloat16* dst, const int4 (&r)[kD / 32]) {
#pragma unroll
  for (int u = 0; u < kD / 32; ++u) {
    const int ch = threadIdx.x + u * kFbThreads;
    const int row = ch / (kD / 8), c8 = ch % (kD / 8);
    *reinterpret_cast<int4*>(dst + row * FbSmem<kD>::kLd + c8 * 8) = r[u];
  }
}


// acc[mi][ni] = 8x8 tiles of Q K^T: rows m0 + 8 mi (+ lane / 4), keys n0 + 8 ni (+ 2 (lane % 4) + {0, 1}).
// The k4 steps of the DMMA walk each 16-wide slice of d as k = 16 kk + 4 (lane % 4) + j for
// j = 0..3 (the same map for both operands, so every k of the slice is summed once): each
// lane's four values of a slice are contiguous, one 8-byte load per fragment per 4 DMMAs.
template <int kD>
__device__ __forceinline__ void fb_scores(const __nv_bfloat16* Qs, const __nv_bfloat16* Ks, int m0, int n0,
                                          double (&acc)[2][4][2]) {
  constexpr int kLd = FbSmem<kD>::kLd;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const __nv_bfloat16* qa = Qs + (m0 + (lane >> 2)) * kLd + 4 * (lane & 3);
  const __nv_bfloat16* kb = Ks + (n0 + (lane >> 2)) * kLd + 4 * (lane & 3);
#pragma unroll 2
  for (int kk = 0; kk < kD / 16; ++kk) {
    uint2 ar[2], br[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) ar[mi] = *reinterpret_cast<const uint2*>(qa + mi * 8 * kLd + 16 * kk);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) br[ni] = *reinterpret_cast<const uint2*>(kb + ni * 8 * kLd + 16 * kk);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a[2], b[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const uint32_t w = j < 2 ? ar[mi].x : ar[mi].y;
        a[mi] = (double)__uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const uint32_t w = j < 2 ? br[ni].x : br[ni].y;
        b[ni] = (double)__uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_f64(acc[mi][ni], a[mi], b[ni]);
    }
  }
}

template <int kD, int kPass>
__global__ void __launch_bounds__(kFbThreads, 2) vs_fb_kernel(const __nv_bfloat16* __restrict__ q,
                                                              const __nv_bfloat16* __restrict__ k, const ExArgs a) {
  using SM = FbSmem<kD>;
  extern __shared__ __align__(16) uint8_t smraw[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smraw + SM::kOffQ);
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smraw + SM::kOffK);
  float(*Ps)[65] = reinterpret_cast<float(*)[65]>(smraw + SM::kOffP);
  double* colsum = reinterpret_cast<double*>(smraw + SM::kOffCol);
  double* red = reinterpret_cast<double*>(smraw + SM::kOffRed);
  int* off = reinterpret_cast<int*>(smraw + SM::kOffOff);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = a.S, nh = a.n_heads;
  if (warp == 0) {  // virtual item offsets of the heads' lists: a warp prefix sum, 32 heads per round
    int o = 0;
    for (int base = 0; base < nh; base += 32) {
      const int h = base + lane;
      const int c = h < nh ? ((a.gate != nullptr && a.gate[h] == 0) ? 0 : a.head_count[h]) : 0;
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      if (h < nh) off[h] = o + incl - c;
      o += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) off[nh] = o;
  }
  __syncthreads();
  const int total = off[nh];
  const int u0 = (int)((int64_t)blockIdx.x * total / gridDim.x), u1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  if (u0 >= u1) return;
  const int m0 = 16 * (warp >> 1), n0 = 32 * (warp & 1);  // warp's 16 rows x 32 keys of the item
  int h = 0;
  while (off[h + 1] <= u0) ++h;
  int cur_q = -1, kreg_item = -1;
  int4 kreg[kD / 32];
  auto item_kb = [&](int u, int hh) { return a.list[(int64_t)hh * a.n_kblk + (u - off[hh])]; };
  auto head_kbase = [&](int hh) {
    const int qh = a.head_ids ? a.head_ids[hh] : hh;
    return k + (int64_t)(qh / a.hpk) * S * kD;
  };
  auto needs_scores = [&](int u) { return kPass == 1 || a.cache == nullptr || u >= a.cache_items; };
  for (int u = u0; u < u1; ++u) {
    while (off[h + 1] <= u) ++h;
    const int kb = item_kb(u, h);
    const int k0 = kb * 64;
    double acc[2][4][2];
    if (needs_scores(u)) {
      if (kreg_item != u) fb_fetch<kD>(head_kbase(h) + (int64_t)k0 * kD, min(64, S - k0), kreg);
      __syncthreads();  // previous item's readers of Qs / Ks are done
      if (cur_q != h) {
        const int qh = a.head_ids ? a.head_ids[h] : h;
        int4 qreg[kD / 32];
        fb_fetch<kD>(q + ((int64_t)qh * S + (S - 64)) * kD, 64, qreg);
        fb_store<kD>(Qs, qreg);
        cur_q = h;
      }
      fb_store<kD>(Ks, kreg);
      __syncthreads();
      // prefetch the next item's keys while this one is scored
      if (u + 1 < u1 && needs_scores(u + 1)) {
        int hn = h;
        while (off[hn + 1] <= u + 1) ++hn;
        const int kbn = item_kb(u + 1, hn);
        fb_fetch<kD>(head_kbase(hn) + (int64_t)kbn * 64 * kD, min(64, S - kbn * 64), kreg);
        kreg_item = u + 1;
      }
      fb_scores<kD>(Qs, Ks, m0, n0, acc);
    }
    double* cw = (a.cache != nullptr && u < a.cache_items) ? a.cache + (size_t)u * (64 * 64) : nullptr;
    // scaled, causally masked scores of this thread's 16 cells
    double s[2][4][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = m0 + 8 * mi + (lane >> 2), jl = n0 + 8 * ni + 2 * (lane & 3) + e;
          double x;
          if (kPass == 2 && !needs_scores(u)) {
            x = cw[i * 64 + jl];
          } else {
            const bool valid = k0 + jl <= S - 64 + i;  // causal (also excludes keys >= S)
            x = valid ? a.scale * acc[mi][ni][e] : -INFINITY;
            if (kPass == 1 && cw != nullptr) cw[i * 64 + jl] = x;
          }
          s[mi][ni][e] = x;
        }
    if (kPass == 1) {
      // per row: max and sum exp over the item's 64 keys (4 lanes x 2 warps hold a row)
      double mx[2], l[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        double m = -INFINITY;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) m = fmax(m, fmax(s[mi][ni][0], s[mi][ni][1]));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
        mx[mi] = m;
      }
      if ((lane & 3) == 0) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) red[(warp & 1) * 64 + m0 + 8 * mi + (lane >> 2)] = mx[mi];
      }
      __syncthreads();
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int i = m0 + 8 * mi + (lane >> 2);
        mx[mi] = fmax(red[i], red[64 + i]);
        double acc_l = 0.0;
        if (mx[mi] != -INFINITY) {
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (s[mi][ni][e] != -INFINITY) acc_l += exp(s[mi][ni][e] - mx[mi]);
        }
        acc_l += __shfl_xor_sync(0xffffffffu, acc_l, 1);
        acc_l += __shfl_xor_sync(0xffffffffu, acc_l, 2);
        l[mi] = acc_l;
      }
      __syncthreads();  // row maxima read: red is reused for the sums
      if ((lane & 3) == 0) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) red[(warp & 1) * 64 + m0 + 8 * mi + (lane >> 2)] = l[mi];
      }
      __syncthreads();
      if ((warp & 1) == 0 && (lane & 3) == 0) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int i = m0 + 8 * mi + (lane >> 2);
          // indexed by list position: the combine visits only the listed items, in kb order
          a.stats[((int64_t)h * 64 + i) * a.n_kblk + (u - off[h])] = make_double2(mx[mi], red[i] + red[64 + i]);
        }
      }
    } else {
      // p = fp32(exp(s - m_i) / l_i) (tensor.py:78); column sums over rows ascending and
      // diagonal sums as vs_exact_kernel (est.sum(axis=0) / np.bincount orders)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int i = m0 + 8 * mi + (lane >> 2);
        const double2 ml = a.row_ml[(int64_t)h * 64 + i];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double x = s[mi][ni][e];
            Ps[i][n0 + 8 * ni + 2 * (lane & 3) + e] = x == -INFINITY ? 0.f : __double2float_rn(exp(x - ml.x) / ml.y);
          }
      }
      __syncthreads();
      // columns on warps 0-1, diagonals on warps 2-5 (concurrently); each sum runs over the
      // rows in ascending order (the reference's order), its loads issued ahead of the adds
      if (tid < 64) {
        double cs = 0.0;
#pragma unroll 16
        for (int ii = 0; ii < 64; ++ii) cs += (double)Ps[ii][tid];
        if (k0 + tid < S) a.vscore[(int64_t)h * S + k0 + tid] = cs;
      } else if (tid < 64 + 127) {
        // diagonal cl = key - row in [-63, 63]; offset o = (S - 64 + row) - (k0 + key)
        const int cl = tid - 64 - 63;
        const int ii0 = max(0, -cl), ii1 = min(64, 64 - cl);
        double ds = 0.0;
#pragma unroll 16
        for (int ii = ii0; ii < ii1; ++ii) ds += (double)Ps[ii][ii + cl];
        const int o = S - 64 - k0 - cl;
        if (o >= 0 && o < S && ds != 0.0) atomicAdd(a.sscore + (int64_t)h * S + o, ds);
      }
      __syncthreads();  // Ps is rewritten by the next item
    }
  }
}

// (m_i, l_i) from the item partials: one warp per (head, row), lane-strided then a
// fixed butterfly, so the order is deterministic.
__global__ void vs_exact_combine_kernel(const ExArgs a) {
  const int h = blockIdx.y;
  if (a.gate != nullptr && a.gate[h] == 0) return;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= a.L) return;
  const double2* st = a.stats + ((int64_t)h * a.L + i) * a.n_kblk;
  // fallback: the listed items' statistics (by list position); otherwise every item's
  const int n_st = a.head_count != nullptr ? a.head_count[h] : a.n_kblk;
  double m = -INFINITY;
  for (int b = lane; b < n_st; b += 32) m = fmax(m, st[b].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  double l = 0.0;
  for (int b = lane; b < n_st; b += 32) {
    const double2 v = st[b];
    if (v.x != -INFINITY) l += v.y * exp(v.x - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) a.row_ml[(int64_t)h * a.L + i] = make_double2(m, l);  // pass 2 divides by l
}

constexpr int kTopkThreads = 256;
constexpr int kTopkCl = 8;

__global__ void __cluster_dims__(kTopkCl, 1, 1) __launch_bounds__(kTopkThreads)
    vs_exact_topk_kernel(const double* __restrict__ vscore, const double* __restrict__ sscore, int S, int k_v,
                         int k_s, const int32_t* gate, int32_t* __restrict__ vert_out,
                         int32_t* __restrict__ slash_out, const int32_t* __restrict__ list,
                         const int32_t* __restrict__ head_count, int n_kblk, int KB, int L) {
  using TK = ClusterTopK<kTopkThreads, kTopkCl>;
  __shared__ typename TK::Storage sm;
  const int hi = blockIdx.y;
  if (gate != nullptr && gate[hi] == 0) return;  // cluster-uniform
  // fallback heads: only the listed items carry nonzero vertical scores, and only the
  // diagonals through them nonzero slash scores (everything else was written +0 by prep)
  int lo_v = 0, hi_v = -1, lo_s = 0, hi_s = -1;
  if (list != nullptr && head_count[hi] > 0) {
    const int32_t* lh = list + (int64_t)hi * n_kblk;  // ascending (vs_exact_list_kernel)
    lo_v = lh[0] * KB;
    hi_v = min(S, (lh[head_count[hi] - 1] + 1) * KB);
    lo_s = max(0, S - L - (hi_v - 1));  // offset o = (S - L + i) - j, i in [0, L), j in [lo_v, hi_v)
    hi_s = min(S, S - lo_v);
  }
  if (blockIdx.z == 0)
    TK::run(sm, vscore + (int64_t)hi * S, S, k_v, false, vert_out + (int64_t)hi * k_v, nullptr, nullptr, lo_v, hi_v);
  else
    TK::run(sm, sscore + (int64_t)hi * S, S, k_s, true, slash_out + (int64_t)hi * k_s, nullptr, nullptr, lo_s, hi_s);
}

int kb_for(int L) { return kKeyT * max(1, (L - 1 + kKeyT - 1) / kKeyT); }

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

static int cache_items_for(int n_heads, int seq_len, int last_q) {
  const int KB = kb_for(last_q);
  if (last_q != 64 || KB != 64) return 0;
  const int64_t n = (int64_t)n_heads * ((seq_len + KB - 1) / KB);
  return (int)std::min<int64_t>(n, kCacheItems);
}

size_t vs_exact_workspace_size(int n_heads, int seq_len, int last_q) {
  const int KB = kb_for(last_q);
  const size_t n_kblk = (seq_len + KB - 1) / KB;
  return al256((size_t)n_heads * last_q * n_kblk * 16) + al256((size_t)n_heads * last_q * 16) +
         2 * al256((size_t)n_heads * seq_len * 8) + al256((size_t)n_heads * n_kblk * 4) + al256((size_t)n_heads * 4) +
         al256((size_t)n_heads * n_kblk) +
         al256((size_t)cache_items_for(n_heads, seq_len, last_q) * 64 * 64 * 8);
}

int vs_exact_run(int dtype, const void* q, const void* k, int Hq, int Hkv, int S, int d, const int32_t* head_ids,
                 int n_heads, int L, int k_v, int k_s, int32_t* vout, int32_t* sout, double* vscore, double* sscore,
                 const int32_t* gate, const float* tile_max, const float* row_mc, const float* row_marg,
                 void* workspace, cudaStream_t st) {
  if (L > kMaxL) return set_error(SPF_ERR_INVALID, "last_q=%d exceeds the supported %d", L, kMaxL);
  ExArgs a{};
  a.S = S;
  a.d = d;
  a.L = L;
  a.KB = kb_for(L);
  a.n_kblk = (S + a.KB - 1) / a.KB;
  a.n_heads = n_heads;
  a.hpk = Hq / Hkv;
  a.head_ids = head_ids;
  a.gate = gate;
  a.tile_max = (L == 64 && a.KB == 64) ? tile_max : nullptr;
  a.row_mc = row_mc;
  a.row_marg = row_marg;
  a.scale = 1.0 / sqrt((double)d);
  a.c = (float)(a.scale * 1.4426950408889634);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  auto take = [&](size_t bytes) {
    uint8_t* p = ws;
    ws += al256(bytes);
    return p;
  };
  a.stats = reinterpret_cast<double2*>(take((size_t)n_heads * L * a.n_kblk * 16));
  a.row_ml = reinterpret_cast<double2*>(take((size_t)n_heads * L * 16));
  a.vscore = vscore ? vscore : reinterpret_cast<double*>(take((size_t)n_heads * S * 8));
  a.sscore = sscore ? sscore : reinterpret_cast<double*>(take((size_t)n_heads * S * 8));
  int32_t* list = reinterpret_cast<int32_t*>(take((size_t)n_heads * a.n_kblk * 4));
  int32_t* head_count = reinterpret_cast<int32_t*>(take((size_t)n_heads * 4));
  uint8_t* sig = take((size_t)n_heads * a.n_kblk);
  const int cache_items = cache_items_for(n_heads, S, L);
  double* cache = reinterpret_cast<double*>(take((size_t)cache_items * 64 * 64 * 8));
  const size_t smem = sizeof(ExSmem) + (size_t)(2 * a.KB + L - 1) * 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)a.n_kblk * n_heads, 148 * 4));
  int rc;
  const bool fallback = tile_max != nullptr && L == 64 && a.KB == 64 && dtype == SPF_DTYPE_BF16 &&
                        (d == 64 || d == 128) && n_heads <= kMaxFbHeads;
  if (fallback) {
    // flagged heads only: list their significant items, score them on the fp64 tensor cores
    a.list = list;
    a.sig = sig;
    a.head_count = head_count;
    a.cache = cache_items > 0 ? cache : nullptr;
    a.cache_items = cache_items;
    const int64_t warps = (int64_t)n_heads * a.n_kblk;
    auto k1 = d == 128 ? vs_fb_kernel<128, 1> : vs_fb_kernel<64, 1>;
    auto k2 = d == 128 ? vs_fb_kernel<128, 2> : vs_fb_kernel<64, 2>;
    const int fb_smem = d == 128 ? FbSmem<128>::kBytes : FbSmem<64>::kBytes;
    static bool fb_attr = false;
    if (!fb_attr) {
      for (auto kk : {vs_fb_kernel<128, 1>, vs_fb_kernel<128, 2>})
        if ((rc = check_cuda(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  FbSmem<128>::kBytes), "vs fallback smem")))
          return rc;
      for (auto kk : {vs_fb_kernel<64, 1>, vs_fb_kernel<64, 2>})
        if ((rc = check_cuda(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  FbSmem<64>::kBytes), "vs fallback smem")))
          return rc;
      fb_attr = true;
    }
    const auto* qb = reinterpret_cast<const __nv_bfloat16*>(q);
    const auto* kbp = reinterpret_cast<const __nv_bfloat16*>(k);
    note_launches(6);  // prep, list, pass A, combine, pass B, top-k
    vs_exact_prep_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
    vs_exact_list_kernel<<<(unsigned)n_heads, kListThreads, 0, st>>>(a);
    k1<<<2 * 148, kFbThreads, fb_smem, st>>>(qb, kbp, a);  // two CTAs per SM
    vs_exact_combine_kernel<<<dim3((unsigned)((L + 7) / 8), (unsigned)n_heads), 256, 0, st>>>(a);
    k2<<<2 * 148, kFbThreads, fb_smem, st>>>(qb, kbp, a);
    vs_exact_topk_kernel<<<dim3(kTopkCl, (unsigned)n_heads, 2), kTopkThreads, 0, st>>>(
        a.vscore, a.sscore, S, k_v, k_s, gate, vout, sout, a.list, a.head_count, a.n_kblk, a.KB, L);
    return check_cuda(cudaGetLastError(), "vs fallback");
  }
  a.tile_max = nullptr;  // the full fp64 path visits every item
  auto launch = [&](auto k1, auto k2, const auto* qq, const auto* kk) {
    if ((rc = check_cuda(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                         "vs exact smem")))
      return rc;
    if ((rc = check_cuda(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                         "vs exact smem")))
      return rc;
    note_launches(4);  // pass A, combine, pass B, top-k
    k1<<<grid, kThreads, smem, st>>>(qq, kk, a);
    vs_exact_combine_kernel<<<dim3((unsigned)((L + 7) / 8), (unsigned)n_heads), 256, 0, st>>>(a);
    k2<<<grid, kThreads, smem, st>>>(qq, kk, a);
    vs_exact_topk_kernel<<<dim3(kTopkCl, (unsigned)n_heads, 2), kTopkThreads, 0, st>>>(
        a.vscore, a.sscore, S, k_v, k_s, gate, vout, sout, nullptr, nullptr, 0, 0, L);
    return check_cuda(cudaGetLastError(), "vs exact");
  };
  if (dtype == SPF_DTYPE_BF16)
    return launch(vs_exact_kernel<__nv_bfloat16, 1>, vs_exact_kernel<__nv_bfloat16, 2>,
                  reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k));
  return launch(vs_exact_kernel<float, 1>, vs_exact_kernel<float, 2>, reinterpret_cast<const float*>(q),
                reinterpret_cast<const float*>(k));
}

}  // namespace spf
