// estimate.cu -- online sparse-index estimation on the GPU.
//
// Vertical-Slash: see estimate_vs_tc.cu (tensor cores, production) and
// estimate_vs_exact.cu (fp64).  The description below is the reference
// algorithm both follow, estimator.py:82-114 (rounding points of tensor.py:61-78):
//   1. score pass   s[i][j] = scale * (q_tail[i] . k[j]) in fp64 (exact-enough:
//                   bf16/fp32 inputs, fp64 FMA chain), masked j > abs_i, plus
//                   per-(row, 64-key block) partial (max, sum exp);
//   2. row stats    m_i, l_i combined from the partials (fixed tree order);
//   3. vertical     p[i][j] = fp32(exp(s - m_i) / l_i) (the reference's fp32
//                   rounding point), vertical[j] = sum_i p (fp64, i ascending,
//                   est.sum(axis=0));
//   4. slash        slash[o] = sum_i p[i][abs_i - o] (fp64, i ascending, the
//                   np.bincount order);
//   5. top-k        block radix select, lowest index wins ties, index 0 forced.
// Block-Sparse, estimator.py:117-143:
//   1. pooling      fp64 block sums / real length -> fp32 (tensor.py:43-58);
//   2. score pass   pooled scores in fp64 for the causal block triangle;
//   3. row pass     block-causal softmax -> fp32, top-min(k_b, r+1) with the
//                   diagonal forced, written straight into the CSR tile layout
//                   (tile start = block * B, sparse_attn.py:30-33).
// fp64 is used for every score so the fp32-rounded probabilities -- and hence
// the selected index sets -- are those of the reference.
#include <cuda_bf16.h>

#include "spf.h"
#include "spf_internal.h"
#include "topk.cuh"

namespace spf {
namespace {

constexpr int kTile = 64;       // rows x keys per score tile
constexpr int kScoreThreads = 256;

template <typename T>
__device__ __forceinline__ double ld_as_double(const T* p) {
  return static_cast<double>(static_cast<float>(*p));
}
template <>
__device__ __forceinline__ double ld_as_double<__nv_bfloat16>(const __nv_bfloat16* p) {
  return static_cast<double>(__bfloat162float(*p));
}

// Block-Sparse pooled scores, fp64: out[r][c] = scale * qp[r] . kp[c] for the block-causal
// triangle (c <= r), one 64x64 tile per CTA.  d is staged in 32-wide chunks (two CTAs
// per SM); each thread owns rows 4 tr .. 4 tr + 3 and columns tk + 16 y, so the column
// operand is read conflict-free (16 consecutive doubles per warp load).
constexpr int kDc = 32;
constexpr int kLdc = 68;

__global__ void __launch_bounds__(kScoreThreads, 2) bs_score_kernel(
    const float* __restrict__ qp, const float* __restrict__ kp, const int32_t* __restrict__ head_ids,
    int heads_per_kv, int N, int d, double scale, double* __restrict__ out) {
  __shared__ double At[kDc * kLdc];
  __shared__ double Bt[kDc * kLdc];
  const int hi = blockIdx.z;
  const int h = head_ids ? head_ids[hi] : hi;
  const int kvh = h / heads_per_kv;
  const int bt = blockIdx.x, at = blockIdx.y;
  if (bt > at) return;  // block-causal triangle only
  const int a0 = at * kTile, b0 = bt * kTile;
  const float* Ah = qp + (int64_t)h * N * d;
  const float* Bh = kp + (int64_t)kvh * N * d;
  const int tid = threadIdx.x, tr = tid >> 4, tk = tid & 15;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int c0 = 0; c0 < d; c0 += kDc) {
    __syncthreads();
    for (int e = tid; e < kTile * kDc; e += kScoreThreads) {
      const int r = e / kDc, c = e % kDc;
      const bool okc = c0 + c < d;
      At[c * kLdc + r] = (okc && a0 + r < N) ? (double)Ah[(int64_t)(a0 + r) * d + c0 + c] : 0.0;
      Bt[c * kLdc + r] = (okc && b0 + r < N) ? (double)Bh[(int64_t)(b0 + r) * d + c0 + c] : 0.0;
    }
    __syncthreads();
    const int cn = min(kDc, d - c0);
#pragma unroll 4
    for (int c = 0; c < cn; ++c) {
      const double2 qa = *reinterpret_cast<const double2*>(At + c * kLdc + 4 * tr);
      const double2 qb = *reinterpret_cast<const double2*>(At + c * kLdc + 4 * tr + 2);
      const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
      double kv[4];
#pragma unroll
      for (int y = 0; y < 4; ++y) kv[y] = Bt[c * kLdc + tk + 16 * y];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[i][y] = fma(qv[i], kv[y], acc[i][y]);
    }
  }
  double* outh = out + (int64_t)hi * N * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + 4 * tr + i;
    if (a >= N) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int b = b0 + tk + 16 * y;
      if (b < N) outh[(int64_t)a * N + b] = (b <= a) ? scale * acc[i][y] : -INFINITY;
    }
  }
}

// Same scores, same per-element fma order (c ascending), for d % 4 == 0: 128 threads per
// 64x64 tile of the block-causal triangle only (blockIdx.x enumerates the lower-triangle
// tiles), 8 rows x 4 columns per thread so the fp64 pipe, not shared memory, is the
// limit; the staged operands are stored with consecutive rows in consecutive lanes
// (conflict-free) from 16-byte global loads.
constexpr int kScore2Threads = 128;

__global__ void __launch_bounds__(kScore2Threads, 4) bs_score_tri_kernel(
    const float* __restrict__ qp, const float* __restrict__ kp, const int32_t* __restrict__ head_ids,
    int heads_per_kv, int N, int d, double scale, double* __restrict__ out) {
  __shared__ __align__(16) double At[kDc * kTile];
  __shared__ __align__(16) double Bt[kDc * kTile];
  const int hi = blockIdx.y;
  const int h = head_ids ? head_ids[hi] : hi;
  const int kvh = h / heads_per_kv;
  // lower-triangle tile t -> (at, bt), bt <= at
  const int t = blockIdx.x;
  int at = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((at + 1) * (at + 2) / 2 <= t) ++at;
  while (at * (at + 1) / 2 > t) --at;
  const int bt = t - at * (at + 1) / 2;
  const int a0 = at * kTile, b0 = bt * kTile;
  const float* Ah = qp + (int64_t)h * N * d;
  const float* Bh = kp + (int64_t)kvh * N * d;
  const int tid = threadIdx.x, tr = tid >> 4, tk = tid & 15;
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int c0 = 0; c0 < d; c0 += kDc) {
    __syncthreads();
    const int cn = min(kDc, d - c0);
    for (int e = tid; e < kTile * (kDc / 4); e += kScore2Threads) {
      const int r = e & (kTile - 1), c4 = (e >> 6) * 4;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (c4 < cn) {
        if (a0 + r < N) a = *reinterpret_cast<const float4*>(Ah + (int64_t)(a0 + r) * d + c0 + c4);
        if (b0 + r < N) b = *reinterpret_cast<const float4*>(Bh + (int64_t)(b0 + r) * d + c0 + c4);
      }
      At[(c4 + 0) * kTile + r] = a.x;
      At[(c4 + 1) * kTile + r] = a.y;
      At[(c4 + 2) * kTile + r] = a.z;
      At[(c4 + 3) * kTile + r] = a.w;
      Bt[(c4 + 0) * kTile + r] = b.x;
      Bt[(c4 + 1) * kTile + r] = b.y;
      Bt[(c4 + 2) * kTile + r] = b.z;
      Bt[(c4 + 3) * kTile + r] = b.w;
    }
    __syncthreads();
    auto step = [&](int c) {
      double qv[8], kv[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double2 v = *reinterpret_cast<const double2*>(At + c * kTile + 8 * tr + 2 * m);
        qv[2 * m] = v.x;
        qv[2 * m + 1] = v.y;
      }
#pragma unroll
      for (int y = 0; y < 4; ++y) kv[y] = Bt[c * kTile + tk + 16 * y];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[i][y] = fma(qv[i], kv[y], acc[i][y]);
    };
    if (cn == kDc) {  // fully unrolled: the shared-memory loads are scheduled ahead of the fmas
#pragma unroll
      for (int c = 0; c < kDc; ++c) step(c);
    } else {
#pragma unroll 1
      for (int c = 0; c < cn; ++c) step(c);
    }
  }
  double* outh = out + (int64_t)hi * N * N;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int a = a0 + 8 * tr + i;
    if (a >= N) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int b = b0 + tk + 16 * y;
      if (b < N) outh[(int64_t)a * N + b] = (b <= a) ? scale * acc[i][y] : -INFINITY;
    }
  }
}

// The same scores on the fp64 tensor cores (DMMA mma.sync m8n8k4 f64; 37 TF/s vs ~20 for the
// FMA kernel above, benchmarks/mb_dmma.cu) for d = 64 / 128: the block-causal tile's 64 pooled
// rows of Q and K staged as fp32 (exact: the pooled means are fp32) with a 4-float pad (the
// 8 rows a fragment load touches fall on distinct banks), converted to fp64 at fragment load;
// 4 warps, each 16 rows x 64 columns (16 accumulators); three CTAs per SM.
constexpr int kScoreDmmaThreads = 128;

template <int kD>
__global__ void __launch_bounds__(kScoreDmmaThreads, 3) bs_score_dmma_kernel(
    const float* __restrict__ qp, const float* __restrict__ kp, const int32_t* __restrict__ head_ids,
    int heads_per_kv, int N, double scale, double* __restrict__ out) {
  constexpr int kLd = kD + 4;
  extern __shared__ __align__(16) float sm_f[];
  float* As = sm_f;
  float* Bs = sm_f + kTile * kLd;
  const int hi = blockIdx.y;
  const int h = head_ids ? head_ids[hi] : hi;
  const int kvh = h / heads_per_kv;
  const int t = blockIdx.x;  // lower-triangle tile t -> (at, bt), bt <= at
  int at = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((at + 1) * (at + 2) / 2 <= t) ++at;
  while (at * (at + 1) / 2 > t) --at;
  const int bt = t - at * (at + 1) / 2;
  const int a0 = at * kTile, b0 = bt * kTile;
  const float* Ah = qp + ((int64_t)h * N + a0) * kD;
  const float* Bh = kp + ((int64_t)kvh * N + b0) * kD;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < kTile * (kD / 4); e += kScoreDmmaThreads) {
    const int r = e / (kD / 4), c4 = (e % (kD / 4)) * 4;
    const float4 a = a0 + r < N ? *reinterpret_cast<const float4*>(Ah + (int64_t)r * kD + c4) : make_float4(0, 0, 0, 0);
    const float4 b = b0 + r < N ? *reinterpret_cast<const float4*>(Bh + (int64_t)r * kD + c4) : make_float4(0, 0, 0, 0);
    *reinterpret_cast<float4*>(As + r * kLd + c4) = a;
    *reinterpret_cast<float4*>(Bs + r * kLd + c4) = b;
  }
  __syncthreads();
  double acc[2][8][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 8; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  // k4 steps walk each 16-wide slice of d as k = 16 kk + 4 (lane % 4) + j, j = 0..3 (the same
  // map for both operands): a lane's four values of a slice are one 16-byte load
  const float* qa = As + (16 * warp + (lane >> 2)) * kLd + 4 * (lane & 3);
  const float* kb = Bs + (lane >> 2) * kLd + 4 * (lane & 3);
#pragma unroll 1
  for (int kk = 0; kk < kD / 16; ++kk) {
    float4 af[2], bf[8];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) af[mi] = *reinterpret_cast<const float4*>(qa + mi * 8 * kLd + 16 * kk);
#pragma unroll
    for (int ni = 0; ni < 8; ++ni) bf[ni] = *reinterpret_cast<const float4*>(kb + ni * 8 * kLd + 16 * kk);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a[2], b[8];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
        a[mi] = (double)(j == 0 ? af[mi].x : j == 1 ? af[mi].y : j == 2 ? af[mi].z : af[mi].w);
#pragma unroll
      for (int ni = 0; ni < 8; ++ni)
        b[ni] = (double)(j == 0 ? bf[ni].x : j == 1 ? bf[ni].y : j == 2 ? bf[ni].z : bf[ni].w);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 8; ++ni)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[mi][ni][0]), "+d"(acc[mi][ni][1])
                       : "d"(a[mi]), "d"(b[ni]));
    }
  }
  double* outh = out + (int64_t)hi * N * N;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int a = a0 + 16 * warp + 8 * mi + (lane >> 2);
    if (a >= N) continue;
#pragma unroll
    for (int ni = 0; ni < 8; ++ni) {
      const int b = b0 + 8 * ni + 2 * (lane & 3);
      const double v0 = (b <= a) ? scale * acc[mi][ni][0] : -INFINITY;
      const double v1 = (b + 1 <= a) ? scale * acc[mi][ni][1] : -INFINITY;
      if (b + 1 < N) *reinterpret_cast<double2*>(outh + (int64_t)a * N + b) = make_double2(v0, v1);
      else if (b < N) outh[(int64_t)a * N + b] = v0;
    }
  }
}

// ---------------------------------------------------------------- Block-Sparse
template <typename T>
__global__ void pool_kernel(const T* __restrict__ x, int64_t n_rows_total, int S, int d, int B,
                            float* __restrict__ pooled) {
  // one thread per (head-row-block, column): fp64 sequential sum / real length -> fp32
  const int n_blk = (S + B - 1) / B;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = n_rows_total * (int64_t)n_blk * d;  // n_rows_total = number of heads
  if (idx >= total) return;
  const int c = (int)(idx % d);
  const int64_t hb = idx / d;
  const int64_t h = hb / n_blk;
  const int r = (int)(hb % n_blk);
  const int r0 = r * B, r1 = min(r0 + B, S);
  const T* base = x + (h * S + r0) * (int64_t)d + c;
  double acc = 0.0;
  for (int i = 0; i < r1 - r0; ++i) acc += ld_as_double(base + (int64_t)i * d);
  pooled[idx] = __double2float_rn(acc / (double)(r1 - r0));
}

// Vectorised pooling: one thread per (head, row block, 16-byte column chunk), the same
// sequential fp64 sum per column as pool_kernel (identical results); requires
// d * sizeof(T) % 16 == 0 and a 16-byte aligned base.
template <typename T>
__global__ void pool_vec_kernel(const T* __restrict__ x, int64_t n_heads, int S, int d, int B,
                                float* __restrict__ pooled) {
  constexpr int kV = 16 / sizeof(T);
  const int n_blk = (S + B - 1) / B;
  const int dv = d / kV;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n_heads * (int64_t)n_blk * dv) return;
  const int cv = (int)(idx % dv);
  const int64_t hb = idx / dv;
  const int64_t h = hb / n_blk;
  const int r = (int)(hb % n_blk);
  const int r0 = r * B, len = min(B, S - r0);
  const uint4* base = reinterpret_cast<const uint4*>(x + (h * S + r0) * (int64_t)d) + cv;
  double acc[kV];
#pragma unroll
  for (int j = 0; j < kV; ++j) acc[j] = 0.0;
#pragma unroll 8
  for (int i = 0; i < len; ++i) {
    const uint4 u = __ldcs(base + (int64_t)i * dv);
    const T* v = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < kV; ++j) acc[j] += ld_as_double(v + j);
  }
  float4* out = reinterpret_cast<float4*>(pooled + hb * d + (int64_t)cv * kV);
#pragma unroll
  for (int j = 0; j < kV; j += 4)
    out[j / 4] = make_float4(__double2float_rn(acc[j] / len), __double2float_rn(acc[j + 1] / len),
                             __double2float_rn(acc[j + 2] / len), __double2float_rn(acc[j + 3] / len));
}

constexpr int kBsThreads = 256;  // 128 measured 2 % slower on C4

// One CTA per (head, block row r): block-causal softmax of the pooled scores
// (fp64, rounded to fp32), top-min(k_b, r+1) with the diagonal forced.  The row's
// exponentials overwrite its scores (scratch), so each is evaluated once.
__global__ void __launch_bounds__(kBsThreads) bs_row_kernel(double* __restrict__ scores, int N, int k_b, int B,
                                                            const int32_t* __restrict__ head_ids,
                                                            const int64_t* __restrict__ tile_offsets,
                                                            int32_t* __restrict__ tile_starts) {
  using TK = BlockTopK<kBsThreads, float>;
  __shared__ typename TK::Storage sm;
  __shared__ double red[kBsThreads / 32];
  extern __shared__ float pv[];  // [N]
  const int hi = blockIdx.y;
  const int h = head_ids ? head_ids[hi] : hi;
  const int r = blockIdx.x;
  const int n = r + 1;
  double* sr = scores + ((int64_t)hi * N + r) * N;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // row max (exact)
  double m = -INFINITY;
  for (int b = tid; b < n; b += kBsThreads) m = fmax(m, sr[b]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[wid] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < kBsThreads / 32; ++w) m = fmax(m, red[w]);
  __syncthreads();
  // denominator (fixed tree order)
  double l = 0.0;
  for (int b = tid; b < n; b += kBsThreads) {  // the exponential is kept in place (same thread reads it back)
    const double e = exp(sr[b] - m);
    sr[b] = e;
    l += e;
  }
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) red[wid] = l;
  __syncthreads();
  l = 0.0;
  for (int w = 0; w < kBsThreads / 32; ++w) l += red[w];
  for (int b = tid; b < n; b += kBsThreads) pv[b] = __double2float_rn(sr[b] / l);
  __syncthreads();
  const int64_t row = (int64_t)h * N + r;
  // a row emptied by spf_csr_guard (speculative sizing overflowed) receives nothing
  if (tile_offsets[row + 1] - tile_offsets[row] < min(k_b, n)) return;
  TK::run(sm, pv, n, min(k_b, n), r, false, tile_starts + tile_offsets[row], B);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename T>
int bs_estimate_impl(const T* q, const T* k, int Hq, int Hkv, int S, int d, const int32_t* head_ids, int n_heads,
                     int k_b, int B, const int64_t* tile_offsets, int32_t* tile_starts, uint8_t* ws,
                     cudaStream_t st) {
  const int N = (S + B - 1) / B;
  float* qp = reinterpret_cast<float*>(ws);
  ws += align256((size_t)Hq * N * d * 4);
  float* kp = reinterpret_cast<float*>(ws);
  ws += align256((size_t)Hkv * N * d * 4);
  double* sc = reinterpret_cast<double*>(ws);  // [n_heads][N][N]
  int rc;
  {
    const int64_t tq = (int64_t)Hq * N * d, tk = (int64_t)Hkv * N * d;
    note_launches(3);  // pool q, pool k, row top-k (+1 block scores below)
    constexpr int kV = 16 / sizeof(T);
    const bool vec = d % kV == 0 && reinterpret_cast<uintptr_t>(q) % 16 == 0 && reinterpret_cast<uintptr_t>(k) % 16 == 0;
    if (vec) {
      pool_vec_kernel<T><<<(unsigned)((tq / kV + 255) / 256), 256, 0, st>>>(q, Hq, S, d, B, qp);
      pool_vec_kernel<T><<<(unsigned)((tk / kV + 255) / 256), 256, 0, st>>>(k, Hkv, S, d, B, kp);
    } else {
      pool_kernel<T><<<(unsigned)((tq + 255) / 256), 256, 0, st>>>(q, Hq, S, d, B, qp);
      pool_kernel<T><<<(unsigned)((tk + 255) / 256), 256, 0, st>>>(k, Hkv, S, d, B, kp);
    }
    if ((rc = check_cuda(cudaGetLastError(), "bs pool"))) return rc;
  }
  const int nt = (N + kTile - 1) / kTile;
  note_launches(1);
  if ((d == 128 || d == 64) && N % 2 == 0) {  // fp64 tensor cores (double2 stores need an even row length)
    const unsigned grid_t = (unsigned)(nt * (nt + 1) / 2);
    const int smem = 2 * kTile * (d + 4) * (int)sizeof(float);
    static bool attr = false;
    if (!attr) {
      if ((rc = check_cuda(cudaFuncSetAttribute(bs_score_dmma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                2 * kTile * (128 + 4) * 4), "bs score smem")))
        return rc;
      if ((rc = check_cuda(cudaFuncSetAttribute(bs_score_dmma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                2 * kTile * (64 + 4) * 4), "bs score smem")))
        return rc;
      attr = true;
    }
    if (d == 128)
      bs_score_dmma_kernel<128><<<dim3(grid_t, (unsigned)n_heads), kScoreDmmaThreads, smem, st>>>(
          qp, kp, head_ids, Hq / Hkv, N, 1.0 / sqrt((double)d), sc);
    else
      bs_score_dmma_kernel<64><<<dim3(grid_t, (unsigned)n_heads), kScoreDmmaThreads, smem, st>>>(
          qp, kp, head_ids, Hq / Hkv, N, 1.0 / sqrt((double)d), sc);
  } else if (d % 4 == 0)
    bs_score_tri_kernel<<<dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)n_heads), kScore2Threads, 0, st>>>(
        qp, kp, head_ids, Hq / Hkv, N, d, 1.0 / sqrt((double)d), sc);
  else
    bs_score_kernel<<<dim3((unsigned)nt, (unsigned)nt, (unsigned)n_heads), kScoreThreads, 0, st>>>(
        qp, kp, head_ids, Hq / Hkv, N, d, 1.0 / sqrt((double)d), sc);
  if ((rc = check_cuda(cudaGetLastError(), "bs score"))) return rc;
  const size_t rsmem = (size_t)N * sizeof(float);
  if ((rc = check_cuda(cudaFuncSetAttribute(bs_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem),
                       "bs row smem attr")))
    return rc;
  bs_row_kernel<<<dim3((unsigned)N, (unsigned)n_heads), kBsThreads, rsmem, st>>>(sc, N, k_b, B, head_ids,
                                                                                 tile_offsets, tile_starts);
  return check_cuda(cudaGetLastError(), "bs row");
}

}  // namespace
}  // namespace spf

using namespace spf;

extern "C" {

size_t spf_vs_estimate_workspace_size(int mode, int dtype, int n_q_heads, int n_kv_heads, int n_heads, int seq_len,
                                      int head_dim, int last_q) {
  if (mode != SPF_VS_EXACT && vs_fast_supported(dtype, head_dim, seq_len, last_q))
    return vs_fast_workspace_size(n_q_heads, n_kv_heads, n_heads, seq_len);
  return vs_exact_workspace_size(n_heads, seq_len, last_q);
}

int spf_vs_estimate(int mode, int dtype, const void* q, const void* k, int n_q_heads, int n_kv_heads, int seq_len,
                    int head_dim, const int32_t* head_ids, int n_heads, int last_q, int k_v, int k_s,
                    int32_t* vertical_out, int32_t* slash_out, double* vscore_out, double* sscore_out,
                    int32_t* uncertain_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (mode != SPF_VS_EXACT && mode != SPF_VS_FAST && mode != SPF_VS_FAST_UNCERTIFIED)
    return set_error(SPF_ERR_INVALID, "unknown estimation mode %d", mode);
  if (dtype != SPF_DTYPE_BF16 && dtype != SPF_DTYPE_F32) return set_error(SPF_ERR_INVALID, "unknown dtype %d", dtype);
  if (last_q < 1 || k_v < 1 || k_s < 1) return set_error(SPF_ERR_INVALID, "Vertical-Slash counts must be >= 1");
  if (last_q > seq_len) return set_error(SPF_ERR_INVALID, "last_q=%d exceeds seq_len=%d", last_q, seq_len);
  if (head_dim < 1 || head_dim > 128) return set_error(SPF_ERR_INVALID, "head_dim must be in [1, 128]");
  if (n_kv_heads < 1 || n_q_heads % n_kv_heads) return set_error(SPF_ERR_INVALID, "bad head counts");
  if (n_heads <= 0) return SPF_OK;
  const size_t need = spf_vs_estimate_workspace_size(mode, dtype, n_q_heads, n_kv_heads, n_heads, seq_len, head_dim,
                                                     last_q);
  if (workspace == nullptr || workspace_bytes < need)
    return set_error(SPF_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
  const int kv = min(k_v, seq_len), ks = min(k_s, seq_len);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  if (mode != SPF_VS_EXACT && vs_fast_supported(dtype, head_dim, seq_len, last_q))
    return vs_estimate_fast(q, k, n_q_heads, n_kv_heads, seq_len, head_dim, head_ids, n_heads, kv, ks, vertical_out,
                            slash_out, vscore_out, sscore_out, uncertain_out, mode == SPF_VS_FAST_UNCERTIFIED, ws,
                            st);
  if (uncertain_out != nullptr) {
    int rc = check_cuda(cudaMemsetAsync(uncertain_out, 0, (size_t)n_heads * sizeof(int32_t), st), "memset flags");
    if (rc) return rc;
  }
  return vs_exact_run(dtype, q, k, n_q_heads, n_kv_heads, seq_len, head_dim, head_ids, n_heads, last_q, kv, ks,
                      vertical_out, slash_out, vscore_out, sscore_out, nullptr, nullptr, nullptr, nullptr, ws, st);
}

size_t spf_bs_estimate_workspace_size(int n_q_heads, int n_kv_heads, int seq_len, int head_dim, int block_size) {
  const size_t N = (seq_len + block_size - 1) / block_size;
  return align256((size_t)n_q_heads * N * head_dim * 4) + align256((size_t)n_kv_heads * N * head_dim * 4) +
         align256((size_t)n_q_heads * N * N * 8);
}

int spf_bs_estimate(int dtype, const void* q, const void* k, int n_q_heads, int n_kv_heads, int seq_len,
                    int head_dim, const int32_t* head_ids, int n_heads, int k_b, int block_size,
                    const int64_t* tile_offsets, int32_t* tile_starts, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (k_b < 1 || block_size < 1) return set_error(SPF_ERR_INVALID, "Block-Sparse counts must be >= 1");
  if (head_dim < 1 || head_dim > 128) return set_error(SPF_ERR_INVALID, "head_dim must be in [1, 128]");
  if (n_kv_heads < 1 || n_q_heads % n_kv_heads) return set_error(SPF_ERR_INVALID, "bad head counts");
  const int N = (seq_len + block_size - 1) / block_size;
  if ((size_t)N * sizeof(float) > 200 * 1024)
    return set_error(SPF_ERR_INVALID, "too many block rows (%d) for the per-row top-k", N);
  if (n_heads <= 0) return SPF_OK;
  // scores scratch is sized for n_heads (the heads actually estimated)
  const size_t need = align256((size_t)n_q_heads * N * head_dim * 4) + align256((size_t)n_kv_heads * N * head_dim * 4) +
                      align256((size_t)n_heads * N * N * 8);
  if (workspace == nullptr || workspace_bytes < need)
    return set_error(SPF_ERR_INVALID, "workspace too small (%zu < %zu)", workspace_bytes, need);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  if (dtype == SPF_DTYPE_BF16)
    return bs_estimate_impl(reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
                            n_q_heads, n_kv_heads, seq_len, head_dim, head_ids, n_heads, k_b, block_size,
                            tile_offsets, tile_starts, ws, st);
  if (dtype == SPF_DTYPE_F32)
    return bs_estimate_impl(reinterpret_cast<const float*>(q), reinterpret_cast<const float*>(k), n_q_heads,
                            n_kv_heads, seq_len, head_dim, head_ids, n_heads, k_b, block_size, tile_offsets,
                            tile_starts, ws, st);
  return set_error(SPF_ERR_INVALID, "unknown dtype %d", dtype);
}

}  // extern "C"
