// estimate_vs_tc.cu -- Vertical-Slash online estimation on the tensor cores
// (the production path of spf_vs_estimate, mode SPF_VS_FAST).
//
// Computes the same quantities as estimator.py:82-114 -- probabilities of the
// last 64 query rows against every key (scale 1/sqrt(d), causal), rounded to
// fp32, summed per key column (vertical) and per diagonal offset (slash) --
// but with the q.k scores on tcgen05 (bf16 operands, fp32 accumulate in TMEM)
// instead of fp64.  The index sets are then certified per head (see
// vs_topk_certify_kernel): if the k-th / (k+1)-th boundary of either top-k is
// closer than the error model of this path, the head is flagged and the
// caller recomputes it on the fp64 path (estimate.cu), so the selected sets
// are those of the reference either way.
//
// Work decomposition:
//   * group  = one kv head and up to 4 of its q-heads being estimated (GQA
//              fusion: the 4 x 64 tail rows share every K tile read);
//   * tile   = 128 consecutive keys (one TMA box per 64-wide d atom);
//   * CTA    = (group, contiguous chunk of tiles); one CTA per SM.
//   Pass 1 (rows in TMEM lanes): S = Qtail K^T, M=128 (two heads) x N=128 keys,
//          per-row online (max, sum exp) -> per-chunk partial row stats.
//   combine: per-row max / sum over chunks (fp64), inverse sums, per-head
//          error scale.
//   Pass 2 (keys in TMEM lanes): S^T = K Qtail^T, M=128 keys x N=64*heads,
//          p = 2^((s-m)*c) / l per element; vertical[j] = in-thread sum over
//          the 64 rows; slash: warp-shuffle diagonal sums, combined across
//          warps in smem and across tiles by (exactly two-term, hence
//          order-free) fp64 atomics into a zeroed vector.
// Warp roles: warp 0 = TMA producer, warp 1 = MMA issuer + TMEM owner,
// warps 2..9 = epilogue (two warps per TMEM lane quarter).
#include <cuda_bf16.h>

#include "spf.h"
#include "spf_internal.h"
#include "spf_ptx.cuh"
#include "cluster_topk.cuh"

namespace spf {
namespace {

constexpr int kTailRows = 64;     // last_q supported by this path
constexpr int kMaxMembers = 4;    // q-heads per group
constexpr int kKeys = 128;        // keys per tile (UMMA M of pass 2, N of pass 1)
constexpr int kStages = 4;        // K tile stages
constexpr int kStatWarps = 2;     // pass 1: warps taking the per-dimension max |k| of each K tile
constexpr int kThreads = 320 + 32 * kStatWarps;  // loader, MMA, 8 epilogue warps, stat warps
constexpr int kEpiThreads = 256;  // warps 2..9
constexpr int kStatWarp = 10;     // first stat warp (pass 1: K statistics for the score error bound)
constexpr int kGroupRows = kMaxMembers * kTailRows;

struct TcArgs {
  int S, Hq, Hkv, hpk, gpk, n_heads, n_tiles, n_chunks;
  const int32_t* head_ids;
  float c_hi, c_lo;  // scale * log2(e) as an unevaluated float pair
  // pass 1 out / combine in
  float* st_m;       // [groups][chunks][256]  mc = fp32(row max * c)
  double* st_l;      // [groups][chunks][256]
  float* st_amax;    // [groups][chunks][256]
  // pass 1 out: max_j |k_jc| per group and dimension (bf16 bits in the low half; zeroed first)
  uint32_t* kabs;             // [groups][kD]
  // combine out
  float* row_marg;            // [n_heads][64]: 2 * score-error bound in log2 units (fp64 path's skip margin)
  int32_t* hopeless;          // [n_heads]: 1 = the bound is too loose to certify: straight to the fp64 path
  int32_t* flags;             // [n_heads]: 1 = the fp64 path re-estimates the head
  int uncertified;            // test hook: no hopeless short-cut, no re-estimation
  // combine out / pass 2 in
  float* row_m;      // [groups][256]  mc of the global row max
  float* row_il;     // [groups][256]
  // pass 2 out
  double* vscore;    // [n_heads][S]
  double* sscore;    // [n_heads][S]  (zeroed before pass 2)
  float* tau;        // [n_heads] eta: bound on the relative error of every score-vector entry
  // for the exact fallback's tile skipping
  float* tile_max;   // [n_heads][n_tiles][64] raw row max per 128-key tile (rows fastest)
  float* row_mc;     // [n_heads][64] mc per slot
  uint8_t* live;     // [groups][n_tiles] pass-2 tile holds a probability that is not flushed to 0
};

// A tile whose largest exponent y = fma(x_max, c, -mc) is below kDeadExp contributes exactly
// nothing: ex2.approx.ftz flushes 2^y < 2^-126 to +0.  One unit of margin covers the last-bit
// difference between the pass-1 and pass-2 accumulation orders of the same dot product.
constexpr float kDeadExp = -127.f;
constexpr int kMaxList = 2048;  // live-tile list capacity per pass-2 CTA (more tiles: no skipping)

struct TcCtrl {
  uint64_t q_full;
  uint64_t k_full[kStages];
  uint64_t k_empty[kStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint32_t tmem_base;
  int nh;
  int n_list;
  int slot[kMaxMembers];
  int head[kMaxMembers];
};

template <int kD>
struct TcLayout {
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQAtom = kGroupRows * 128;  // bytes per 64-wide d atom of the tail rows
  static constexpr int kKAtom = kKeys * 128;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kAtoms * kQAtom;
  static constexpr int kStageBytes = kAtoms * kKAtom;
  static constexpr int kOffRow = kOffK + kStages * kStageBytes;      // pass 2: float2 (m, il) [256]
  static constexpr int kOffDiag = kOffRow + kGroupRows * 8;          // pass 2: float [2][4 members][4 wk][3][32]
  static constexpr int kDiagBytes = 2 * kMaxMembers * 4 * 3 * 32 * 4;
  static constexpr int kOffList = kOffDiag + kDiagBytes;             // pass 2: live tile list
  static constexpr int kOffCtrl = kOffList + kMaxList * 4;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(TcCtrl);
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// Members of group gy: the (4*sub .. 4*sub+3)-th slots (ascending) whose head maps to kv head gy / gpk.
// Group gy's members (q-heads of one kv head, at most kMaxMembers, in list order): slot = index
// in the head list, head = q-head id.  Called by a whole warp: 32 list entries per round with
// a ballot (one serial pass of dependent loads per entry cost ~10 us per CTA); lane 0 stores.
__device__ int group_members(const TcArgs& a, int gy, int* slot, int* head) {
  const int lane = threadIdx.x & 31;
  const int kvh = gy / a.gpk, sub = gy % a.gpk;
  const int lo = kMaxMembers * sub, hi = kMaxMembers * (sub + 1);
  int seen = 0;
  for (int base = 0; base < a.n_heads; base += 32) {
    const int i = base + lane;
    const int h = i < a.n_heads ? (a.head_ids ? a.head_ids[i] : i) : -1;
    const bool match = h >= 0 && h / a.hpk == kvh;
    const unsigned m = __ballot_sync(0xffffffffu, match);
    const int rank = seen + __popc(m & ((1u << lane) - 1u));
    if (match && rank >= lo && rank < hi) {
      slot[rank - lo] = i;
      head[rank - lo] = h;
    }
    seen += __popc(m);
  }
  return min(kMaxMembers, max(0, seen - lo));
}

template <int kD, int kPass>
__global__ void __launch_bounds__(kThreads, 1)
    vs_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k, const TcArgs a) {
  using L = TcLayout<kD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  TcCtrl* ctrl = reinterpret_cast<TcCtrl*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gy = blockIdx.y, chunk = blockIdx.x;
  const int S = a.S;
  const int t_begin = (int)((int64_t)chunk * a.n_tiles / a.n_chunks);
  const int t_end = (int)((int64_t)(chunk + 1) * a.n_tiles / a.n_chunks);
  const int kvh = gy / a.gpk;

  if (warp == 0) {
    const int nh = group_members(a, gy, ctrl->slot, ctrl->head);
    if (lane == 0) ctrl->nh = nh;
  }
  if (threadIdx.x == 0) {
    if ((sbase & 1023u) != 0) {
      printf("spf: dynamic smem not 1024-aligned\n");
      __trap();
    }
    mbar_init(&ctrl->q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&ctrl->k_full[s], 1);
      mbar_init(&ctrl->k_empty[s], kPass == 1 ? 1 + kStatWarps : 1);  // pass 1: MMA commit + K-statistics warps
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctrl->acc_full[b], 1);
      mbar_init(&ctrl->acc_empty[b], kEpiThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nh = ctrl->nh;
  if (nh == 0 || chunk >= a.n_tiles) return;  // CTA-uniform, before TMEM allocation
  if (kPass == 2) {  // every member goes to the fp64 path anyway: no pass 2 for this group
    bool all_hopeless = true;
    for (int mm = 0; mm < nh; ++mm) all_hopeless = all_hopeless && a.hopeless[ctrl->slot[mm]] != 0;
    if (all_hopeless) return;
  }
  if (kPass == 2) {
    // row stats per member pair and tail row: {-mc(2p), -mc(2p+1), 1/l(2p), 1/l(2p+1)}
    float4* rs = reinterpret_cast<float4*>(smem + L::kOffRow);
    for (int r = threadIdx.x; r < 2 * kTailRows; r += kThreads) {
      const int pr = r / kTailRows, i = r % kTailRows;
      const int64_t b0 = (int64_t)gy * kGroupRows + (2 * pr) * kTailRows + i, b1 = b0 + kTailRows;
      rs[r] = make_float4(-a.row_m[b0], -a.row_m[b1], a.row_il[b0], a.row_il[b1]);
    }
  }
  if (warp == 1) tmem_alloc(&ctrl->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctrl->tmem_base;
  // Pass 1: chunk c takes tiles T-1-c, T-1-c-n_chunks, ... (interleaved, highest first), so
  // every chunk meets the diagonal region first, sets its running row max early and skips
  // the exponentials of the tiles that flush to zero -- balanced across chunks.  Pass 2: the
  // group's live tiles (a.live) are split evenly over its chunks.
  int n_tiles_cta = kPass == 1 ? (chunk < a.n_tiles ? (a.n_tiles - chunk + a.n_chunks - 1) / a.n_chunks : 0)
                               : t_end - t_begin;
  int* s_list = reinterpret_cast<int*>(smem + L::kOffList);
  bool use_list = false;
  if (kPass == 2) {
    if (warp == 0) {
      const uint8_t* lv_g = a.live + (int64_t)gy * a.n_tiles;
      int nl = 0;
      for (int b = 0; b < a.n_tiles; b += 32) nl += __popc(__ballot_sync(0xffffffffu, b + lane < a.n_tiles && lv_g[b + lane]));
      const int lo = (int)((int64_t)chunk * nl / a.n_chunks), hi = (int)((int64_t)(chunk + 1) * nl / a.n_chunks);
      int n = -1;
      if (hi - lo <= kMaxList) {
        int rank = 0;
        n = 0;
        for (int b = 0; b < a.n_tiles && rank < hi; b += 32) {
          const int t = b + lane;
          const bool lv = t < a.n_tiles && lv_g[t];
          const unsigned m = __ballot_sync(0xffffffffu, lv);
          const int r = rank + __popc(m & ((1u << lane) - 1));
          if (lv && r >= lo && r < hi) s_list[r - lo] = t;
          rank += __popc(m);
        }
        n = hi - lo;
      }
      if (lane == 0) ctrl->n_list = n;
    }
    __syncthreads();
    if (ctrl->n_list >= 0) {
      use_list = true;
      n_tiles_cta = ctrl->n_list;
    }
  }
  auto tile_of = [&](int t) {
    return kPass == 1 ? a.n_tiles - 1 - (chunk + t * a.n_chunks) : (use_list ? s_list[t] : t_begin + t);
  };

  if (warp == 0) {
    // =============================== TMA producer ===============================
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      mbar_arrive_expect_tx(&ctrl->q_full, (uint32_t)(nh * L::kAtoms * kTailRows * 128));
      for (int mm = 0; mm < nh; ++mm)
        for (int at = 0; at < L::kAtoms; ++at)
          tma_load_3d(smem + L::kOffQ + at * L::kQAtom + mm * (kTailRows * 128), &tm_q, &ctrl->q_full, at * 64,
                      S - kTailRows, ctrl->head[mm]);
      for (int t = 0; t < n_tiles_cta; ++t) {
        const int st = t % kStages;
        mbar_wait(&ctrl->k_empty[st], ((t / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctrl->k_full[st], (uint32_t)L::kStageBytes);
        uint8_t* kst = smem + L::kOffK + st * L::kStageBytes;
        for (int at = 0; at < L::kAtoms; ++at)
          tma_load_3d(kst + at * L::kKAtom, &tm_k, &ctrl->k_full[st], at * 64, tile_of(t) * kKeys, kvh);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =============================== MMA issuer =================================
    if (lane == 0) {
      const uint32_t q_addr = sbase + L::kOffQ;
      mbar_wait(&ctrl->q_full, 0);
      tc_fence_after();
      const int nb = (nh + 1) / 2;
      for (int t = 0; t < n_tiles_cta; ++t) {
        const int st = t % kStages, buf = t & 1;
        mbar_wait(&ctrl->k_full[st], (t / kStages) & 1);
        mbar_wait(&ctrl->acc_empty[buf], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = sbase + L::kOffK + st * L::kStageBytes;
        if (kPass == 1) {
          constexpr uint32_t idesc = umma_idesc_bf16(128, kKeys, 0, 0);
          for (int b = 0; b < nb; ++b) {
#pragma unroll
            for (int ks = 0; ks < kD / 16; ++ks) {
              const int at = ks >> 2;
              const uint32_t koff = (ks & 3) * 32;
              const uint64_t ad = umma_desc_sw128(q_addr + at * L::kQAtom + b * (128 * 128) + koff, 0, 1024);
              const uint64_t bd = umma_desc_sw128(k_addr + at * L::kKAtom + koff, 0, 1024);
              mma_bf16_ss(tmem + buf * 256 + b * 128, ad, bd, idesc, ks > 0 ? 1u : 0u);
            }
          }
        } else {
          const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)(nh * kTailRows), 0, 0);
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks) {
            const int at = ks >> 2;
            const uint32_t koff = (ks & 3) * 32;
            const uint64_t ad = umma_desc_sw128(k_addr + at * L::kKAtom + koff, 0, 1024);
            const uint64_t bd = umma_desc_sw128(q_addr + at * L::kQAtom + koff, 0, 1024);
            mma_bf16_ss(tmem + buf * 256, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        }
        mma_commit(&ctrl->k_empty[st]);
        mma_commit(&ctrl->acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= kStatWarp) {
    // ======================= K statistics (pass 1 only) =========================
    // max_j |k_jc| per dimension c over the group's keys: the input of the bound on the
    // tensor-core score error (vs_tc_combine_kernel).  Stat warp w takes keys
    // [w * kKeys / kStatWarps, ...) of every staged SW128 tile; lane l owns the 8 dims of
    // logical 16-byte chunk (l & 15) and half (l >> 4) of the warp's keys (each 128-byte row
    // holds 64 dims of one key, chunks permuted by row & 7).
    if (kPass == 1) {
      constexpr int kRowsPerHalf = kKeys / kStatWarps / 2;
      const int cc = lane & 15, at = cc >> 3, c = cc & 7;
      const int kh = (warp - kStatWarp) * 2 + (lane >> 4);
      uint32_t amx[4] = {0u, 0u, 0u, 0u};  // |k| maxima of the lane's 8 dims, bf16x2
      for (int t = 0; t < n_tiles_cta; ++t) {
        const int st = t % kStages;
        mbar_wait(&ctrl->k_full[st], (t / kStages) & 1);
        const uint8_t* kst = smem + L::kOffK + st * L::kStageBytes + at * L::kKAtom;
        // keys past S are TMA zero fill: they cannot raise a maximum
#pragma unroll 8
        for (int r = kh * kRowsPerHalf; r < (kh + 1) * kRowsPerHalf; ++r) {
          const uint4 x = *reinterpret_cast<const uint4*>(kst + r * 128 + ((c ^ (r & 7)) << 4));
          // bf16 magnitudes order like their bit patterns: per-half unsigned max
          amx[0] = __vmaxu2(amx[0], x.x & 0x7fff7fffu);
          amx[1] = __vmaxu2(amx[1], x.y & 0x7fff7fffu);
          amx[2] = __vmaxu2(amx[2], x.z & 0x7fff7fffu);
          amx[3] = __vmaxu2(amx[3], x.w & 0x7fff7fffu);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctrl->k_empty[st]);  // K consumed: the stage may be refilled
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) amx[w] = __vmaxu2(amx[w], __shfl_xor_sync(0xffffffffu, amx[w], 16));
      if ((lane >> 4) == 0 && n_tiles_cta > 0) {
        uint32_t* dst = a.kabs + (int64_t)gy * kD + at * 64 + c * 8;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          atomicMax(dst + 2 * w, amx[w] & 0xffffu);
          atomicMax(dst + 2 * w + 1, amx[w] >> 16);
        }
      }
    }
  } else {
    // =============================== epilogue warps =============================
    // Exponents are formed as y = s*c - mc with one FFMA, c = scale*log2(e) and
    // mc = fp32(m*c) for the running row max m.  Pass 2 reuses the very mc the
    // row sum was taken against, so the rounding of mc cancels between p's
    // numerator and l; packed f32x2 ops handle two values per instruction.
    const int e = warp - 2;
    const int quarter = warp & 3;        // TMEM lane quarter this warp may access
    const int half = e >> 2;             // which pair of members
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float c = a.c_hi;
    const uint64_t c2 = pack_f32x2(c, c);
    if (kPass == 1) {
      const int row = quarter * 32 + lane;          // row of M-block `half`
      const int mm = 2 * half + (row >> 6);         // member (warp-uniform)
      const int i = row & 63;
      const int abs_i = S - kTailRows + i;
      const bool active = mm < nh;
      float m_run = -INFINITY, mc_run = -INFINITY, amax = 0.f;
      double l_run = 0.0;
      for (int t = 0; t < n_tiles_cta; ++t) {
        const int buf = t & 1;
        const int tile = tile_of(t);
        const int tile0 = tile * kKeys;
        mbar_wait(&ctrl->acc_full[buf], (t >> 1) & 1);
        tc_fence_after();
        if (active) {
          uint32_t x[kKeys];
          tmem_ld32x32b_x64(tmem + lane_off + buf * 256 + half * 128, x);
          tmem_ld32x32b_x64(tmem + lane_off + buf * 256 + half * 128 + 64, x + 64);
          tmem_wait_ld();
          tc_fence_before();
          if (lane == 0) mbar_arrive(&ctrl->acc_empty[buf]);
          const int n_valid = min(kKeys, abs_i - tile0 + 1);  // keys tile0 .. abs_i (abs_i < S)
          float tmax = -INFINITY, tmin = INFINITY;
          if (n_valid >= kKeys) {
            float mx0 = -INFINITY, mx1 = -INFINITY, mn0 = INFINITY, mn1 = INFINITY;
#pragma unroll
            for (int j = 0; j < kKeys; j += 4) {
              mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
              mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
              mn0 = fmin3(mn0, u2f(x[j]), u2f(x[j + 1]));
              mn1 = fmin3(mn1, u2f(x[j + 2]), u2f(x[j + 3]));
            }
            tmax = fmaxf(mx0, mx1);
            tmin = fminf(mn0, mn1);
          } else {
#pragma unroll
            for (int j = 0; j < kKeys; ++j) {
              const bool ok = j < n_valid;
              tmax = ok ? fmaxf(tmax, u2f(x[j])) : tmax;
              tmin = ok ? fminf(tmin, u2f(x[j])) : tmin;
              x[j] = ok ? x[j] : 0xf149f2cau;  // -1e30 (finite): 2^(y) underflows to 0
            }
          }
          a.tile_max[((int64_t)ctrl->slot[mm] * a.n_tiles + tile) * kTailRows + i] = tmax;
          // every exponent of this row below the flush threshold: the tile adds exactly 0
          const bool dead = n_valid <= 0 || (m_run != -INFINITY && tmax <= m_run && fmaf(tmax, c, -mc_run) < kDeadExp);
          const bool warp_dead = __all_sync(0xffffffffu, dead);
          if (n_valid > 0) {
            amax = fmax3(amax, fabsf(tmax), fabsf(tmin));
            if (tmax > m_run) {
              const float mc_new = tmax * c;
              if (m_run != -INFINITY) l_run *= exp2((double)mc_run - (double)mc_new);
              m_run = tmax;
              mc_run = mc_new;
            }
            if (!warp_dead) {
              const uint64_t nm2 = pack_f32x2(-mc_run, -mc_run);
              uint64_t s0 = 0, s1 = 0;
#pragma unroll
              for (int j = 0; j < kKeys; j += 4) {
                float y0, y1, y2, y3;
                unpack_f32x2(ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, nm2), y0, y1);
                unpack_f32x2(ffma2(pack_f32x2(u2f(x[j + 2]), u2f(x[j + 3])), c2, nm2), y2, y3);
                s0 = fadd2(s0, pack_f32x2(ex2_approx(y0), ex2_approx(y1)));
                s1 = fadd2(s1, pack_f32x2(ex2_approx(y2), ex2_approx(y3)));
              }
              float a0, a1;
              unpack_f32x2(fadd2(s0, s1), a0, a1);
              l_run += (double)(a0 + a1);
            }
          }
        } else {
          tc_fence_before();
          if (lane == 0) mbar_arrive(&ctrl->acc_empty[buf]);
        }
      }
      if (active) {
        const int64_t o = ((int64_t)gy * a.n_chunks + chunk) * kGroupRows + mm * kTailRows + i;
        a.st_m[o] = mc_run;
        a.st_l[o] = l_run;
        a.st_amax[o] = amax;
      }
    } else {
      // row stats of this warp's member pair: {-mc(2h), -mc(2h+1), 1/l(2h), 1/l(2h+1)} per tail row
      const float4* rs = reinterpret_cast<const float4*>(smem + L::kOffRow) + half * kTailRows;
      float* diag = reinterpret_cast<float*>(smem + L::kOffDiag);
      const int m0 = 2 * half, m1 = 2 * half + 1;
      const bool act = m0 < nh;  // warp-uniform
      const uint32_t col0 = (uint32_t)(m0 * kTailRows);
      const uint32_t col1 = (uint32_t)((m1 < nh ? m1 : m0) * kTailRows);
      for (int t = 0; t < n_tiles_cta; ++t) {
        const int buf = t & 1;
        const int tile0 = tile_of(t) * kKeys;
        const int j = tile0 + quarter * 32 + lane;  // this thread's key
        mbar_wait(&ctrl->acc_full[buf], (t >> 1) & 1);
        tc_fence_after();
        // partial diagonal sums: [pair][wk][95][2 members]
        float2* dbuf = reinterpret_cast<float2*>(diag + (t & 1) * (2 * 4 * 96 * 2)) + (half * 4 + quarter) * 96;
        if (act) {
          // row i sees key j iff j <= S - 64 + i; only the last tiles have masked rows
          const int i_min = j - (S - kTailRows);
          const bool full = tile0 + kKeys - 1 <= S - kTailRows;  // CTA-uniform
          uint64_t vs0 = 0, vs1 = 0, acc = 0;
#pragma unroll
          for (int seg = 0; seg < 2; ++seg) {  // two 32-row halves keep the x registers at 64
            uint32_t x0[32], x1[32];
            tmem_ld32x32b_x32(tmem + lane_off + buf * 256 + col0 + seg * 32, x0);
            tmem_ld32x32b_x32(tmem + lane_off + buf * 256 + col1 + seg * 32, x1);
            tmem_wait_ld();
            if (seg == 1) {
              tc_fence_before();
              if (lane == 0) mbar_arrive(&ctrl->acc_empty[buf]);
            }
#pragma unroll
            for (int ii = 0; ii < 32; ++ii) {
              const int i = seg * 32 + ii;
              const float4 r = rs[i];
              float y0, y1;
              unpack_f32x2(ffma2(pack_f32x2(u2f(x0[ii]), u2f(x1[ii])), c2, pack_f32x2(r.x, r.y)), y0, y1);
              uint64_t pp = fmul2(pack_f32x2(ex2_approx(y0), ex2_approx(y1)), pack_f32x2(r.z, r.w));
              if (!full) pp = (i >= i_min) ? pp : 0ull;
              if (i & 1) vs1 = fadd2(vs1, pp); else vs0 = fadd2(vs0, pp);
              // systolic diagonal sums: lane l holds diagonal (key j0 + l - i) of both members
              acc = fadd2(acc, pp);
              if (lane == 31) {
                dbuf[94 - i] = *reinterpret_cast<const float2*>(&acc);
                acc = 0ull;
              }
              acc = __shfl_sync(0xffffffffu, acc, (lane + 31) & 31);
            }
          }
          if (lane >= 1) dbuf[lane - 1] = *reinterpret_cast<const float2*>(&acc);
          float v0a, v1a, v0b, v1b;
          unpack_f32x2(vs0, v0a, v1a);
          unpack_f32x2(vs1, v0b, v1b);
          if (j < S) {
            a.vscore[(int64_t)ctrl->slot[m0] * S + j] = (double)(v0a + v0b);
            if (m1 < nh) a.vscore[(int64_t)ctrl->slot[m1] * S + j] = (double)(v1a + v1b);
          }
        } else {
          tc_fence_before();
          if (lane == 0) mbar_arrive(&ctrl->acc_empty[buf]);
        }
        named_bar_sync(1, kEpiThreads);
        // combine: diagonal c = tile0 + cl (its key at row 0), cl in [-63, 127]; offset o = S - 64 - c.
        // Warp-chunk wk holds the diagonals cl in [32 wk - 63, 32 wk + 31] at index cl - 32 wk + 63.
        const float* dsum = diag + (t & 1) * (2 * 4 * 96 * 2);
        const int et = threadIdx.x - 64;
        for (int idx = et; idx < nh * 191; idx += kEpiThreads) {
          const int mm = idx / 191;
          const int cl = idx % 191 - 63;
          double sum = 0.0;
#pragma unroll
          for (int wk = 0; wk < 4; ++wk) {
            const int k = cl - 32 * wk + 63;
            if (k >= 0 && k <= 94) sum += (double)dsum[(((mm >> 1) * 4 + wk) * 96 + k) * 2 + (mm & 1)];
          }
          const int cd = tile0 + cl;
          const int o = S - kTailRows - cd;
          if (o < 0 || o >= S) continue;
          double* dst = a.sscore + (int64_t)ctrl->slot[mm] * S + o;
          if (cl >= 0 && cl <= kKeys - kTailRows)
            *dst = sum;  // the whole diagonal lies in this tile
          else
            atomicAdd(dst, sum);  // exactly two tiles contribute: order-free
        }
        // the next tile writes the other diag buffer; one barrier per tile keeps the reuse distance at 2
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Error model of the tensor-core scores (no tcgen05 accumulation spec is published, so the
// bound assumes the weakest behaviour consistent with fp32 accumulation): bf16 x bf16
// products are exact; each K=16 MMA step adds its 16 products to the accumulator after
// aligning all 17 addends to the largest with at least 24 kept bits (truncation), then
// rounds (or truncates) to fp32.  One step errs by <= 17 * 2^-23 * max addend + 2^-23 * |sum|
// <= 18 * 2^-23 * (sum of |products| so far), so over d/16 steps
//     |fl(q.k) - q.k| <= gamma * sum_c |q_c| |k_c|,   gamma = (d/16) * 18 * 2^-23,
// and sum_c |q_c||k_c| <= sum_c |q_c| * max_j |k_jc| (the per-dimension maxima of pass 1).
// The bound is rigorous under that model, whatever the cancellation in q.k (it scales with
// sum |q_c k_c|, not with |q.k|), and it is the same for pass 2's transposed product.
template <int kD>
__device__ __forceinline__ double score_gamma() { return (kD / 16) * 18.0 * 0x1p-23; }

// Per-row combine of the chunk partials (fp64); per row the score-error bound E_i and the
// fp64 path's skip margin; per head the certification bound eta and the hopeless flag.
//
// eta bounds the relative error of every vertical / slash entry of the fast path against
// the reference's fp64 values (estimator.py:100-110 with tensor.py:78's fp32 rounding):
//   p = exp(s_ij) / sum_k exp(s_ik): numerator and normaliser each off by <= e^(c' E_i) with
//   c' = scale (nats per raw unit)                                -> expm1(2 scale E_max)
//   the fp32 constant c_hi = fl(scale log2 e) scales every exponent: |x| c 2^-24 per side
//                                                                  -> 2 ln2 c amax 2^-24
//   ex2.approx (2^-21), fp32 partial row sums (2^-19), 1/l and p roundings, the
//   reference's own fp32 rounding of p, fp32 partial column / diagonal sums (2^-18)
//                                                                  -> 2^-16 (with margin)
// Values flushed to zero by ex2.approx.ftz (true p < 2^-126) are the absolute term of the
// certification (cluster_topk.cuh).
constexpr double kHopelessEta = 0x1p-12;  // larger: no top-k boundary of a long sequence is that wide
template <int kD>
__global__ void __launch_bounds__(kGroupRows) vs_tc_combine_kernel(const TcArgs a, const __nv_bfloat16* __restrict__ q) {
  __shared__ int slot[kMaxMembers], head[kMaxMembers], nh_s;
  __shared__ float amax_s[kGroupRows];
  __shared__ float err_s[kGroupRows];
  __shared__ float kabs_s[kD];
  const int gy = blockIdx.x;
  if (threadIdx.x < 32) {
    const int n = group_members(a, gy, slot, head);
    if (threadIdx.x == 0) nh_s = n;
  }
  for (int c = threadIdx.x; c < kD; c += blockDim.x)
    kabs_s[c] = __uint_as_float(a.kabs[(int64_t)gy * kD + c] << 16);
  __syncthreads();
  const int nh = nh_s;
  const int r = threadIdx.x;
  const int mm = r / kTailRows;
  const double c64 = (double)a.c_hi + (double)a.c_lo;
  float amax = 0.f, err = 0.f;
  if (mm < nh) {
    float m = -INFINITY;
    // unrolled: the chunk partials' loads are independent (one round trip per 8, not per chunk)
#pragma unroll 8
    for (int c = 0; c < a.n_chunks; ++c) {
      const int64_t o = ((int64_t)gy * a.n_chunks + c) * kGroupRows + r;
      if (a.st_l[o] > 0.0) m = fmaxf(m, a.st_m[o]);
    }
    double l = 0.0;  // st_m holds mc = fp32(m * c): rescale in the exponent domain the sums were taken in
#pragma unroll 8
    for (int c = 0; c < a.n_chunks; ++c) {
      const int64_t o = ((int64_t)gy * a.n_chunks + c) * kGroupRows + r;
      const double lc = a.st_l[o];
      if (lc > 0.0) l += lc * exp2((double)a.st_m[o] - (double)m);
      amax = fmaxf(amax, a.st_amax[o]);
    }
    a.row_m[(int64_t)gy * kGroupRows + r] = m;
    a.row_il[(int64_t)gy * kGroupRows + r] = (float)(1.0 / l);
    const int i = r % kTailRows;
    a.row_mc[(int64_t)slot[mm] * kTailRows + i] = m;
    // E_i = gamma * sum_c |q_ic| max_j |k_jc| (fp64: exact products of bf16 values, tiny sum error)
    // (fp32: bf16 x bf16 products are exact, kD positive terms err by < kD 2^-24 relative)
    const int4* qr = reinterpret_cast<const int4*>(q + ((int64_t)head[mm] * a.S + (a.S - kTailRows + i)) * kD);
    float sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int c8 = 0; c8 < kD / 8; ++c8) {
      const int4 x = __ldg(qr + c8);
      const uint32_t w[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t ab = w[e] & 0x7fff7fffu;
        sa[e] = fmaf(__uint_as_float(ab << 16), kabs_s[c8 * 8 + 2 * e], sa[e]);
        sa[e] = fmaf(__uint_as_float(ab & 0xffff0000u), kabs_s[c8 * 8 + 2 * e + 1], sa[e]);
      }
    }
    const double sabs = ((double)sa[0] + sa[1]) + ((double)sa[2] + sa[3]);
    const double e_i = score_gamma<kD>() * sabs * (1.0 + 0x1p-15);
    err = (float)(e_i * (1.0 + 0x1p-20));
    // fp64 path: an item is skipped when its tensor-core scores sit > 151 + marg (log2 units)
    // below the row max; the true scores can be E_i higher and the true max E_i lower
    a.row_marg[(int64_t)slot[mm] * kTailRows + i] = (float)(2.0 * e_i * c64 * (1.0 + 0x1p-20));
  }
  amax_s[r] = amax;
  err_s[r] = err;
  __syncthreads();
  if (r < nh) {
    float mx = 0.f, emax = 0.f;
#pragma unroll 16
    for (int i = 0; i < kTailRows; ++i) {
      mx = fmaxf(mx, amax_s[r * kTailRows + i]);
      emax = fmaxf(emax, err_s[r * kTailRows + i]);
    }
    const double scale = c64 * 0.6931471805599453;  // nats per raw score unit
    const double eta = expm1(2.0 * scale * (double)emax) + 2.0 * 0.6931471805599453 * c64 * (double)mx * 0x1p-24 +
                       0x1p-16;
    a.tau[slot[r]] = (float)(eta * (1.0 + 0x1p-20));
    const int hopeless = (eta > kHopelessEta && !a.uncertified) ? 1 : 0;
    a.hopeless[slot[r]] = hopeless;
    if (hopeless) a.flags[slot[r]] = 1;  // straight to the fp64 path
  }
}

// Pass-2 tile liveness per group: a tile is live if any member row has an exponent at or
// above kDeadExp there (tile_max and the final mc from pass 1 / combine).  Dead tiles'
// vertical scores are written here (zeros); their slash contributions are zero already.
__global__ void __launch_bounds__(256) vs_tc_live_kernel(const TcArgs a) {
  // 32 tiles per CTA; the 8 warps split the (member, row) pairs and OR their verdicts
  __shared__ int slot[kMaxMembers], head[kMaxMembers], nh_s;
  __shared__ int lv[32];
  const int gy = blockIdx.y;
  if (threadIdx.x < 32) {
    const int n = group_members(a, gy, slot, head);
    if (threadIdx.x == 0) nh_s = n;
  }
  if (threadIdx.x < 32) lv[threadIdx.x] = 0;
  __syncthreads();
  const int nh = nh_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // warp w: tiles 4w .. 4w+3 of the CTA's 32; lanes read 32 consecutive rows (coalesced)
  for (int u = 4 * w; u < 4 * w + 4; ++u) {
    const int tu = blockIdx.x * 32 + u;
    if (tu >= a.n_tiles) break;
    bool live = false;
    for (int r = lane; r < nh * kTailRows; r += 32) {
      const int mm = r / kTailRows, i = r % kTailRows;
      live |= fmaf(a.tile_max[((int64_t)slot[mm] * a.n_tiles + tu) * kTailRows + i], a.c_hi,
                   -a.row_mc[(int64_t)slot[mm] * kTailRows + i]) >= kDeadExp;
    }
    const bool any = __any_sync(0xffffffffu, live);
    if (lane == 0) lv[u] = any ? 1 : 0;
  }
  __syncthreads();
  const int t = blockIdx.x * 32 + lane;
  if (threadIdx.x < 32 && t < a.n_tiles) a.live[(int64_t)gy * a.n_tiles + t] = (uint8_t)lv[threadIdx.x];
  for (int u = 0; u < 32; ++u) {  // zero the vertical scores of the dead tiles (coalesced)
    const int tu = blockIdx.x * 32 + u;
    if (tu >= a.n_tiles || lv[u]) continue;
    for (int x = threadIdx.x; x < nh * kKeys; x += 256) {
      const int mm = x / kKeys, j = tu * kKeys + x % kKeys;
      if (j < a.S) a.vscore[(int64_t)slot[mm] * a.S + j] = 0.0;
    }
  }
}

// Top-k (estimator.py:59-79) of the fp64 score vectors plus certification of the
// selected set against the error threshold tau: flag the head when the
// boundary (k-th vs (k+1)-th, the k-th vs (k-1)-th when index 0 must be forced,
// or index 0 vs the k-th) is closer than tau * (k-th value), or the k-th value
// ties.  One cluster of kTopkCl CTAs per vector (cluster_topk.cuh).
constexpr int kTopkThreads = 256;
constexpr int kTopkCl = 8;

__global__ void __cluster_dims__(kTopkCl, 1, 1) __launch_bounds__(kTopkThreads)
    vs_topk_certify_kernel(const double* __restrict__ vscore, const double* __restrict__ sscore, int S, int k_v,
                           int k_s, const float* __restrict__ tau, const int32_t* __restrict__ hopeless,
                           int32_t* __restrict__ vert_out, int32_t* __restrict__ slash_out,
                           int32_t* __restrict__ uncertain) {
  using TK = ClusterTopK<kTopkThreads, kTopkCl>;
  __shared__ typename TK::Storage sm;
  const int hi = blockIdx.y;
  if (hopeless[hi]) return;  // written before this launch: cluster-uniform
  if (blockIdx.z == 0)
    TK::run(sm, vscore + (int64_t)hi * S, S, k_v, false, vert_out + (int64_t)hi * k_v, tau + hi, uncertain + hi);
  else
    TK::run(sm, sscore + (int64_t)hi * S, S, k_s, true, slash_out + (int64_t)hi * k_s, tau + hi, uncertain + hi);
}

template <int kD>
int vs_fast_impl(const __nv_bfloat16* q, const __nv_bfloat16* k, int Hq, int Hkv, int S, const int32_t* head_ids,
                 int n_heads, int k_v, int k_s, int32_t* vout, int32_t* sout, double* vscore, double* sscore,
                 int32_t* uncertain, bool uncertified, uint8_t* ws, cudaStream_t st) {
  using L = TcLayout<kD>;
  TcArgs a{};
  a.S = S;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.hpk = Hq / Hkv;
  a.gpk = (a.hpk + kMaxMembers - 1) / kMaxMembers;
  a.n_heads = n_heads;
  a.head_ids = head_ids;
  a.n_tiles = (S + kKeys - 1) / kKeys;
  const int n_groups = Hkv * a.gpk;
  // active groups are at most min(n_groups, ceil(n_heads/1)); size chunks for ~one CTA per SM
  const int active = min(n_groups, n_heads);
  a.n_chunks = max(1, min(a.n_tiles, 148 / active));  // one wave: at most one CTA per SM
  const double c64 = 1.4426950408889634 / sqrt((double)kD);
  a.c_hi = (float)c64;
  a.c_lo = (float)(c64 - (double)a.c_hi);
  auto take = [&](size_t bytes) {
    uint8_t* p = ws;
    ws += (bytes + 255) & ~size_t(255);
    return p;
  };
  const size_t part = (size_t)n_groups * a.n_chunks * kGroupRows;
  a.st_m = reinterpret_cast<float*>(take(part * 4));
  a.st_l = reinterpret_cast<double*>(take(part * 8));
  a.st_amax = reinterpret_cast<float*>(take(part * 4));
  a.row_m = reinterpret_cast<float*>(take((size_t)n_groups * kGroupRows * 4));
  a.row_il = reinterpret_cast<float*>(take((size_t)n_groups * kGroupRows * 4));
  a.tau = reinterpret_cast<float*>(take((size_t)n_heads * 4));
  a.kabs = reinterpret_cast<uint32_t*>(take((size_t)n_groups * kD * 4));
  a.row_marg = reinterpret_cast<float*>(take((size_t)n_heads * kTailRows * 4));
  a.hopeless = reinterpret_cast<int32_t*>(take((size_t)n_heads * 4));
  a.vscore = vscore ? vscore : reinterpret_cast<double*>(take((size_t)n_heads * S * 8));
  a.sscore = sscore ? sscore : reinterpret_cast<double*>(take((size_t)n_heads * S * 8));
  a.tile_max = reinterpret_cast<float*>(take((size_t)n_heads * kTailRows * a.n_tiles * 4));
  a.row_mc = reinterpret_cast<float*>(take((size_t)n_heads * kTailRows * 4));
  a.live = take((size_t)n_groups * a.n_tiles);
  int32_t* flags_ws = reinterpret_cast<int32_t*>(take((size_t)n_heads * 4));

  CUtensorMap tq, tk;
  int rc;
  if ((rc = make_tmap_bf16_3d(&tq, q, kD, S, Hq, kTailRows))) return rc;
  if ((rc = make_tmap_bf16_3d(&tk, k, kD, S, Hkv, kKeys))) return rc;
  static bool attr_done[2] = {false, false};
  if (!attr_done[kD / 64 - 1]) {
    if ((rc = check_cuda(cudaFuncSetAttribute(vs_tc_kernel<kD, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              L::kSmem), "vs_tc smem attr")))
      return rc;
    if ((rc = check_cuda(cudaFuncSetAttribute(vs_tc_kernel<kD, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              L::kSmem), "vs_tc smem attr")))
      return rc;
    attr_done[kD / 64 - 1] = true;
  }
  if ((rc = check_cuda(cudaMemsetAsync(a.sscore, 0, (size_t)n_heads * S * 8, st), "memset slash"))) return rc;
  if (uncertain && (rc = check_cuda(cudaMemsetAsync(uncertain, 0, (size_t)n_heads * 4, st), "memset flags")))
    return rc;
  int32_t* flags = uncertain ? uncertain : flags_ws;
  if (!uncertain && (rc = check_cuda(cudaMemsetAsync(flags, 0, (size_t)n_heads * 4, st), "memset flags"))) return rc;
  if ((rc = check_cuda(cudaMemsetAsync(a.kabs, 0, (size_t)n_groups * kD * 4, st), "memset kabs"))) return rc;
  a.flags = flags;
  a.uncertified = uncertified ? 1 : 0;
  const dim3 grid((unsigned)a.n_chunks, (unsigned)n_groups);
  note_launches(5);  // pass 1, combine, liveness, pass 2, top-k
  vs_tc_kernel<kD, 1><<<grid, kThreads, L::kSmem, st>>>(tq, tk, a);
  if ((rc = check_cuda(cudaGetLastError(), "vs_tc pass 1"))) return rc;
  vs_tc_combine_kernel<kD><<<n_groups, kGroupRows, 0, st>>>(a, q);
  vs_tc_live_kernel<<<dim3((unsigned)((a.n_tiles + 31) / 32), (unsigned)n_groups), 256, 0, st>>>(a);
  vs_tc_kernel<kD, 2><<<grid, kThreads, L::kSmem, st>>>(tq, tk, a);
  if ((rc = check_cuda(cudaGetLastError(), "vs_tc pass 2"))) return rc;
  vs_topk_certify_kernel<<<dim3(kTopkCl, (unsigned)n_heads, 2), kTopkThreads, 0, st>>>(a.vscore, a.sscore, S, k_v,
                                                                                        k_s, a.tau, a.hopeless, vout, sout,
                                                                                        flags);
  if ((rc = check_cuda(cudaGetLastError(), "vs_tc top-k"))) return rc;
  if (uncertified) return SPF_OK;
  // uncertified heads: fp64 re-estimation in the same stream (no host sync), skipping the
  // tiles whose probabilities round to exactly 0
  return vs_exact_run(SPF_DTYPE_BF16, q, k, Hq, Hkv, S, kD, head_ids, n_heads, kTailRows, k_v, k_s, vout, sout,
                      a.vscore, a.sscore, flags, a.tile_max, a.row_mc, a.row_marg, ws, st);
}

}  // namespace

bool vs_fast_supported(int dtype, int head_dim, int seq_len, int last_q) {
  return dtype == SPF_DTYPE_BF16 && (head_dim == 64 || head_dim == 128) && last_q == kTailRows &&
         seq_len >= kTailRows;
}

size_t vs_fast_workspace_size(int n_q_heads, int n_kv_heads, int n_heads, int seq_len) {
  const size_t hpk = n_q_heads / max(1, n_kv_heads);
  const size_t n_groups = (size_t)n_kv_heads * ((hpk + kMaxMembers - 1) / kMaxMembers);
  const size_t n_tiles = (seq_len + kKeys - 1) / kKeys;
  const size_t n_chunks = std::max<size_t>(1, std::min<size_t>(n_tiles, 148));
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t part = n_groups * n_chunks * kGroupRows;
  return al(part * 4) + al(part * 8) + al(part * 4) + 2 * al(n_groups * kGroupRows * 4) + al(n_heads * 4) +
         al(n_groups * 128 * 4) + al((size_t)n_heads * kTailRows * 4) + al(n_heads * 4) +
         2 * al((size_t)n_heads * seq_len * 8) + al((size_t)n_heads * kTailRows * n_tiles * 4) +
         al((size_t)n_heads * kTailRows * 4) + al(n_groups * n_tiles) + al(n_heads * 4) +
         vs_exact_workspace_size(n_heads, seq_len, kTailRows);
}

int vs_estimate_fast(const void* q, const void* k, int Hq, int Hkv, int S, int d, const int32_t* head_ids,
                     int n_heads, int k_v, int k_s, int32_t* vout, int32_t* sout, double* vscore, double* sscore,
                     int32_t* uncertain, bool uncertified, void* workspace, cudaStream_t st) {
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  const auto* qb = reinterpret_cast<const __nv_bfloat16*>(q);
  const auto* kb = reinterpret_cast<const __nv_bfloat16*>(k);
  if (d == 128)
    return vs_fast_impl<128>(qb, kb, Hq, Hkv, S, head_ids, n_heads, k_v, k_s, vout, sout, vscore, sscore, uncertain,
                             uncertified, ws, st);
  return vs_fast_impl<64>(qb, kb, Hq, Hkv, S, head_ids, n_heads, k_v, k_s, vout, sout, vscore, sscore, uncertain,
                          uncertified, ws, st);
}

}  // namespace spf
