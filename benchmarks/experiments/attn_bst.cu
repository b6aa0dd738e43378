// attn_bst.cu -- EXPERIMENT (not built into libspf.so; measured, not adopted): transposed-step
// sparse attention for heads whose 64-row blocks rarely share a tile (Block-Sparse heads),
// bf16 I/O.  To try it: copy into paper_2407_02490_b200/csrc/, declare attn_bst_supported /
// launch_sparse_attn_bst in spf_internal.h and route the pair heads to it in capi.cu
// (spf_sparse_flash_rows_ex).  Parity: tests/test_attention_gpu.py's paired-box and
// transposed tests passed with it routed (raise path, odd tile counts, LSE).
//
// Result (profiles/r02/bs_transposed_experiment.txt, C4-shaped BS(100) layer at 256K, 56/8
// heads): 99-102 ms vs the paired-box kernel's 92-97 ms; with one CTA per SM and 3/2/2-deep
// K/V/P rings 126 ms.  Both kernels are bound by the L2 -> SM traffic of the K/V tiles, not
// by the MMAs: each 64-key tile feeds only its own 64-row block (64 FLOP per byte of K+V),
// ncu on this kernel: 108 GB through L2 in 10.8 ms (10 TB/s, near the ~11.5 TB/s L2 cap),
// tensor pipe 28 % busy.  Removing the paired-box kernel's structural zeros frees tensor
// cycles the L2 cannot feed.
//
// Same contract as attn_fwd.cu (_core.pyx:72-192: per 64-row block its tiles, per-cell
// causal mask, one streaming-softmax state per row, zero rows without coverage); the heads
// routed here have no residual columns (BS layouts never do).
//
// A CTA owns ONE row block (64 queries) and walks its tiles two at a time (from the diagonal
// down).  The step is transposed so that no MMA carries structural zeros:
//   S^T[128 keys x 64 queries] = K[128 x d] . Q[64 x d]^T     (M128 x N64 x K=d, both K-major)
//   O^T[d x 64 queries]       += V^T[d x 128] . P^T[128 x 64]  (M=d x N64 x K128, both MN-major:
//                                                                V as loaded by TMA, P^T written
//                                                                by the softmax threads)
// The paired-box kernel (attn_bs.cu) spends half of every M128 x N128 QK and K128 PV on zeros;
// here both MMAs are dense, so a Block-Sparse step costs what a union step with full overlap
// costs.
//
// Softmax across TMEM lanes: thread k (TMEM lane k) holds key k's scores for all 64 queries,
// so a query's row maximum spans 128 threads.  The running maxima m_q are kept lazily: the
// exponent is taken against the stored m_q (shared memory) and only when some score would
// exceed it by more than 2^kLazy (bar.red.or over the 128 softmax threads, one barrier per
// step) is the step's exact column maximum reduced across the threads and O^T and the partial
// sums rescaled.  The diagonal tile comes first, so after step 0 the maxima rarely move.  With
// m_q <= the true maximum, p <= 2^kLazy stays well inside fp32/bf16 range and O, l are the
// same flash-attention sums (the common factor cancels in O / l).  Row sums are kept per
// thread (per key) and reduced once at the end in a fixed order.
//
// TMEM (256 columns, two CTAs per SM): S^T double-buffered in [0,64) and [64,128) fp32, O^T in
// [128,192).  Shared memory: Q 16 KB, one K and one V stage of two 64-key boxes (32 KB each),
// P^T 16 KB (single-buffered: P(t+1) is written once PV(t) retired).  An absent box (odd tile
// count) is a TMA load past the end of the sequence: zeros, masked out.
#include "spf_internal.h"
#include "spf_ptx.cuh"

#include <math.h>

namespace spf {

namespace {

constexpr int kQ = 64;          // queries per CTA (one row block)
constexpr int kBox = 64;        // keys per tile
constexpr int kKeys = 128;      // two tiles per step
constexpr int kThreads = 192;   // loader, MMA issuer, 4 softmax warps (one per TMEM lane quarter)
constexpr float kNoMax = -1e30f;
constexpr int kSK = 1, kSV = 1, kSP = 1;  // K / V / P^T ring depths (3/2/2 with one CTA per SM: 126 ms)
constexpr int kMinBlocks = 2;             // CTAs per SM (shared memory: the rings)  // stored maximum of a query that has seen no key yet (finite: no NaN)
constexpr float kLazy = 20.f;   // p <= 2^kLazy before the stored maxima are raised

struct TDesc {
  int box[2];    // first key of each box
  int width[2];  // keys of the box inside the sequence (0: absent)
  int end;       // 1: no more steps
};

struct TCtrl {
  uint64_t q_full;
  uint64_t k_full[kSK], k_empty[kSK], v_full[kSV], v_empty[kSV];
  uint64_t d_full[2], d_empty[2];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full[kSP], p_empty[kSP], o_ready;
  uint32_t tmem_base, pad;
  TDesc desc[2];
  float m[kQ];        // stored row maxima (log2 units), one per query
  float alpha[kQ];    // rescale factors of the last raise; row sums in the epilogue
  float red[4][kQ];   // per-warp column maxima (raise path)
};

template <int kD>
struct TLayout {
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQAtom = kQ * 128;       // one 64-wide d atom of the 64 queries
  static constexpr int kKAtom = kKeys * 128;    // one 64-wide d atom of the 128 keys (SW128 rows)
  static constexpr int kQBytes = kAtoms * kQAtom;
  static constexpr int kStage = kAtoms * kKAtom;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kSK * kStage;
  static constexpr int kPBytes = kKeys * 128;  // P^T: 128 key rows x 64 queries (128 B), SW128
  static constexpr int kOffP = kOffV + kSV * kStage;
  static constexpr int kOffCtrl = kOffP + kSP * kPBytes;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(TCtrl);
  static constexpr uint32_t kTxBox = kBox * kD * 2;
  static constexpr uint32_t kTmemCols = 256;
  static constexpr uint32_t kColO = 128;
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// bar.red.or over `n` threads of named barrier `id`: true in every thread if any passed true
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "bar.red.or.pred p, %2, %3, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

template <int kD>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    sparse_attn_bst_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const AttnArgs p, int n_rows,
                           float scale_log2) {
  using L = TLayout<kD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  TCtrl* ctrl = reinterpret_cast<TCtrl*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work item: head major (the listed heads in order, so the CTAs in flight share one kv
  // head's K/V in L2), heavy (late) row blocks first
  const int item = blockIdx.x;
  const int hl = item / n_rows;
  const int h = p.pair_heads[hl];
  if (h < 0 || h >= p.Hq) return;
  if (!pair_preferred(p.pair_stats, hl)) return;  // the union kernel runs this head
  const int r = n_rows - 1 - item % n_rows;
  const int kvh = h / (p.Hq / p.Hkv);
  const int S = p.S;
  const int R0 = r * kBox;
  const int64_t row = (int64_t)h * n_rows + r;

  if (threadIdx.x == 0) {
    mbar_init(&ctrl->q_full, 1);
    for (int s = 0; s < kSK; ++s) {
      mbar_init(&ctrl->k_full[s], 1);
      mbar_init(&ctrl->k_empty[s], 1);
    }
    for (int s = 0; s < kSV; ++s) {
      mbar_init(&ctrl->v_full[s], 1);
      mbar_init(&ctrl->v_empty[s], 1);
    }
    for (int s = 0; s < kSP; ++s) {
      mbar_init(&ctrl->p_full[s], 128);
      mbar_init(&ctrl->p_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->d_full[s], 1);
      mbar_init(&ctrl->d_empty[s], 5);  // 4 softmax warps + the MMA warp
      mbar_init(&ctrl->s_full[s], 1);
      mbar_init(&ctrl->s_empty[s], 4);
    }
    mbar_init(&ctrl->o_ready, 1);
    fence_mbar_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + kQ) ctrl->m[threadIdx.x - 64] = kNoMax;
  if (warp == 1) tmem_alloc(&ctrl->tmem_base, L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctrl->tmem_base;

  if (warp == 0) {
    // =============================== loader warp ===============================
    if (lane == 0) {
      const int64_t a0 = p.tile_offsets[row];
      const int64_t n = p.tile_offsets[row + 1] - a0;
      const int64_t steps = (n + 1) >> 1;
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(&ctrl->q_full, L::kQBytes);
#pragma unroll
      for (int a = 0; a < L::kAtoms; ++a)
        tma_load_3d(smem + L::kOffQ + a * L::kQAtom, &tm_q, &ctrl->q_full, a * 64, R0, h);
      for (int64_t i = 0; i <= steps; ++i) {
        const int sd = (int)(i & 1);
        mbar_wait(&ctrl->d_empty[sd], (int)((i >> 1) & 1) ^ 1);
        TDesc& d = ctrl->desc[sd];
        if (i == steps) {
          d.end = 1;
          mbar_arrive(&ctrl->d_full[sd]);
          break;
        }
        int box[2];
        bool has[2];
        box[0] = p.tile_starts[a0 + n - 1 - 2 * i];  // descending: the diagonal block first
        has[0] = true;
        has[1] = 2 * i + 1 < n;
        box[1] = has[1] ? p.tile_starts[a0 + n - 2 - 2 * i] : S;
        // K(i): the stage is free once QK(i - kSK) retired
        const int ks = (int)(i % kSK), vs = (int)(i % kSV);
        mbar_wait(&ctrl->k_empty[ks], (int)((i / kSK) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctrl->k_full[ks], 2 * L::kTxBox);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int kr = has[b] ? box[b] : S;  // absent: past the end -> zero fill
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a)
            tma_load_3d(smem + L::kOffK + ks * L::kStage + a * L::kKAtom + b * (kBox * 128), &tm_k, &ctrl->k_full[ks], a * 64, kr,
                        kvh);
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          d.box[b] = box[b];
          // keys of the box that exist: inside [0, S) (a tile may start before 0 or end past S)
          d.width[b] = has[b] ? max(0, min(kBox, S - box[b])) : 0;
        }
        d.end = 0;
        mbar_arrive(&ctrl->d_full[sd]);
        // V(i): the stage is free once PV(i - kSV) retired
        mbar_wait(&ctrl->v_empty[vs], (int)((i / kSV) & 1) ^ 1);
        mbar_arrive_expect_tx(&ctrl->v_full[vs], 2 * L::kTxBox);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int kr = has[b] ? box[b] : S;
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a)
            tma_load_3d(smem + L::kOffV + vs * L::kStage + a * L::kKAtom + b * (kBox * 128), &tm_v, &ctrl->v_full[vs], a * 64, kr,
                        kvh);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =============================== MMA issuer ================================
    constexpr uint32_t idesc_qk = umma_idesc_bf16(128, kQ, 0, 0);
    constexpr uint32_t idesc_pv = umma_idesc_bf16(kD, kQ, 1, 1);
    const uint32_t tO = tmem + L::kColO;
    const uint32_t klo = sw128_lo(sbase + L::kOffK, 0);
    const uint32_t qlo = sw128_lo(sbase + L::kOffQ, 0);
    const uint32_t vlo = sw128_lo(sbase + L::kOffV, L::kKAtom);  // LBO: next 64-wide d atom (M)
    const uint32_t plo = sw128_lo(sbase + L::kOffP, L::kKAtom);  // one 64-query atom (N)
    constexpr uint32_t dhi = sw128_hi(1024);
    mbar_wait(&ctrl->q_full, 0);
    tc_fence_after();
    for (int t = 0;; ++t) {
      const int sd = t & 1;
      mbar_wait(&ctrl->d_full[sd], (t >> 1) & 1);
      const bool end = *reinterpret_cast<volatile int*>(&ctrl->desc[sd].end) != 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);  // the slot may be rewritten once all have read it
      if (!end) {
        const int ks = t % kSK;
        mbar_wait(&ctrl->k_full[ks], (t / kSK) & 1);
        if (t >= 2) mbar_wait(&ctrl->s_empty[sd], ((t >> 1) & 1) ^ 1);  // softmax read S(t - 2)
        tc_fence_after();
        // S^T(t) = K Q^T: 128 keys x 64 queries
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t aoff = ((k >> 2) * L::kKAtom + (k & 3) * 32) >> 4;
          const uint32_t boff = ((k >> 2) * L::kQAtom + (k & 3) * 32) >> 4;
          mma_bf16_ss_w2(tmem + sd * kQ, klo + ((ks * L::kStage) >> 4) + aoff, dhi, qlo + boff, dhi, idesc_qk,
                         k > 0 ? 1u : 0u);
        }
        mma_commit_w(&ctrl->s_full[sd]);
        mma_commit_w(&ctrl->k_empty[ks]);
      }
      if (t >= 1) {
        // O^T += V^T(t - 1) P^T(t - 1) over the step's 128 keys (16 per MMA: 2048 B of rows)
        const int u = t - 1;
        const int vs = u % kSV, ps = u % kSP;
        mbar_wait(&ctrl->p_full[ps], (u / kSP) & 1);
        mbar_wait(&ctrl->v_full[vs], (u / kSV) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k)
          mma_bf16_ss_w2(tO, vlo + ((vs * L::kStage + k * 2048) >> 4), dhi, plo + ((ps * L::kPBytes + k * 2048) >> 4), dhi, idesc_pv,
                         (u > 0 || k > 0) ? 1u : 0u);
        mma_commit_w(&ctrl->p_empty[ps]);
        mma_commit_w(&ctrl->v_empty[vs]);
      }
      if (end) break;
    }
    mma_commit_w(&ctrl->o_ready);
    __syncwarp();
  } else {
    // =============================== softmax warps =============================
    // thread kk = TMEM lane kk = key kk of the step (box kk / 64); 64 columns = the queries
    const int quarter = warp & 3;
    const int kk = quarter * 32 + lane;
    const int bx = kk >> 6, kin = kk & 63;
    const int stid = threadIdx.x - 64;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float lp[kQ];  // this key slot's share of every query's row sum
#pragma unroll
    for (int j = 0; j < kQ; ++j) lp[j] = 0.f;
    int t = 0;
    for (;; ++t) {
      const int sd = t & 1;
      mbar_wait(&ctrl->d_full[sd], (t >> 1) & 1);
      const TDesc& d = ctrl->desc[sd];
      const int end = d.end;
      const int box = d.box[bx], width = d.width[bx];
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);
      if (end) break;
      // key position and its causal reach: queries j < jlo (row R0 + j < key) do not see it
      const int kpos = box + kin;
      const bool kvalid = kin < width && kpos >= 0;
      const int jlo = kvalid ? min(kQ, max(0, kpos - R0)) : kQ;
      const bool any_mask = __any_sync(0xffffffffu, jlo > 0);
      mbar_wait(&ctrl->s_full[sd], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t s_addr = tmem + lane_off + sd * kQ;
      // y = s * c - m (stored maxima, finite); masked cells -inf (set before the subtraction)
      uint32_t y[kQ];
      auto scores = [&]() {
        tmem_ld32x32b_x64(s_addr, y);
        tmem_wait_ld();
        if (any_mask) {
#pragma unroll
          for (int j = 0; j < kQ; ++j) y[j] = j < jlo ? 0xff800000u : y[j];
        }
        const float4* m4 = reinterpret_cast<const float4*>(ctrl->m);
#pragma unroll
        for (int j = 0; j < kQ; j += 4) {
          const float4 mv = m4[j >> 2];
          y[j] = __float_as_uint(fmaf(u2f(y[j]), scale_log2, -mv.x));
          y[j + 1] = __float_as_uint(fmaf(u2f(y[j + 1]), scale_log2, -mv.y));
          y[j + 2] = __float_as_uint(fmaf(u2f(y[j + 2]), scale_log2, -mv.z));
          y[j + 3] = __float_as_uint(fmaf(u2f(y[j + 3]), scale_log2, -mv.w));
        }
      };
      scores();
      bool over;
      {
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int j = 0; j < kQ; j += 8) {
          mx0 = fmax3(mx0, u2f(y[j]), u2f(y[j + 1]));
          mx1 = fmax3(mx1, u2f(y[j + 2]), u2f(y[j + 3]));
          mx2 = fmax3(mx2, u2f(y[j + 4]), u2f(y[j + 5]));
          mx3 = fmax3(mx3, u2f(y[j + 6]), u2f(y[j + 7]));
        }
        // a query that saw no key before (m = kNoMax) gives ~1e30 here and raises
        over = fmax3(mx0, mx1, fmaxf(mx2, mx3)) > kLazy;
      }
      if (bar_red_or(1, 128, over)) {
        // raise (rare): the step's exact column maxima over the 128 keys, S re-read from TMEM
        // in 8-column slices (the buffer is released only after this decision)
#pragma unroll 1
        for (int c = 0; c < kQ; c += 8) {
          uint32_t x[8];
          tmem_ld32x32b_x8(s_addr + c, x);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float v = (any_mask && c + j < jlo) ? -INFINITY : u2f(x[j]) * scale_log2;
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
            if (lane == 0) ctrl->red[quarter][c + j] = v;
          }
        }
        named_bar_sync(2, 128);
        if (stid < kQ) {
          const float mo = ctrl->m[stid];
          const float mn = fmaxf(mo, fmaxf(fmaxf(ctrl->red[0][stid], ctrl->red[1][stid]),
                                           fmaxf(ctrl->red[2][stid], ctrl->red[3][stid])));
          ctrl->alpha[stid] = mn == mo ? 1.f : ex2_approx(mo - mn);  // kNoMax: 2^-huge = 0
          ctrl->m[stid] = mn;
        }
        named_bar_sync(2, 128);
#pragma unroll
        for (int j = 0; j < kQ; ++j) lp[j] *= ctrl->alpha[j];
        if (t > 0) {
          // O^T columns (queries) rescaled: needs PV(t - 1) retired
          mbar_wait(&ctrl->p_empty[(t - 1) % kSP], ((t - 1) / kSP) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < kQ; c += 8) {
            uint32_t o[8];
            tmem_ld32x32b_x8(tmem + lane_off + L::kColO + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = __float_as_uint(u2f(o[j]) * ctrl->alpha[c + j]);
            tmem_st32x32b_x8(tmem + lane_off + L::kColO + c, o);
          }
          tmem_wait_st();
        }
        scores();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->s_empty[sd]);
      // p = 2^y; row-sum shares; P^T row kk as bf16 (SW128: 16-byte chunk c at c ^ (kk & 7))
      uint32_t ph[kQ / 2];
#pragma unroll
      for (int j = 0; j < kQ; j += 2) {
        const float p0 = ex2_approx(u2f(y[j])), p1 = ex2_approx(u2f(y[j + 1]));
        lp[j] += p0;
        lp[j + 1] += p1;
        ph[j >> 1] = pack_bf16x2(p0, p1);
      }
      const int ps = t % kSP;
      const uint32_t prow = sbase + L::kOffP + ps * L::kPBytes + kk * 128;
      if (t >= kSP) mbar_wait(&ctrl->p_empty[ps], ((t / kSP) & 1) ^ 1);  // PV(t - kSP) has read it
#pragma unroll
      for (int c = 0; c < 8; ++c)
        st_shared_v4(prow + ((c ^ (kk & 7)) << 4), ph[4 * c], ph[4 * c + 1], ph[4 * c + 2], ph[4 * c + 3]);
      fence_proxy_async_smem();
      mbar_arrive(&ctrl->p_full[ps]);
    }
    // ---- epilogue: row sums (fixed order over the 128 key slots), O^T / l -> global ----
    mbar_wait(&ctrl->o_ready, 0);
    tc_fence_after();
    float* lred = reinterpret_cast<float*>(smem + L::kOffK);  // K stage is free: every MMA retired
#pragma unroll
    for (int j = 0; j < kQ; ++j) lred[kk * (kQ + 1) + j] = lp[j];
    named_bar_sync(2, 128);
    if (stid < kQ) {
      float l = 0.f;
      for (int k2 = 0; k2 < kKeys; ++k2) l += lred[k2 * (kQ + 1) + stid];
      ctrl->alpha[stid] = l;
      const int q = R0 + stid;
      if (p.lse != nullptr && q < S)
        p.lse[(int64_t)h * S + q] = (t > 0 && l > 0.f) ? (ctrl->m[stid] + log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
    named_bar_sync(2, 128);
    uint32_t o[kQ];
    if (t > 0) {
      tmem_ld32x32b_x64(tmem + lane_off + L::kColO, o);
      tmem_wait_ld();
    }
    const int dout = p.d_out;
    if (kk < dout) {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + ((int64_t)h * S + R0) * dout + kk;
#pragma unroll
      for (int j = 0; j < kQ; ++j) {
        const float l = ctrl->alpha[j];
        const float v = (t > 0 && l > 0.f) ? u2f(o[j]) / l : 0.f;
        if (R0 + j < S) out[(int64_t)j * dout] = __float2bfloat16_rn(v);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, L::kTmemCols);
  }
}

template <int kD>
int launch_bst_impl(const AttnArgs& a, cudaStream_t stream) {
  using L = TLayout<kD>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_tmap_bf16_3d(&tq, a.q_hi, kD, a.S, a.Hq, kQ))) return rc;
  if ((rc = make_tmap_bf16_3d(&tk, a.k_hi, kD, a.S, a.Hkv, kBox))) return rc;
  if ((rc = make_tmap_bf16_3d(&tv, a.v_hi, kD, a.S, a.Hkv, kBox))) return rc;
  auto kern = sparse_attn_bst_kernel<kD>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(bst attn smem)");
    attr_done = true;
  }
  const int n_rows = (a.S + kBox - 1) / kBox;
  const long long grid = (long long)n_rows * a.n_pair;
  if (grid == 0) return 0;
  if (grid > 0x7fffffffLL) return set_error(2, "attention grid too large");
  note_launches(1);
  kern<<<(unsigned)grid, kThreads, L::kSmem, stream>>>(tq, tk, tv, a, n_rows, a.scale * 1.4426950408889634f);
  return check_cuda(cudaGetLastError(), "sparse_attn_bst launch");
}

}  // namespace

bool attn_bst_supported(const AttnArgs& a) {
  return !a.split && !a.out_f32 && a.B == kBox && a.kD == 128 && a.work_order == nullptr;
}

int launch_sparse_attn_bst(const AttnArgs& a, cudaStream_t stream) { return launch_bst_impl<128>(a, stream); }

}  // namespace spf
