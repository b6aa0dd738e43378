// attn_bs.cu -- paired-box sparse attention for heads whose two 64-row blocks per
// 128-row CTA rarely share a tile (Block-Sparse heads: every block row picks its own
// k_b key blocks), bf16 I/O.
//
// Same contract as attn_fwd.cu (_core.pyx:72-192: per 64-row block its tiles, per-cell
// causal mask, one streaming-softmax state per row, zero rows without coverage); the
// heads routed here have no residual columns (BS layouts never do).
//
// The union kernel (attn_fwd.cu) gives both row blocks of a CTA every tile of either,
// so a BS CTA runs ~2 k_b steps of an M128 x N64 QK with half the rows masked.  Here a
// step pairs the i-th tile of row block r0 with the i-th tile of row block r1 (both
// walked from the diagonal down): one M128 x N128 x K=d QK (full tensor rate, where the
// N64 one is shared-memory bound; profiles/r01/mma_pair_microbench.txt) whose rows
// 0..63 keep the first 64 columns and rows 64..127 the last 64, and one M128 x N=d x
// K128 PV with the off-block half of P zero.  Each thread still exponentiates 64 keys
// per step, and there are max(n0, n1) steps instead of |tiles(r0) U tiles(r1)|.
//
// TMEM (256 columns, two CTAs per SM): S [0,128) fp32, P written back over its first
// 64 columns as bf16 pairs, O [128,256).  With P over S, QK(t+1) is issued after PV(t)
// (in-order pipe), so S(t) ready also implies PV(t-1) retired.  Shared memory: Q 32 KB,
// one K and one V stage of two 64-key boxes (the chain leaves a whole softmax step for
// the next loads).  An absent box (the shorter list ran out) is a TMA load past the
// end of the sequence: zeros, masked out.
#include "spf_internal.h"
#include "spf_ptx.cuh"

#include <math.h>

namespace spf {

namespace {

constexpr int kRows = 128;
constexpr int kBox = 64;
constexpr int kKeys = 128;  // two boxes per step
// SPF_PAIR_HALVES=2 (with union pairing): two softmax warps per TMEM lane quarter, each
// exponentiating 64 of a row's 128 keys (both read all 128 for the max)
#ifndef SPF_PAIR_HALVES
#define SPF_PAIR_HALVES 1
#endif
constexpr int kHalves = SPF_PAIR_HALVES;
constexpr int kThreads = 64 + 128 * kHalves;

struct PairDesc {
  int box[2];    // first key of each box (-1: absent)
  int width[2];  // keys of the box inside the sequence
  int seg[2];    // union pairing: bit h set = row block h of the CTA owns the box (0: absent)
  int end;       // 1: no more steps
};

// SPF_PAIR_UNION=1 (experiment): a step takes the next TWO items of the union of the
// CTA's two tile lists (descending), so every row exponentiates up to 128 keys per step --
// the union kernel's work in half the steps, for heads without residual columns.
#ifndef SPF_PAIR_UNION
#define SPF_PAIR_UNION 0
#endif
constexpr bool kUnion = SPF_PAIR_UNION != 0;


// !kDB (the default): two CTAs per SM, one S with P written over it -- a serial
// softmax -> PV -> QK chain per CTA that the co-resident CTA interleaves with.
// kDB (SPF_PAIR_DB=1): one CTA per SM owning all 512 TMEM columns -- S(t) in
// [128 (t&1), +128), O [256,384), P(t) in [384 + 64 (t&1), +64) -- so QK(t+1) overlaps the
// softmax of step t; identical results, but measured 10-14 % slower than two interleaved
// CTAs (profiles/r01/attn_bottleneck_experiments.txt).
#ifndef SPF_PAIR_DB
#define SPF_PAIR_DB 0
#endif
constexpr bool kDB = SPF_PAIR_DB != 0;
static_assert(kHalves == 1 || (kHalves == 2 && kUnion && kDB), "split softmax rows: union pairing, one CTA per SM");
constexpr int kStages = kDB ? 2 : 1;

struct PCtrl {
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t d_full[2], d_empty[2];
  uint64_t s_full[2], s_free[2], p_full[2], o_ready;
  uint32_t tmem_base, pad;
  PairDesc desc[2];
  float lsum[2][128];  // split softmax: each half's row sums, combined in the epilogue
};

template <int kD>
struct PLayout {
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQBytes = kRows * kD * 2;
  static constexpr int kAtomStage = kKeys * 128;  // one 64-wide d atom of 128 keys (SW128 rows)
  static constexpr int kStage = kAtoms * kAtomStage;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kStage;
  static constexpr int kOffCtrl = kOffV + kStages * kStage;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(PCtrl);
  static constexpr uint32_t kTxBox = kBox * kD * 2;
  static constexpr uint32_t kTmemCols = kDB ? 512 : 256;
  static constexpr uint32_t kColO = kDB ? 256 : 128;
};
// TMEM column of S(t) / P(t)
__device__ __forceinline__ uint32_t s_col(int t) { return kDB ? (uint32_t)(t & 1) * 128 : 0u; }
__device__ __forceinline__ uint32_t p_col(int t) { return kDB ? 384u + (uint32_t)(t & 1) * 64 : 0u; }

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// SPF_PAIR_TRACE=1 (debug): clock64 stamps of softmax warp 2 (lane 0) per step in the union-pairing
// path, 8 slots per (CTA, step), for the first spf_debug_pair_trace CTAs.
#ifndef SPF_PAIR_TRACE
#define SPF_PAIR_TRACE 0
#endif
constexpr int kPTraceSteps = 64;
__device__ unsigned long long* g_ptrace = nullptr;
__device__ int g_ptrace_ctas = 0;
__device__ __forceinline__ void ptrace(bool on, int step, int ev) {
  if (!SPF_PAIR_TRACE || !on) return;
  unsigned long long* tr = g_ptrace;
  if (tr == nullptr || (int)blockIdx.x >= g_ptrace_ctas || step >= kPTraceSteps) return;
  tr[((int64_t)blockIdx.x * kPTraceSteps + step) * 8 + ev] = (unsigned long long)clock64();
}

template <int kD>
__global__ void __launch_bounds__(kThreads, kDB ? 1 : 2)
    sparse_attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                            const __grid_constant__ CUtensorMap tm_v, const AttnArgs p, int n_ctile,
                            float scale_log2) {
  using L = PLayout<kD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  PCtrl* ctrl = reinterpret_cast<PCtrl*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work item: head major (the listed heads in order), heavy (late) row tiles first.
  // Block-Sparse tiles are scattered over the whole causal prefix, so the CTAs in flight
  // should share one kv head's K/V (<= 2 * S * d * 2 bytes) in L2 rather than span all
  // kv heads (heads-fastest order: 524 GB of DRAM reads per C4 launch instead of 59 GB).
  const int item = blockIdx.x;
  const int h = p.pair_heads[item / n_ctile];
  if (h < 0 || h >= p.Hq) return;
  if (!pair_preferred(p.pair_stats, item / n_ctile)) return;  // the union kernel runs this head
  const int ct = n_ctile - 1 - item % n_ctile;
  const int kvh = h / (p.Hq / p.Hkv);
  const int S = p.S;
  const int n_rows = (S + kBox - 1) / kBox;
  const int R0 = ct * kRows;
  const int r0 = R0 / kBox;
  const bool has_r1 = r0 + 1 < n_rows;

  if (threadIdx.x == 0) {
    mbar_init(&ctrl->q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->k_full[s], 1);
      mbar_init(&ctrl->k_empty[s], 1);
      mbar_init(&ctrl->v_full[s], 1);
      mbar_init(&ctrl->v_empty[s], 1);
      mbar_init(&ctrl->d_full[s], 1);
      mbar_init(&ctrl->d_empty[s], 4 * kHalves);
      mbar_init(&ctrl->s_full[s], 1);
      mbar_init(&ctrl->s_free[s], 4 * kHalves);
      mbar_init(&ctrl->p_full[s], 128 * kHalves);
    }
    mbar_init(&ctrl->o_ready, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&ctrl->tmem_base, L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctrl->tmem_base;

  if (warp == 0) {
    // =============================== loader warp ===============================
    const int64_t row_a = (int64_t)h * n_rows + r0;
    const int64_t a0 = p.tile_offsets[row_a], n0 = p.tile_offsets[row_a + 1] - a0;
    const int64_t a1 = has_r1 ? p.tile_offsets[row_a + 1] : 0;
    const int64_t n1 = has_r1 ? p.tile_offsets[row_a + 2] - a1 : 0;
    const int64_t steps = n0 > n1 ? n0 : n1;
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(&ctrl->q_full, L::kQBytes);
#pragma unroll
      for (int a = 0; a < L::kAtoms; ++a)
        tma_load_3d(smem + L::kOffQ + a * (kRows * 128), &tm_q, &ctrl->q_full, a * 64, R0, h);
      int64_t j0 = n0 - 1, j1 = n1 - 1;  // union walk: next candidate of each ascending list
      auto next_item = [&](int& start, int& seg) {
        const bool h0 = j0 >= 0, h1 = j1 >= 0;
        if (!h0 && !h1) return false;
        const int s0 = h0 ? p.tile_starts[a0 + j0] : 0;
        const int s1 = h1 ? p.tile_starts[a1 + j1] : 0;
        if (h0 && (!h1 || s0 >= s1)) {
          start = s0;
          seg = 1;
          --j0;
          if (h1 && s1 == s0) {
            seg = 3;
            --j1;
          }
        } else {
          start = s1;
          seg = 2;
          --j1;
        }
        return true;
      };
      for (int64_t i = 0; kUnion || i <= steps; ++i) {
        const int sd = (int)(i & 1);
        mbar_wait(&ctrl->d_empty[sd], (int)((i >> 1) & 1) ^ 1);
        PairDesc& d = ctrl->desc[sd];
        int box[2], seg[2];
        bool more = true;
        if (kUnion) {
          more = next_item(box[0], seg[0]);
          if (more && !next_item(box[1], seg[1])) {
            box[1] = S;
            seg[1] = 0;
          }
        } else {
          more = i < steps;
          box[0] = i < n0 ? p.tile_starts[a0 + n0 - 1 - i] : -1;  // descending: the diagonal block first
          box[1] = i < n1 ? p.tile_starts[a1 + n1 - 1 - i] : -1;
          seg[0] = box[0] >= 0 ? 1 : 0;
          seg[1] = box[1] >= 0 ? 2 : 0;
        }
        if (!more) {
          d.end = 1;
          mbar_arrive(&ctrl->d_full[sd]);
          break;
        }
        // K(i): its stage is free once QK(i - kStages) retired
        const int st = (int)(i % kStages);
        const int sph = (int)((i / kStages) & 1);
        mbar_wait(&ctrl->k_empty[st], sph ^ 1);
        mbar_arrive_expect_tx(&ctrl->k_full[st], 2 * L::kTxBox);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int row = seg[b] ? box[b] : S;  // absent: past the end -> zero fill
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a)
            tma_load_3d(smem + L::kOffK + st * L::kStage + a * L::kAtomStage + b * (kBox * 128), &tm_k,
                        &ctrl->k_full[st], a * 64, row, kvh);
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          d.box[b] = box[b];
          d.width[b] = seg[b] ? min(kBox, S - box[b]) : 0;
          d.seg[b] = seg[b];
        }
        d.end = 0;
        mbar_arrive(&ctrl->d_full[sd]);
        // V(i): its stage is free once PV(i - kStages) retired
        mbar_wait(&ctrl->v_empty[st], sph ^ 1);
        mbar_arrive_expect_tx(&ctrl->v_full[st], 2 * L::kTxBox);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int row = seg[b] ? box[b] : S;
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a)
            tma_load_3d(smem + L::kOffV + st * L::kStage + a * L::kAtomStage + b * (kBox * 128), &tm_v,
                        &ctrl->v_full[st], a * 64, row, kvh);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // =============================== MMA issuer ================================
    constexpr uint32_t idesc_qk = umma_idesc_bf16(128, kKeys, 0, 0);
    constexpr uint32_t idesc_pv = umma_idesc_bf16(128, kD, 0, 1);
    const uint32_t tO = tmem + L::kColO;
    const uint32_t qlo0 = sw128_lo(sbase + L::kOffQ, 0);
    const uint32_t klo0 = sw128_lo(sbase + L::kOffK, 0);
    const uint32_t vlo0 = sw128_lo(sbase + L::kOffV, L::kAtomStage);  // LBO: next 64-wide d atom
    constexpr uint32_t dhi = sw128_hi(1024);
    mbar_wait(&ctrl->q_full, 0);
    tc_fence_after();
    auto issue_pv = [&](int u) {  // O += P(u) V(u) over the step's 128 keys
      const int st = u % kStages;
      mbar_wait(&ctrl->p_full[u & 1], (u >> 1) & 1);
      mbar_wait(&ctrl->v_full[st], (u / kStages) & 1);
      tc_fence_after();
      const uint32_t vd = vlo0 + ((uint32_t)(st * L::kStage) >> 4);
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k)
        mma_bf16_ts_w2(tO, tmem + p_col(u) + k * 8, vd + ((k * 2048) >> 4), dhi, idesc_pv, (u > 0 || k > 0) ? 1u : 0u);
      mma_commit_w(&ctrl->v_empty[st]);
    };
    int t = 0;
    for (;; ++t) {
      const int sd = t & 1;
      mbar_wait(&ctrl->d_full[sd], (t >> 1) & 1);
      if (*reinterpret_cast<volatile int*>(&ctrl->desc[sd].end)) break;
      const int st = t % kStages;
      mbar_wait(&ctrl->k_full[st], (t / kStages) & 1);
      if (kDB && t >= 2) mbar_wait(&ctrl->s_free[t & 1], ((t - 2) >> 1) & 1);  // softmax(t-2) read S
      tc_fence_after();
      // S(t) = Q K^T over 128 keys (single-buffered: the previous PV has read P out of S)
      const uint32_t kd = klo0 + ((uint32_t)(st * L::kStage) >> 4);
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t aoff = ((k >> 2) * (kRows * 128) + (k & 3) * 32) >> 4;
        const uint32_t boff = ((k >> 2) * L::kAtomStage + (k & 3) * 32) >> 4;
        mma_bf16_ss_w2(tmem + s_col(t), qlo0 + aoff, dhi, kd + boff, dhi, idesc_qk, k > 0 ? 1u : 0u);
      }
      mma_commit_w(&ctrl->s_full[t & 1]);
      mma_commit_w(&ctrl->k_empty[st]);
      if (kDB) {
        if (t > 0) issue_pv(t - 1);  // PV(t-1) behind QK(t): the next S is never late for PV
      } else {
        issue_pv(t);
      }
    }
    if (kDB && t > 0) issue_pv(t - 1);
    mma_commit_w(&ctrl->o_ready);
    __syncwarp();
  } else {
    // =============================== softmax warps =============================
    // rows 0..63 (lane quarters 0, 1) = row block r0 -> S columns 0..63 (box 0);
    // rows 64..127 (quarters 2, 3) = row block r1 -> S columns 64..127 (box 1)
    const int quarter = warp & 3;
    const int half = quarter >> 1;
    const int kh = kHalves > 1 ? (warp - 2) >> 2 : 0;  // key half of a 128-key step (split softmax)
    const int row = quarter * 32 + lane;
    const int q = R0 + row;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    int t = 0;
    for (;; ++t) {
      const int sd = t & 1;
      mbar_wait(&ctrl->d_full[sd], (t >> 1) & 1);
      const PairDesc& d = ctrl->desc[sd];
      if (d.end) break;
      const bool tr0 = warp == 2 && lane == 0;
      ptrace(tr0, t, 0);
      if (kUnion) {
        // both boxes may belong to this row's block: up to 128 keys per row
        int lo[2], hi[2];
        bool any = false;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          lo[b] = 0;
          hi[b] = 0;
          if (((d.seg[b] >> half) & 1) && q < S) {
            const int bx = d.box[b];
            lo[b] = max(0, -bx);
            hi[b] = min(d.width[b], q - bx + 1);
          }
          any = any || hi[b] > lo[b];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);
        const bool warp_skip = !__any_sync(0xffffffffu, any);
        mbar_wait(&ctrl->s_full[t & 1], (t >> 1) & 1);
        tc_fence_after();
        ptrace(tr0, t, 1);
        uint32_t x[kKeys];  // x[0, 64): this warp's own key half (box kh), x[64, 128): the other box
        float alpha = 1.f;
        bool rescale = false;
        if (!warp_skip) {
          tmem_ld32x32b_x64(tmem + lane_off + s_col(t) + kh * kBox, x);
          tmem_ld32x32b_x64(tmem + lane_off + s_col(t) + (kh ^ 1) * kBox, x + kBox);
          tmem_wait_ld();
          ptrace(tr0, t, 2);
          const int lo_a = kh ? lo[1] : lo[0], hi_a = kh ? hi[1] : hi[0];
          const int lo_b = kh ? lo[0] : lo[1], hi_b = kh ? hi[0] : hi[1];
          if (!(lo_a == 0 && hi_a == kBox)) {
#pragma unroll
            for (int j = 0; j < kBox; ++j) x[j] = (j >= lo_a && j < hi_a) ? x[j] : 0xff800000u;
          }
          if (!(lo_b == 0 && hi_b == kBox)) {
#pragma unroll
            for (int j = 0; j < kBox; ++j) x[kBox + j] = (j >= lo_b && j < hi_b) ? x[kBox + j] : 0xff800000u;
          }
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int j = 0; j < kKeys; j += 8) {
            mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
            mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
            mx2 = fmax3(mx2, u2f(x[j + 4]), u2f(x[j + 5]));
            mx3 = fmax3(mx3, u2f(x[j + 6]), u2f(x[j + 7]));
          }
          const float mx = fmax3(mx0, mx1, fmaxf(mx2, mx3));
          ptrace(tr0, t, 3 + (__float_as_uint(mx) == 0x7fc00001u ? 1 : 0));
          if (any) {
            const float m_tile = mx * scale_log2;
            if (m_run == -INFINITY) {
              m_run = m_tile;
            } else if (m_tile > m_run + 8.f) {
              alpha = exp2f(m_run - m_tile);
              m_run = m_tile;
              rescale = true;
            }
          }
          const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
          const uint64_t c2 = pack_f32x2(scale_log2, scale_log2);
          const uint64_t m2 = pack_f32x2(neg_m, neg_m);
          uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
          // own keys first (x[0, 64)), then -- one warp per quarter -- the other box (x[64, 128));
          // p packs in place: x[j/2] is already consumed
#pragma unroll
          for (int j = 0; j < kKeys / kHalves; j += 2) {
            const uint64_t yv = ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, m2);
            float y0, y1;
            unpack_f32x2(yv, y0, y1);
            const float p0 = ex2_approx(y0), p1 = ex2_approx(y1);
            const uint64_t pp = pack_f32x2(p0, p1);
            switch ((j >> 1) & 3) {
              case 0: s0 = fadd2(s0, pp); break;
              case 1: s1 = fadd2(s1, pp); break;
              case 2: s2 = fadd2(s2, pp); break;
              default: s3 = fadd2(s3, pp); break;
            }
            x[j >> 1] = pack_bf16x2(p0, p1);
          }
          ptrace(tr0, t, 4 + (__float_as_uint(x[0]) == 0x7fc00001u ? 1 : 0));
          float sa, sb;
          unpack_f32x2(fadd2(fadd2(s0, s1), fadd2(s2, s3)), sa, sb);
          l_run = l_run * alpha + (sa + sb);
        } else {
#pragma unroll
          for (int j = 0; j < kKeys / 2; ++j) x[j] = 0u;
        }
        if (kDB) {  // S(t) consumed (QK(t+2) may overwrite it)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctrl->s_free[t & 1]);
        }
        if (t > 0 && __any_sync(0xffffffffu, rescale)) {
          // single S: S(t) ready implies PV(t-1) retired; double-buffered: wait for PV(t-1)
          if (kDB) {
            mbar_wait(&ctrl->v_empty[(t - 1) % kStages], ((t - 1) / kStages) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < kD / kHalves; c += 32) {  // this half's O columns
            uint32_t o[32];
            const uint32_t oc = L::kColO + kh * (kD / kHalves) + c;
            tmem_ld32x32b_x32(tmem + lane_off + oc, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(u2f(o[j]) * alpha);
            tmem_st32x32b_x32(tmem + lane_off + oc, o);
          }
        }
        if (kHalves == 1) {
          tmem_st32x32b_x32(tmem + lane_off + p_col(t), x);
          tmem_st32x32b_x32(tmem + lane_off + p_col(t) + 32, x + 32);
        } else {
          tmem_st32x32b_x32(tmem + lane_off + p_col(t) + kh * 32, x);  // P of this half's 64 keys
        }
        tmem_wait_st();
        ptrace(tr0, t, 6);
        tc_fence_before();
        mbar_arrive(&ctrl->p_full[t & 1]);
        continue;
      }
      const int box = d.box[half];
      int hi = 0;
      if (box >= 0 && q < S) hi = min(d.width[half], q - box + 1);  // causal inside the block
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);
      const bool warp_skip = !__any_sync(0xffffffffu, hi > 0);
      mbar_wait(&ctrl->s_full[t & 1], (t >> 1) & 1);  // also orders P(t) after QK(t)
      tc_fence_after();
      uint32_t ph[32];
      float alpha = 1.f;
      bool rescale = false;
      if (!warp_skip) {
        uint32_t x[kBox];
        tmem_ld32x32b_x64(tmem + lane_off + s_col(t) + half * kBox, x);
        tmem_wait_ld();
        if (hi < kBox) {
#pragma unroll
          for (int j = 0; j < kBox; ++j) x[j] = j < hi ? x[j] : 0xff800000u;
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int j = 0; j < kBox; j += 8) {
          mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
          mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
          mx2 = fmax3(mx2, u2f(x[j + 4]), u2f(x[j + 5]));
          mx3 = fmax3(mx3, u2f(x[j + 6]), u2f(x[j + 7]));
        }
        const float mx = fmax3(mx0, mx1, fmaxf(mx2, mx3));
        if (hi > 0) {
          const float m_tile = mx * scale_log2;
          if (m_run == -INFINITY) {
            m_run = m_tile;
          } else if (m_tile > m_run + 8.f) {
            alpha = exp2f(m_run - m_tile);
            m_run = m_tile;
            rescale = true;
          }
        }
        const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
        const uint64_t c2 = pack_f32x2(scale_log2, scale_log2);
        const uint64_t m2 = pack_f32x2(neg_m, neg_m);
        uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
        for (int j = 0; j < kBox; j += 2) {
          const uint64_t yv = ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, m2);
          float y0, y1;
          unpack_f32x2(yv, y0, y1);
          const float p0 = ex2_approx(y0), p1 = ex2_approx(y1);
          const uint64_t pp = pack_f32x2(p0, p1);
          switch ((j >> 1) & 3) {
            case 0: s0 = fadd2(s0, pp); break;
            case 1: s1 = fadd2(s1, pp); break;
            case 2: s2 = fadd2(s2, pp); break;
            default: s3 = fadd2(s3, pp); break;
          }
          ph[j >> 1] = pack_bf16x2(p0, p1);
        }
        float sa, sb;
        unpack_f32x2(fadd2(fadd2(s0, s1), fadd2(s2, s3)), sa, sb);
        l_run = l_run * alpha + (sa + sb);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) ph[j] = 0u;
      }
      if (kDB) {  // S(t) consumed (QK(t+2) may overwrite it)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctrl->s_free[t & 1]);
      }
      // O rescale needs PV(t-1) retired: in the single-buffered chain S(t) ready implies it;
      // double-buffered, S(t) implies PV(t-2), so wait for PV(t-1)'s V-stage release (the
      // previous phase of that stage, PV(t-3), is retired: no aliasing)
      if (t > 0 && __any_sync(0xffffffffu, rescale)) {
        if (kDB) {
          mbar_wait(&ctrl->v_empty[(t - 1) % kStages], ((t - 1) / kStages) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t o[32];
          tmem_ld32x32b_x32((tmem + lane_off + L::kColO) + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(u2f(o[j]) * alpha);
          tmem_st32x32b_x32((tmem + lane_off + L::kColO) + c, o);
        }
      }
      // P row: this block's 64 keys, zeros for the other block's 64 (bf16 pairs, K-major)
      uint32_t z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = 0u;
      // P(t)'s buffer was last read by PV(t-2), retired before QK(t) completed
      tmem_st32x32b_x32(tmem + lane_off + p_col(t) + half * 32, ph);
      tmem_st32x32b_x32(tmem + lane_off + p_col(t) + (half ^ 1) * 32, z);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctrl->p_full[t & 1]);
    }
    // ---- epilogue: O / l -> global (bf16) ----
    mbar_wait(&ctrl->o_ready, 0);
    tc_fence_after();
    if (kHalves > 1) {  // the halves' row sums
      ctrl->lsum[kh][row] = l_run;
      named_bar_sync(1, 128 * kHalves);
      l_run = ctrl->lsum[0][row] + ctrl->lsum[1][row];
    }
    const float inv = (t > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
    const int dout = p.d_out;
    const int64_t obase = ((int64_t)h * S + min(q, S - 1)) * dout;
    if (p.lse != nullptr && q < S && kh == 0)
      p.lse[(int64_t)h * S + q] = (t > 0 && l_run > 0.f) ? (m_run + log2f(l_run)) * 0.6931471805599453f : -INFINITY;
#pragma unroll
    for (int c = kh * (kD / kHalves); c < (kh + 1) * (kD / kHalves); c += 32) {
      uint32_t o[32];
      __syncwarp();
      tmem_ld32x32b_x32((tmem + lane_off + L::kColO) + c, o);
      tmem_wait_ld();
      if (q >= S) continue;
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + obase;
      if (dout == kD) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          int4 w;
          w.x = (int)pack_bf16x2(u2f(o[j]) * inv, u2f(o[j + 1]) * inv);
          w.y = (int)pack_bf16x2(u2f(o[j + 2]) * inv, u2f(o[j + 3]) * inv);
          w.z = (int)pack_bf16x2(u2f(o[j + 4]) * inv, u2f(o[j + 5]) * inv);
          w.w = (int)pack_bf16x2(u2f(o[j + 6]) * inv, u2f(o[j + 7]) * inv);
          *reinterpret_cast<int4*>(out + c + j) = w;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (c + j < dout) out[c + j] = __float2bfloat16_rn(u2f(o[j]) * inv);
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

// Per listed head: sum over the 128-row CTAs of |tiles(r0) U tiles(r1)| (union kernel steps) and
// max(n0, n1) (paired-box steps).  Grid (n_pair, kStatCtas), one warp per row-block pair; the
// shared tiles are counted by binary-searching r0's starts in r1's ascending list.
constexpr int kStatCtas = 32;
__global__ void __launch_bounds__(256) pair_stats_kernel(const AttnArgs p, int n_rows,
                                                          unsigned long long* __restrict__ stats) {
  const int h = p.pair_heads[blockIdx.x];
  if (h < 0 || h >= p.Hq) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pairs = (n_rows + 1) / 2;
  unsigned long long u_sum = 0, m_sum = 0;
  for (int pp = blockIdx.y * 8 + warp; pp < n_pairs; pp += gridDim.y * 8) {
    const int64_t row = (int64_t)h * n_rows + 2 * pp;
    const int64_t a0 = p.tile_offsets[row], n0 = p.tile_offsets[row + 1] - a0;
    const bool has1 = 2 * pp + 1 < n_rows;
    const int64_t a1 = has1 ? p.tile_offsets[row + 1] : 0, n1 = has1 ? p.tile_offsets[row + 2] - a1 : 0;
    int common = 0;
    for (int64_t i = lane; i < n0; i += 32) {
      const int x = p.tile_starts[a0 + i];
      int64_t lo = 0, hi = n1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (p.tile_starts[a1 + mid] < x) lo = mid + 1; else hi = mid;
      }
      common += (lo < n1 && p.tile_starts[a1 + lo] == x) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) common += __shfl_xor_sync(0xffffffffu, common, o);
    u_sum += (unsigned long long)(n0 + n1 - common);
    m_sum += (unsigned long long)(n0 > n1 ? n0 : n1);
  }
  if (lane == 0 && (u_sum | m_sum)) {
    atomicAdd(&stats[2 * blockIdx.x], u_sum);
    atomicAdd(&stats[2 * blockIdx.x + 1], m_sum);
  }
}

template <int kD>
int launch_pair_impl(const AttnArgs& a, cudaStream_t stream) {
  using L = PLayout<kD>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_tmap_bf16_3d(&tq, a.q_hi, kD, a.S, a.Hq, kRows))) return rc;
  if ((rc = make_tmap_bf16_3d(&tk, a.k_hi, kD, a.S, a.Hkv, kBox))) return rc;
  if ((rc = make_tmap_bf16_3d(&tv, a.v_hi, kD, a.S, a.Hkv, kBox))) return rc;
  auto kern = sparse_attn_pair_kernel<kD>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(pair attn smem)");
    attr_done = true;
  }
  const int n_ctile = (a.S + kRows - 1) / kRows;
  const long long grid = (long long)n_ctile * a.n_pair;
  if (grid == 0) return 0;
  if (grid > 0x7fffffffLL) return set_error(2, "attention grid too large");
  note_launches(1);
  kern<<<(unsigned)grid, kThreads, L::kSmem, stream>>>(tq, tk, tv, a, n_ctile, a.scale * 1.4426950408889634f);
  return check_cuda(cudaGetLastError(), "sparse_attn_pair launch");
}

}  // namespace

bool attn_pair_supported(const AttnArgs& a) {
  return !a.split && !a.out_f32 && a.B == kBox && (a.kD == 128 || a.kD == 64) && a.work_order == nullptr;
}

int launch_pair_stats(const AttnArgs& a, unsigned long long* stats, cudaStream_t stream) {
  int rc = check_cuda(cudaMemsetAsync(stats, 0, sizeof(unsigned long long) * 2 * a.n_pair, stream), "pair stats memset");
  if (rc) return rc;
  const int n_rows = (a.S + kBox - 1) / kBox;
  note_launches(1);
  pair_stats_kernel<<<dim3((unsigned)a.n_pair, kStatCtas), 256, 0, stream>>>(a, n_rows, stats);
  return check_cuda(cudaGetLastError(), "pair stats launch");
}

int launch_sparse_attn_pairs(const AttnArgs& a, cudaStream_t stream) {
  if (a.kD == 128) return launch_pair_impl<128>(a, stream);
  return launch_pair_impl<64>(a, stream);
}

}  // namespace spf

// Debug: point the SPF_PAIR_TRACE stamps at a device buffer of n_ctas * 64 * 8 uint64.
extern "C" int spf_debug_pair_trace(void* buf, int n_ctas) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  if (cudaMemcpyToSymbol(spf::g_ptrace, &p, sizeof(p)) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(spf::g_ptrace_ctas, &n_ctas, sizeof(int)) == cudaSuccess ? 0 : 1;
}
