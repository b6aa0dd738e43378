// attn_fwd.cu -- sparse FlashAttention forward over a per-row tile/column layout
// (the hot kernel of the MInference pre-fill path), hand-written for sm_100a.
//
// Semantics follow the reference kernel contract exactly
// (/root/reference/pkg/src/sparseprefill/_core.pyx:72-192 and _core_py.py:17-66):
//   * for every query-block row r (B query rows) the row's tiles are visited,
//     tile keys = [max(s,0), min(s+B,S)), per-cell causal mask key <= query;
//   * then the row's residual columns in chips of B, the allowed keys of a
//     query being the leading columns <= query (_core.pyx:172-179);
//   * one streaming-softmax state per query row; out = acc / l, zero row if l == 0.
//
// B200 design:
//   * one CTA = 128 query rows of one q-head (UMMA M = 128).  The row blocks
//     it covers (2 when B = 64) are merged into one union step list; each step
//     carries a segment mask so a row block never sees another block's keys.
//   * step = 64 keys: a TMA-loaded box of K/V (tiles) or a warp-gathered chip
//     of K/V rows (columns), double-buffered in shared memory;
//   * S = Q K^T   : tcgen05.mma M128 N64 K=d, fp32 accumulator in TMEM
//                   (two S buffers so QK(t+1) overlaps softmax(t));
//   * O += P V    : tcgen05.mma M128 N=d K64, P bf16 in SW128 smem, V MN-major,
//                   fp32 accumulator resident in TMEM for the whole row tile;
//   * warp roles: warp0 = loader (TMA + gathers + union merge), warp1 = MMA
//     issuer (one thread) + TMEM owner, warps2-5 = softmax (thread <-> row).
//   * online softmax in the exp2 domain with lazy rescaling (only when the
//     running max grows by > 8, i.e. p <= 256); results are identical up to
//     rounding to the reference's exact-max recurrence.
//   * fp32 I/O (the drop-in numpy path) runs the same kernel on a bf16x2 split
//     (x = hi + lo, three products per GEMM) so it stays on the tensor cores
//     while meeting the 1e-3 relative tolerance.
#include "spf_internal.h"
#include "spf_ptx.cuh"

#include <math.h>

namespace spf {

namespace {

constexpr int kRows = 128;   // query rows per CTA
constexpr int kBox = 64;     // keys per step
constexpr int kStages = 2;   // K/V stages
constexpr int kThreads = 192;

enum : int { kTile = 0, kChip = 1, kEnd = 2 };

struct StepDesc {
  int kind;
  int box;     // tile: first key of the loaded box
  int width;   // tile: valid keys in the box ([box, box+width)); chip: number of keys
  int pad;
  unsigned long long segmask;
  int pmax[kBox];  // chip: running max of the chip's keys (prefix rule)
};

struct Ctrl {
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[2];
  uint64_t s_empty[2];
  uint64_t p_full;
  uint64_t pv_done;
  uint32_t tmem_base;
  uint32_t pad;
  StepDesc desc[kStages];
};

template <int kD, bool kSplit>
struct Layout {
  static constexpr int kCopies = kSplit ? 2 : 1;
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQBytes = kRows * kD * 2;   // one copy
  static constexpr int kKBytes = kBox * kD * 2;    // one copy of K (or V) per stage
  static constexpr int kPBytes = kRows * kBox * 2;
  static constexpr int kOffQ = 0;
  static constexpr int kOffStage = kOffQ + kCopies * kQBytes;
  static constexpr int kStageBytes = 2 * kCopies * kKBytes;  // K copies then V copies
  static constexpr int kOffP = kOffStage + kStages * kStageBytes;
  static constexpr int kOffCtrl = kOffP + kCopies * kPBytes;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(Ctrl);
  static constexpr uint32_t kTxStage = 2u * kCopies * kKBytes;
  static constexpr uint32_t kTxQ = kCopies * kQBytes;
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

template <int kD, bool kSplit>
__global__ void __launch_bounds__(kThreads, kSplit ? 1 : 2)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_q2,
                           const __grid_constant__ CUtensorMap tm_k2, const __grid_constant__ CUtensorMap tm_v2,
                           const AttnArgs p, int n_ctile, float scale_log2) {
  using L = Layout<kD, kSplit>;
  extern __shared__ __align__(1024) uint8_t smem[];
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work item: heavy (late) row tiles first, heads fastest --------------------
  int item = blockIdx.x;
  if (p.work_order != nullptr) item = p.work_order[item];
  const int ct = n_ctile - 1 - item / p.Hq;
  const int h = item % p.Hq;
  const int kvh = h / (p.Hq / p.Hkv);
  const int S = p.S, B = p.B;
  const int n_rows = (S + B - 1) / B;
  const int R0 = ct * kRows;
  const int r_first = R0 / B;
  const int r_last = min((R0 + kRows - 1) / B, n_rows - 1);
  const int G = r_last - r_first + 1;  // <= 64 (host checks B >= 2)

  if (threadIdx.x == 0) {
    if ((sbase & 1023u) != 0) {
      printf("spf: dynamic smem not 1024-aligned\n");
      __trap();
    }
    mbar_init(&ctrl->q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&ctrl->kv_full[s], 1);
      mbar_init(&ctrl->kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->s_full[s], 1);
      mbar_init(&ctrl->s_empty[s], 128);
    }
    mbar_init(&ctrl->p_full, 128);
    mbar_init(&ctrl->pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&ctrl->tmem_base, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctrl->tmem_base;

  if (warp == 0) {
    // =============================== loader warp ===============================
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(&ctrl->q_full, L::kTxQ);
#pragma unroll
      for (int a = 0; a < L::kAtoms; ++a) {
        tma_load_3d(smem + L::kOffQ + a * (kRows * 128), &tm_q, &ctrl->q_full, a * 64, R0, h);
        if (kSplit) tma_load_3d(smem + L::kOffQ + L::kQBytes + a * (kRows * 128), &tm_q2, &ctrl->q_full, a * 64, R0, h);
      }
    }
    const int64_t row0 = (int64_t)h * n_rows + r_first;
    int64_t pos[64], endp[64];
    int cur[64];
    for (int g = 0; g < G; ++g) {
      pos[g] = p.tile_offsets[row0 + g];
      endp[g] = p.tile_offsets[row0 + g + 1];
      cur[g] = pos[g] < endp[g] ? p.tile_starts[pos[g]] : INT_MAX;
    }
    int t = 0;
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_hi) + (int64_t)kvh * S * kD;
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_hi) + (int64_t)kvh * S * kD;
    const __nv_bfloat16* kb2 = kSplit ? reinterpret_cast<const __nv_bfloat16*>(p.k_lo) + (int64_t)kvh * S * kD : nullptr;
    const __nv_bfloat16* vb2 = kSplit ? reinterpret_cast<const __nv_bfloat16*>(p.v_lo) + (int64_t)kvh * S * kD : nullptr;

    // --- tiles: union over the G row blocks, ascending start ---
    while (true) {
      int best = INT_MAX;
      for (int g = 0; g < G; ++g) best = min(best, cur[g]);
      if (best == INT_MAX) break;
      unsigned long long mask = 0ull;
      for (int g = 0; g < G; ++g) {
        if (cur[g] == best) {
          mask |= 1ull << g;
          ++pos[g];
          cur[g] = pos[g] < endp[g] ? p.tile_starts[pos[g]] : INT_MAX;
        }
      }
      for (int sub = 0; sub * kBox < B; ++sub) {
        const int st = t % kStages;
        if (lane == 0) {
          mbar_wait(&ctrl->kv_empty[st], ((t / kStages) & 1) ^ 1);
          StepDesc& d = ctrl->desc[st];
          d.kind = kTile;
          d.box = best + sub * kBox;
          d.width = min(kBox, B - sub * kBox);
          d.segmask = mask;
          uint8_t* kst = smem + L::kOffStage + st * L::kStageBytes;
          uint8_t* vst = kst + L::kCopies * L::kKBytes;
          mbar_arrive_expect_tx(&ctrl->kv_full[st], L::kTxStage);
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a) {
            tma_load_3d(kst + a * (kBox * 128), &tm_k, &ctrl->kv_full[st], a * 64, best + sub * kBox, kvh);
            tma_load_3d(vst + a * (kBox * 128), &tm_v, &ctrl->kv_full[st], a * 64, best + sub * kBox, kvh);
            if (kSplit) {
              tma_load_3d(kst + L::kKBytes + a * (kBox * 128), &tm_k2, &ctrl->kv_full[st], a * 64, best + sub * kBox, kvh);
              tma_load_3d(vst + L::kKBytes + a * (kBox * 128), &tm_v2, &ctrl->kv_full[st], a * 64, best + sub * kBox, kvh);
            }
          }
        }
        __syncwarp();
        ++t;
      }
    }
    // --- column chips: per row block, chips of B columns, split in 64-key steps ---
    for (int g = 0; g < G; ++g) {
      const int64_t cb = p.col_offsets[row0 + g], ce = p.col_offsets[row0 + g + 1];
      for (int64_t c0 = cb; c0 < ce; c0 += B) {
        const int64_t chip_end = min(c0 + (int64_t)B, ce);
        int running = INT_MIN;
        for (int64_t s0 = c0; s0 < chip_end; s0 += kBox) {
          const int n = (int)min((int64_t)kBox, chip_end - s0);
          const int st = t % kStages;
          if (lane == 0) mbar_wait(&ctrl->kv_empty[st], ((t / kStages) & 1) ^ 1);
          __syncwarp();
          StepDesc& d = ctrl->desc[st];
          // prefix max of the keys (two 32-wide warp scans)
          int key_a = lane < n ? p.col_indices[s0 + lane] : INT_MIN;
          int key_b = lane + 32 < n ? p.col_indices[s0 + lane + 32] : INT_MIN;
          int pa = key_a, pb = key_b;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            int xa = __shfl_up_sync(0xffffffffu, pa, off);
            int xb = __shfl_up_sync(0xffffffffu, pb, off);
            if (lane >= off) { pa = max(pa, xa); pb = max(pb, xb); }
          }
          pa = max(pa, running);
          const int tail_a = __shfl_sync(0xffffffffu, pa, 31);
          pb = max(pb, tail_a);
          d.pmax[lane] = pa;
          d.pmax[lane + 32] = pb;
          running = __shfl_sync(0xffffffffu, pb, 31);
          if (lane == 0) {
            d.kind = kChip;
            d.box = 0;
            d.width = n;
            d.segmask = 1ull << g;
          }
          // gather K/V rows (16-byte chunks), writing the SW128 layout by hand
          uint8_t* kst = smem + L::kOffStage + st * L::kStageBytes;
          uint8_t* vst = kst + L::kCopies * L::kKBytes;
          constexpr int kChunksPerRow = kD / 8;
          for (int idx = lane; idx < kBox * kChunksPerRow; idx += 32) {
            const int j = idx / kChunksPerRow;
            const int c16 = idx % kChunksPerRow;
            const int atom = c16 >> 3, c = c16 & 7;
            const uint32_t off = atom * (kBox * 128) + (j >> 3) * 1024 + (j & 7) * 128 + ((c ^ (j & 7)) << 4);
            int4 kv = make_int4(0, 0, 0, 0), vv = make_int4(0, 0, 0, 0);
            int4 kv2 = make_int4(0, 0, 0, 0), vv2 = make_int4(0, 0, 0, 0);
            if (j < n) {
              const int key = p.col_indices[s0 + j];
              const int64_t e = (int64_t)key * kD + c16 * 8;
              kv = __ldg(reinterpret_cast<const int4*>(kb + e));
              vv = __ldg(reinterpret_cast<const int4*>(vb + e));
              if (kSplit) {
                kv2 = __ldg(reinterpret_cast<const int4*>(kb2 + e));
                vv2 = __ldg(reinterpret_cast<const int4*>(vb2 + e));
              }
            }
            *reinterpret_cast<int4*>(kst + off) = kv;
            *reinterpret_cast<int4*>(vst + off) = vv;
            if (kSplit) {
              *reinterpret_cast<int4*>(kst + L::kKBytes + off) = kv2;
              *reinterpret_cast<int4*>(vst + L::kKBytes + off) = vv2;
            }
          }
          fence_proxy_async_smem();
          __threadfence_block();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctrl->kv_full[st]);
          ++t;
        }
      }
    }
    // --- end marker ---
    {
      const int st = t % kStages;
      if (lane == 0) {
        mbar_wait(&ctrl->kv_empty[st], ((t / kStages) & 1) ^ 1);
        ctrl->desc[st].kind = kEnd;
        mbar_arrive(&ctrl->kv_full[st]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // =============================== MMA issuer ================================
    if (lane == 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(128, kBox, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, kD, 0, 1);
      const uint32_t q_addr = sbase + L::kOffQ;
      const uint32_t p_addr = sbase + L::kOffP;
      const uint32_t tO = tmem + 128;
      mbar_wait(&ctrl->q_full, 0);
      tc_fence_after();

      auto issue_pv = [&](int u) {
        mbar_wait(&ctrl->p_full, u & 1);
        tc_fence_after();
        const int st = u % kStages;
        const uint32_t v_addr = sbase + L::kOffStage + st * L::kStageBytes + L::kCopies * L::kKBytes;
#pragma unroll
        for (int k = 0; k < kBox / 16; ++k) {
          const uint64_t a_hi = umma_desc_sw128(p_addr + k * 32, 0, 1024);
          const uint64_t b_hi = umma_desc_sw128(v_addr + k * 2048, kBox * 128, 1024);
          mma_bf16_ss(tO, a_hi, b_hi, idesc_pv, (u > 0 || k > 0) ? 1u : 0u);
          if (kSplit) {
            const uint64_t a_lo = umma_desc_sw128(p_addr + L::kPBytes + k * 32, 0, 1024);
            const uint64_t b_lo = umma_desc_sw128(v_addr + L::kKBytes + k * 2048, kBox * 128, 1024);
            mma_bf16_ss(tO, a_hi, b_lo, idesc_pv, 1u);
            mma_bf16_ss(tO, a_lo, b_hi, idesc_pv, 1u);
          }
        }
        mma_commit(&ctrl->pv_done);
        mma_commit(&ctrl->kv_empty[st]);
      };

      int t = 0;
      for (;; ++t) {
        const int st = t % kStages;
        mbar_wait(&ctrl->kv_full[st], (t / kStages) & 1);
        const int kind = *reinterpret_cast<volatile int*>(&ctrl->desc[st].kind);
        if (kind == kEnd) break;
        const int sb = t & 1;
        mbar_wait(&ctrl->s_empty[sb], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = sbase + L::kOffStage + st * L::kStageBytes;
        const uint32_t tS = tmem + sb * kBox;
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const int atom = k >> 2;
          const uint32_t koff = (k & 3) * 32;
          const uint64_t a_hi = umma_desc_sw128(q_addr + atom * (kRows * 128) + koff, 0, 1024);
          const uint64_t b_hi = umma_desc_sw128(k_addr + atom * (kBox * 128) + koff, 0, 1024);
          mma_bf16_ss(tS, a_hi, b_hi, idesc_qk, k > 0 ? 1u : 0u);
          if (kSplit) {
            const uint64_t a_lo = umma_desc_sw128(q_addr + L::kQBytes + atom * (kRows * 128) + koff, 0, 1024);
            const uint64_t b_lo = umma_desc_sw128(k_addr + L::kKBytes + atom * (kBox * 128) + koff, 0, 1024);
            mma_bf16_ss(tS, a_hi, b_lo, idesc_qk, 1u);
            mma_bf16_ss(tS, a_lo, b_hi, idesc_qk, 1u);
          }
        }
        mma_commit(&ctrl->s_full[sb]);
        if (t > 0) issue_pv(t - 1);
      }
      if (t > 0) issue_pv(t - 1);
    }
    __syncwarp();
  } else {
    // =============================== softmax warps =============================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = R0 + row;
    const int seg = (q < S) ? (q / B - r_first) : -1;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t p_row = sbase + L::kOffP + (row >> 3) * 1024 + (row & 7) * 128;
    const int sw = row & 7;
    float m_run = -INFINITY, l_run = 0.f;
    int t = 0;
    for (;; ++t) {
      const int st = t % kStages;
      mbar_wait(&ctrl->kv_full[st], (t / kStages) & 1);
      const StepDesc& d = ctrl->desc[st];
      const int kind = d.kind;
      if (kind == kEnd) break;
      const int sb = t & 1;
      mbar_wait(&ctrl->s_full[sb], (t >> 1) & 1);
      tc_fence_after();
      uint32_t x[kBox];
      tmem_ld32x32b_x64(tmem + lane_off + sb * kBox, x);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&ctrl->s_empty[sb]);

      // valid key slots for this row: a contiguous range [lo, hi)
      int lo = 0, hi = 0;
      if (seg >= 0 && ((d.segmask >> seg) & 1ull)) {
        if (kind == kTile) {
          lo = max(0, -d.box);
          hi = min(d.width, min(S - d.box, q - d.box + 1));
        } else {
          int a = 0, b = d.width;
          while (a < b) {
            const int m = (a + b) >> 1;
            if (d.pmax[m] <= q) a = m + 1; else b = m;
          }
          hi = a;
        }
      }
      // branch-free masking: invalid slots become -inf (ex2(-inf) = +0)
      if (!(lo == 0 && hi == kBox)) {
#pragma unroll
        for (int j = 0; j < kBox; ++j) x[j] = (j >= lo && j < hi) ? x[j] : 0xff800000u;
      }
      // row max: four independent 3-input max chains (FMNMX3)
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int j = 0; j < kBox; j += 8) {
        mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
        mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
        mx2 = fmax3(mx2, u2f(x[j + 4]), u2f(x[j + 5]));
        mx3 = fmax3(mx3, u2f(x[j + 6]), u2f(x[j + 7]));
      }
      const float mx = fmax3(mx0, mx1, fmaxf(mx2, mx3));
      float alpha = 1.f;
      bool rescale = false;
      if (hi > lo) {
        const float m_tile = mx * scale_log2;
        if (m_run == -INFINITY) {
          m_run = m_tile;
        } else if (m_tile > m_run + 8.f) {
          alpha = exp2f(m_run - m_tile);
          m_run = m_tile;
          rescale = true;
        }
      }
      uint32_t ph[kBox / 2];
      uint32_t pl[kSplit ? kBox / 2 : 1];
      // p = 2^(x*c - m): packed FFMA2, MUFU ex2, packed FADD2 row sums
      const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
      const uint64_t c2 = pack_f32x2(scale_log2, scale_log2);
      const uint64_t m2 = pack_f32x2(neg_m, neg_m);
      uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
      for (int j = 0; j < kBox; j += 2) {
        const uint64_t y = ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, m2);
        float y0, y1;
        unpack_f32x2(y, y0, y1);
        const float p0 = ex2_approx(y0), p1 = ex2_approx(y1);
        const uint64_t pp = pack_f32x2(p0, p1);
        switch ((j >> 1) & 3) {
          case 0: s0 = fadd2(s0, pp); break;
          case 1: s1 = fadd2(s1, pp); break;
          case 2: s2 = fadd2(s2, pp); break;
          default: s3 = fadd2(s3, pp); break;
        }
        ph[j >> 1] = pack_bf16x2(p0, p1);
        if (kSplit) {
          const __nv_bfloat162 hb = *reinterpret_cast<const __nv_bfloat162*>(&ph[j >> 1]);
          const float2 hf = __bfloat1622float2(hb);
          pl[j >> 1] = pack_bf16x2(p0 - hf.x, p1 - hf.y);
        }
      }
      float sa, sb2;
      unpack_f32x2(fadd2(fadd2(s0, s1), fadd2(s2, s3)), sa, sb2);
      const float sum = sa + sb2;
      l_run = l_run * alpha + sum;

      if (t > 0) {
        mbar_wait(&ctrl->pv_done, (t - 1) & 1);
        tc_fence_after();
        // tcgen05.ld/st are warp-collective (.sync.aligned): decide per warp.
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < kD; c += 32) {
            uint32_t o[32];
            tmem_ld32x32b_x32(tmem + lane_off + 128 + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(u2f(o[j]) * alpha);
            tmem_st32x32b_x32(tmem + lane_off + 128 + c, o);
          }
          tmem_wait_st();
        }
      }
      // P row -> SW128 K-major smem (chunk c of 8 keys lands at chunk c ^ (row & 7))
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        st_shared_v4(p_row + ((c ^ sw) << 4), ph[4 * c], ph[4 * c + 1], ph[4 * c + 2], ph[4 * c + 3]);
        if (kSplit)
          st_shared_v4(p_row + L::kPBytes + ((c ^ sw) << 4), pl[4 * c], pl[4 * c + 1], pl[4 * c + 2], pl[4 * c + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&ctrl->p_full);
    }
    // ---- epilogue: O / l -> global ----
    if (t > 0) {
      mbar_wait(&ctrl->pv_done, (t - 1) & 1);
      tc_fence_after();
    }
    {
      const float inv = (t > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
      const int dout = p.d_out;
      const int64_t obase = ((int64_t)h * S + min(q, S - 1)) * dout;
#pragma unroll
      for (int c = 0; c < kD; c += 32) {
        uint32_t o[32];
        __syncwarp();
        if (t > 0) {  // warp-uniform: every lane loads, only rows < S store
          tmem_ld32x32b_x32(tmem + lane_off + 128 + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0u;
        }
        if (q >= S) {
        } else if (p.out_f32) {
          float* out = reinterpret_cast<float*>(p.out) + obase;
          if (dout == kD) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(out + c + j) =
                  make_float4(u2f(o[j]) * inv, u2f(o[j + 1]) * inv, u2f(o[j + 2]) * inv, u2f(o[j + 3]) * inv);
          } else {
            for (int j = 0; j < 32; ++j)
              if (c + j < dout) out[c + j] = u2f(o[j]) * inv;
          }
        } else {
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
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int kD, bool kSplit>
int launch_impl(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout<kD, kSplit>;
  CUtensorMap tq, tk, tv, tq2, tk2, tv2;
  int rc;
  if ((rc = make_tmap_bf16_3d(&tq, a.q_hi, kD, a.S, a.Hq, kRows))) return rc;
  if ((rc = make_tmap_bf16_3d(&tk, a.k_hi, kD, a.S, a.Hkv, kBox))) return rc;
  if ((rc = make_tmap_bf16_3d(&tv, a.v_hi, kD, a.S, a.Hkv, kBox))) return rc;
  if (kSplit) {
    if ((rc = make_tmap_bf16_3d(&tq2, a.q_lo, kD, a.S, a.Hq, kRows))) return rc;
    if ((rc = make_tmap_bf16_3d(&tk2, a.k_lo, kD, a.S, a.Hkv, kBox))) return rc;
    if ((rc = make_tmap_bf16_3d(&tv2, a.v_lo, kD, a.S, a.Hkv, kBox))) return rc;
  } else {
    tq2 = tq;
    tk2 = tk;
    tv2 = tv;
  }
  auto kern = sparse_attn_fwd_kernel<kD, kSplit>;
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(attn smem)");
    attr_done = true;
  }
  const int n_ctile = (a.S + kRows - 1) / kRows;
  const long long grid = (long long)n_ctile * a.Hq;
  if (grid == 0) return 0;
  if (grid > 0x7fffffffLL) return set_error(2, "attention grid too large");
  const float scale_log2 = a.scale * 1.4426950408889634f;
  note_launches(1);
  kern<<<(unsigned)grid, kThreads, L::kSmem, stream>>>(tq, tk, tv, tq2, tk2, tv2, a, n_ctile, scale_log2);
  return check_cuda(cudaGetLastError(), "sparse_attn_fwd launch");
}

}  // namespace

int launch_sparse_attn(const AttnArgs& a, cudaStream_t stream) {
  if (a.B < 2) return set_error(2, "block_size must be >= 2 for the sm_100a kernel (got %d)", a.B);
  if (a.Hkv <= 0 || a.Hq % a.Hkv != 0) return set_error(2, "n_q_heads must be a multiple of n_kv_heads");
  if (a.kD == 128) return a.split ? launch_impl<128, true>(a, stream) : launch_impl<128, false>(a, stream);
  if (a.kD == 64) return a.split ? launch_impl<64, true>(a, stream) : launch_impl<64, false>(a, stream);
  return set_error(2, "padded head_dim must be 64 or 128 (got %d)", a.kD);
}

}  // namespace spf
