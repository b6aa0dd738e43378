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
//   * one CTA = 128 query rows of one q-head (UMMA M = 128), two CTAs per SM.  The row
//     blocks it covers (2 when B = 64) are merged into one union step list; each step
//     carries a segment mask so a row block never sees another block's keys.
//   * step = 64 keys: a TMA-loaded box of K/V (tiles) or a cp.async-gathered chip of
//     K/V rows (columns), in 3-deep K / 2-deep V rings in shared memory;
//   * S = Q K^T   : tcgen05.mma M128 N64 K=d, fp32 accumulator in TMEM columns [0,64),
//                   released as soon as the softmax has read it so QK(t+1) overlaps
//                   softmax(t);
//   * O += P V    : tcgen05.mma M128 N=d K64 with A = P (bf16, its own double-buffered
//                   TMEM columns [64,128)), V MN-major from shared memory, fp32 O resident
//                   in TMEM [128,256) for the whole row tile; the epilogue stages O / l in
//                   the idle K ring and writes it with tensor-map stores;
//   * warp roles: warp0 = loader (TMA + gathers + union merge), warp1 = MMA
//     issuer (elected lane) + TMEM owner, warps2-5 = softmax (thread <-> row).
//   * online softmax in the exp2 domain with lazy rescaling (only when the
//     running max grows by > 8, i.e. p <= 256); results are identical up to
//     rounding to the reference's exact-max recurrence.
//   * fp32 I/O (the drop-in numpy path) runs the same kernel on a bf16x2 split
//     (x = hi + lo, three products per GEMM) so it stays on the tensor cores
//     while meeting the 1e-3 relative tolerance.
#include "spf_internal.h"
#include "spf_ptx.cuh"

#include <math.h>
#include <stdlib.h>

namespace spf {

namespace {

constexpr int kRows = 128;   // query rows per CTA
constexpr int kBox = 64;     // keys per step

enum : int { kTile = 0, kChip = 1, kEnd = 2 };


struct StepDesc {
  unsigned long long segmask;
  int box;      // tile: first key of the loaded box
  short kind;
  short width;  // tile: valid keys in the box ([box, box+width)); chip: number of keys
  int pmax[kBox];  // chip: running max of the chip's keys (prefix rule)
};

// Ring depths: K is loaded one step ahead of V and released as soon as its
// QK^T completes, so it gets the deeper ring; V (and the step descriptor that
// travels with it) is released after PV.
// TMEM columns (256 per CTA, two CTAs per SM): bf16 path = S [0,64) single-buffered,
// P(t) in [64 + 32*(t&1), +32) (separate, so QK(t+1) only waits for the softmax to READ
// S(t), not for PV(t)), O [128,256).  The split (fp32 I/O) path needs 64 P columns per
// step and keeps P over S with two S buffers: S/P [0,64) and [64,128), O [128,256).
template <bool kSplit>
constexpr bool kSepP = !kSplit;

// One softmax warp per TMEM lane quarter (two, each exponentiating half a row, was
// measured 14 % slower on C2: more warps per SMSP delay the MMA and loader warps more
// than the shorter softmax helps).
template <bool kSplit>
constexpr int kSoftHalves = 1;
template <bool kSplit>
constexpr int kThreadsT = 64 + 128 * kSoftHalves<kSplit>;

template <bool kSplit>
struct Rings {
  static constexpr int kK = kSplit ? 2 : 3;
  static constexpr int kV = 2;
  static constexpr int kD = 3;  // step descriptors: written with K (one step ahead), freed by the softmax
};

template <bool kSplit>
struct Ctrl {
  uint64_t q_full;
  uint64_t k_full[Rings<kSplit>::kK];
  uint64_t k_empty[Rings<kSplit>::kK];
  uint64_t v_full[Rings<kSplit>::kV];
  uint64_t v_empty[Rings<kSplit>::kV];
  uint64_t d_full[Rings<kSplit>::kD];
  uint64_t d_empty[Rings<kSplit>::kD];
  // split layout: S/P buffers 0 and 1.  Separate-P layout: [0] = the single S buffer
  // written / read ([1] unused; PV issued two steps behind QK measured 3.7 % slower,
  // profiles/r01/attn_bottleneck_experiments.txt).
  uint64_t s_full[2];
  uint64_t s_free[2];
  // P(t) written, one barrier per S/P buffer: a softmax warp can run one step ahead
  // of another, and a single barrier would let its step-(t+1) arrivals complete
  // step t's phase before the slow warp's P(t) is in TMEM
  uint64_t p_full[2];
  uint64_t o_ready;  // all PVs retired (committed once after the last one)
  uint32_t tmem_base;
  uint32_t pad;
  StepDesc desc[Rings<kSplit>::kD];
};
// two CTAs per SM need kSmem <= 115712 B (228 KB minus 1 KB reserved per CTA)
static_assert(sizeof(Ctrl<false>) <= 1024, "control block too large for two CTAs per SM");

template <int kD, bool kSplit>
struct Layout {
  static constexpr int kCopies = kSplit ? 2 : 1;
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQBytes = kRows * kD * 2;   // one copy
  static constexpr int kKBytes = kBox * kD * 2;    // one copy of one K (or V) tile
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kCopies * kQBytes;
  static constexpr int kOffV = kOffK + Rings<kSplit>::kK * kCopies * kKBytes;
  static constexpr int kOffCtrl = kOffV + Rings<kSplit>::kV * kCopies * kKBytes;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(Ctrl<kSplit>);
  static constexpr uint32_t kTxKV = kCopies * kKBytes;
  static constexpr uint32_t kTxQ = kCopies * kQBytes;
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

// One step of the loader's schedule.
struct StepInfo {
  int kind;
  int box, width;
  unsigned long long mask;
  int64_t s0;  // chip: first column index (into col_indices)
  int n;       // chip: keys in this step
  bool first;  // chip: first 64-key step of a chip (prefix max restarts)
};

template <int kD, bool kSplit>
__global__ void __launch_bounds__(kThreadsT<kSplit>, kSplit ? 1 : 2)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_q2,
                           const __grid_constant__ CUtensorMap tm_k2, const __grid_constant__ CUtensorMap tm_v2,
                           const __grid_constant__ CUtensorMap tm_o, const AttnArgs p, int n_ctile,
                           float scale_log2) {
  using L = Layout<kD, kSplit>;
  using R = Rings<kSplit>;
  extern __shared__ __align__(1024) uint8_t smem[];
  Ctrl<kSplit>* ctrl = reinterpret_cast<Ctrl<kSplit>*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work item: heavy (late) row tiles first, heads fastest (a kv-head-major order, as the
  // paired-box kernel uses for the scattered Block-Sparse tiles, measured 0.7-1.1 % slower on
  // C2-shaped VS / A-shape layers: their K/V windows are local) ----------------------------
  int item = blockIdx.x;
  if (p.work_order != nullptr) item = p.work_order[item];
  const int ct = n_ctile - 1 - item / p.Hq;
  const int h = item % p.Hq;
  const int kvh = h / (p.Hq / p.Hkv);
  // routed to the paired-box kernel (attn_bs.cu)?  The first listed entry of this head decides;
  // every warp scans the list 32 entries per ballot (the same answer in all warps)
  for (int base = 0; base < p.n_pair; base += 32) {
    const int i = base + (threadIdx.x & 31);
    const unsigned m = __ballot_sync(0xffffffffu, i < p.n_pair && p.pair_heads[i] == h);
    if (m) {
      if (pair_preferred(p.pair_stats, base + __ffs(m) - 1)) return;
      break;
    }
  }
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
    for (int s = 0; s < R::kK; ++s) {
      mbar_init(&ctrl->k_full[s], 1);
      mbar_init(&ctrl->k_empty[s], 1);
    }
    for (int s = 0; s < R::kV; ++s) {
      mbar_init(&ctrl->v_full[s], 1);
      mbar_init(&ctrl->v_empty[s], 1);
    }
    for (int s = 0; s < R::kD; ++s) {
      mbar_init(&ctrl->d_full[s], 1);
      mbar_init(&ctrl->d_empty[s], 4 * kSoftHalves<kSplit>);  // one arrival per softmax warp
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->s_full[s], 1);
      // separate-P layout: S is released by the softmax warps once read (one arrival each)
      mbar_init(&ctrl->s_free[s], (kSepP<kSplit> && s == 0) ? 4 * kSoftHalves<kSplit> : 1);
    }
    mbar_init(&ctrl->p_full[0], 128 * kSoftHalves<kSplit>);
    mbar_init(&ctrl->p_full[1], 128 * kSoftHalves<kSplit>);
    mbar_init(&ctrl->o_ready, 1);
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
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_hi) + (int64_t)kvh * S * kD;
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_hi) + (int64_t)kvh * S * kD;
    const __nv_bfloat16* kb2 = kSplit ? reinterpret_cast<const __nv_bfloat16*>(p.k_lo) + (int64_t)kvh * S * kD : nullptr;
    const __nv_bfloat16* vb2 = kSplit ? reinterpret_cast<const __nv_bfloat16*>(p.v_lo) + (int64_t)kvh * S * kD : nullptr;

    // ---- step generator (warp-uniform) ----
    // Tiles: union over the G row blocks, DESCENDING start (the diagonal tile first,
    // so the running max is set early and lazy rescales are rare).  Lane l walks the
    // lists of row blocks l and l + 32 from their ends, holding the next kBuf starts
    // in registers; one warp max-reduction per union tile.
    constexpr int kBuf = 8;
    int cur[2], bn[2];
    int64_t nxt[2], beg[2];
    int buf[2][kBuf];
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int g = lane + 32 * sl;
      beg[sl] = g < G ? p.tile_offsets[row0 + g] : 0;
      nxt[sl] = (g < G ? p.tile_offsets[row0 + g + 1] : 0) - 1;  // next index to fetch (descending)
      bn[sl] = 0;
    }
    auto refill = [&](int sl) {
#pragma unroll
      for (int u = 0; u < kBuf; ++u) buf[sl][u] = (nxt[sl] - u >= beg[sl]) ? p.tile_starts[nxt[sl] - u] : INT_MIN;
      const int64_t avail = nxt[sl] - beg[sl] + 1;
      bn[sl] = (int)(avail < kBuf ? avail : kBuf);
      nxt[sl] -= bn[sl];
    };
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      if (nxt[sl] >= beg[sl]) refill(sl);
      cur[sl] = bn[sl] > 0 ? buf[sl][0] : INT_MIN;
    }
    int phase = 0;           // 0: tiles, 1: chips, 2: done
    int tile_best = 0, tile_sub = 0, n_sub = (B + kBox - 1) / kBox;
    unsigned long long tile_mask = 0ull;
    bool tile_open = false;
    int cg = 0;              // chips: row block
    int64_t c0 = 0, cend = 0, s0 = 0, chip_end = 0;
    bool chip_open = false, chip_first = false;
    if (G > 0) {
      c0 = p.col_offsets[row0];
      cend = p.col_offsets[row0 + 1];
    }
    auto next_step = [&](StepInfo& st) {
      if (phase == 0) {
        if (!tile_open) {
          const int best = __reduce_max_sync(0xffffffffu, max(cur[0], cur[1]));
          if (best == INT_MIN) {
            phase = 1;
          } else {
            const bool hit0 = cur[0] == best, hit1 = cur[1] == best;
            tile_mask = (unsigned long long)__ballot_sync(0xffffffffu, hit0) |
                        ((unsigned long long)__ballot_sync(0xffffffffu, hit1) << 32);
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              if (sl == 0 ? hit0 : hit1) {
#pragma unroll
                for (int u = 0; u + 1 < kBuf; ++u) buf[sl][u] = buf[sl][u + 1];
                if (--bn[sl] == 0 && nxt[sl] >= beg[sl]) refill(sl);
                cur[sl] = bn[sl] > 0 ? buf[sl][0] : INT_MIN;
              }
            }
            tile_best = best;
            tile_sub = 0;
            tile_open = true;
          }
        }
        if (phase == 0) {
          st.kind = kTile;
          st.box = tile_best + tile_sub * kBox;
          st.width = min(kBox, B - tile_sub * kBox);
          st.mask = tile_mask;
          if (++tile_sub == n_sub) tile_open = false;
          return;
        }
      }
      if (phase == 1) {
        // chips: per row block, chips of B columns, each split in 64-key steps
        while (!chip_open) {
          if (c0 < cend) {
            chip_end = min(c0 + (int64_t)B, cend);
            s0 = c0;
            chip_open = true;
            chip_first = true;
          } else if (++cg < G) {
            c0 = p.col_offsets[row0 + cg];
            cend = p.col_offsets[row0 + cg + 1];
          } else {
            phase = 2;
            break;
          }
        }
        if (phase == 1) {
          st.kind = kChip;
          st.s0 = s0;
          st.n = (int)min((int64_t)kBox, chip_end - s0);
          st.mask = 1ull << cg;
          st.first = chip_first;
          chip_first = false;
          s0 += kBox;
          if (s0 >= chip_end) {
            chip_open = false;
            c0 = chip_end;
          }
          return;
        }
      }
      st.kind = kEnd;
    };

    // gather 64 rows (16-byte chunks) of K or V by column index into a SW128 tile
    // gather 64 rows (16-byte chunks) of K or V by column index into a SW128 tile: every
    // lane's cp.async copies are in flight at once (rows past the chip are zero-filled), one
    // wait, a proxy fence, then lane 0's arrival (benchmarks/bench_columns.py: a chip step
    // cost ~13x a tile step with per-chunk __ldg round trips; completing the copies into the
    // mbarrier asynchronously gained only 3 % more and draws synccheck "missing wait" reports)
    auto gather = [&](uint8_t* dst, const __nv_bfloat16* src, const __nv_bfloat16* src2, const StepInfo& st,
                      uint64_t* bar) {
      constexpr int kChunksPerRow = kD / 8;
      // the chip's column indices: lane l holds keys l and l + 32
      const int key_a = lane < st.n ? p.col_indices[st.s0 + lane] : 0;
      const int key_b = lane + 32 < st.n ? p.col_indices[st.s0 + lane + 32] : 0;
      const uint32_t dbase = smem_u32(dst);
#pragma unroll 8
      for (int idx = lane; idx < kBox * kChunksPerRow; idx += 32) {
        const int j = idx / kChunksPerRow;
        const int c16 = idx % kChunksPerRow;
        const int atom = c16 >> 3, c = c16 & 7;
        const uint32_t off = atom * (kBox * 128) + (j >> 3) * 1024 + (j & 7) * 128 + ((c ^ (j & 7)) << 4);
        const int kj = __shfl_sync(0xffffffffu, j < 32 ? key_a : key_b, j & 31);
        const bool valid = j < st.n;
        const int64_t e = (int64_t)(valid ? kj : 0) * kD + c16 * 8;
        cp_async_16_zfill(dbase + off, src + e, valid);
        if (kSplit) cp_async_16_zfill(dbase + L::kKBytes + off, src2 + e, valid);
      }
      cp_async_wait_all();
      fence_proxy_async_smem();
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };

    int running = INT_MIN;  // chip prefix max, carried across a chip's 64-key steps
    // descriptor of step t (kind, box/width, segment mask, chip prefix max), ring of R::kD
    auto write_desc = [&](int t, const StepInfo& st) {
      const int sd = t % R::kD;
      if (lane == 0) mbar_wait(&ctrl->d_empty[sd], ((t / R::kD) & 1) ^ 1);
      __syncwarp();
      StepDesc& d = ctrl->desc[sd];
      if (st.kind == kChip) {
        if (st.first) running = INT_MIN;
        // prefix max of the keys (two 32-wide warp scans)
        int key_a = lane < st.n ? p.col_indices[st.s0 + lane] : INT_MIN;
        int key_b = lane + 32 < st.n ? p.col_indices[st.s0 + lane + 32] : INT_MIN;
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
      }
      if (lane == 0) {
        d.kind = (short)st.kind;
        d.box = st.kind == kChip ? 0 : st.box;
        d.width = (short)(st.kind == kChip ? st.n : st.width);
        d.segmask = st.mask;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_full[sd]);
    };

    auto issue_k = [&](int t, const StepInfo& st) {
      const int sk = t % R::kK;
      uint8_t* kst = smem + L::kOffK + sk * (L::kCopies * L::kKBytes);
      if (lane == 0) mbar_wait(&ctrl->k_empty[sk], ((t / R::kK) & 1) ^ 1);
      __syncwarp();
      if (st.kind == kTile) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&ctrl->k_full[sk], L::kTxKV);
#pragma unroll
          for (int a = 0; a < L::kAtoms; ++a) {
            tma_load_3d(kst + a * (kBox * 128), &tm_k, &ctrl->k_full[sk], a * 64, st.box, kvh);
            if (kSplit) tma_load_3d(kst + L::kKBytes + a * (kBox * 128), &tm_k2, &ctrl->k_full[sk], a * 64, st.box, kvh);
          }
        }
      } else {
        gather(kst, kb, kb2, st, &ctrl->k_full[sk]);
      }
      __syncwarp();
      write_desc(t, st);
    };

    auto issue_v = [&](int t, const StepInfo& st) {
      const int sv = t % R::kV;
      uint8_t* vst = smem + L::kOffV + sv * (L::kCopies * L::kKBytes);
      if (lane == 0) mbar_wait(&ctrl->v_empty[sv], ((t / R::kV) & 1) ^ 1);
      __syncwarp();
      if (st.kind == kChip) {
        gather(vst, vb, vb2, st, &ctrl->v_full[sv]);
      } else if (lane == 0) {
        mbar_arrive_expect_tx(&ctrl->v_full[sv], L::kTxKV);
#pragma unroll
        for (int a = 0; a < L::kAtoms; ++a) {
          tma_load_3d(vst + a * (kBox * 128), &tm_v, &ctrl->v_full[sv], a * 64, st.box, kvh);
          if (kSplit) tma_load_3d(vst + L::kKBytes + a * (kBox * 128), &tm_v2, &ctrl->v_full[sv], a * 64, st.box, kvh);
        }
      }
      __syncwarp();
    };

    // schedule: K (and the descriptor) of step t+1 is issued before V of step t
    StepInfo pend;
    bool have_pend = false;
    int t = 0;
    while (true) {
      StepInfo st;
      next_step(st);
      if (st.kind != kEnd) issue_k(have_pend ? t + 1 : t, st);
      else write_desc(have_pend ? t + 1 : t, st);  // end marker through the descriptor ring
      if (have_pend) {
        issue_v(t, pend);
        ++t;
      }
      if (st.kind == kEnd) break;
      pend = st;
      have_pend = true;
    }
  } else if (warp == 1) {
    // =============================== MMA issuer ================================
    {  // whole warp, warp-uniform; elected lane issues
      constexpr uint32_t idesc_qk = umma_idesc_bf16(128, kBox, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, kD, 0, 1);
      const uint32_t tO = tmem + 128;
      // Descriptors are formed once; per MMA only a constant (and a per-stage) offset is
      // added to the 14-bit start-address field (smem offsets >> 4, no carry out of it).
      const uint32_t qlo0 = sw128_lo(sbase + L::kOffQ, 0);
      const uint32_t klo0 = sw128_lo(sbase + L::kOffK, 0);
      const uint32_t vlo0 = sw128_lo(sbase + L::kOffV, kBox * 128);
      constexpr uint32_t dhi = sw128_hi(1024);
      constexpr uint32_t kStageKV = (uint32_t)(L::kCopies * L::kKBytes);
      mbar_wait(&ctrl->q_full, 0);
      tc_fence_after();

      auto issue_pv = [&](int u) {
        const int sv = u % R::kV;
        mbar_wait(&ctrl->p_full[u & 1], (u >> 1) & 1);
        mbar_wait(&ctrl->v_full[sv], (u / R::kV) & 1);
        tc_fence_after();
        const uint32_t vd = vlo0 + ((sv * kStageKV) >> 4);
        // P(u): own columns (separate-P) or over S(u) (split: hi in cols 0..31, lo in 32..63)
        const uint32_t tP = kSepP<kSplit> ? tmem + kBox + (u & 1) * (kBox / 2) : tmem + (u & 1) * kBox;
#pragma unroll
        for (int k = 0; k < kBox / 16; ++k) {
          const uint32_t b_hi = vd + ((k * 2048) >> 4);
          mma_bf16_ts_w2(tO, tP + k * 8, b_hi, dhi, idesc_pv, (u > 0 || k > 0) ? 1u : 0u);
          if (kSplit) {
            const uint32_t b_lo = vd + ((L::kKBytes + k * 2048) >> 4);
            mma_bf16_ts_w2(tO, tP + k * 8, b_lo, dhi, idesc_pv, 1u);
            mma_bf16_ts_w2(tO, tP + 32 + k * 8, b_hi, dhi, idesc_pv, 1u);
          }
        }
        mma_commit_w(&ctrl->v_empty[sv]);
        if (!kSepP<kSplit>) mma_commit_w(&ctrl->s_free[u & 1]);
      };

      int t = 0;
      for (;; ++t) {
        const int sd = t % R::kD;
        mbar_wait(&ctrl->d_full[sd], (t / R::kD) & 1);
        const int kind = *reinterpret_cast<volatile short*>(&ctrl->desc[sd].kind);
        if (kind == kEnd) break;
        const int sk = t % R::kK;
        const int sb = kSepP<kSplit> ? 0 : t & 1;
        mbar_wait(&ctrl->k_full[sk], (t / R::kK) & 1);
        if (kSepP<kSplit>) {
          if (t > 0) mbar_wait(&ctrl->s_free[0], (t - 1) & 1);  // softmax(t-1) has read S
        } else {
          mbar_wait(&ctrl->s_free[sb], ((t >> 1) & 1) ^ 1);
        }
        tc_fence_after();
        const uint32_t kd = klo0 + ((sk * kStageKV) >> 4);
        const uint32_t tS = tmem + sb * kBox;
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t aoff = ((k >> 2) * (kRows * 128) + (k & 3) * 32) >> 4;
          const uint32_t boff = ((k >> 2) * (kBox * 128) + (k & 3) * 32) >> 4;
          mma_bf16_ss_w2(tS, qlo0 + aoff, dhi, kd + boff, dhi, idesc_qk, k > 0 ? 1u : 0u);
          if (kSplit) {
            mma_bf16_ss_w2(tS, qlo0 + aoff, dhi, kd + boff + (L::kKBytes >> 4), dhi, idesc_qk, 1u);
            mma_bf16_ss_w2(tS, qlo0 + aoff + (L::kQBytes >> 4), dhi, kd + boff, dhi, idesc_qk, 1u);
          }
        }
        mma_commit_w(&ctrl->s_full[sb]);
        mma_commit_w(&ctrl->k_empty[sk]);
        if (t > 0) issue_pv(t - 1);
      }
      if (t > 0) issue_pv(t - 1);
      mma_commit_w(&ctrl->o_ready);
    }
    __syncwarp();
  } else {
    // =============================== softmax warps =============================
    // kHalves warps per TMEM lane quarter; thread <-> (row, key half).  Every thread
    // reads its row's whole 64-key S slice (the row max needs all of it) but
    // exponentiates and writes P for its own kCols keys only, keeps l for its half
    // (the halves agree on m bit for bit) and rescales / stores its kD / kHalves
    // columns of O.  Two halves = twice the warps to hide the exp/FMA latency chain.
    constexpr int kHalves = kSoftHalves<kSplit>;
    constexpr int kCols = kBox / kHalves;
    constexpr int kOCols = kD / kHalves;
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int c0 = half * kCols;       // first key (S column) of this thread's half
    const int oc0 = half * kOCols;     // first O column of this thread's half
    const int row = quarter * 32 + lane;
    const int q = R0 + row;
    const int seg = (q < S) ? (q / B - r_first) : -1;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    int t = 0;
    for (;; ++t) {
      const int sd = t % R::kD;
      mbar_wait(&ctrl->d_full[sd], (t / R::kD) & 1);
      const StepDesc& d = ctrl->desc[sd];
      const int kind = d.kind;
      if (kind == kEnd) break;
      const int sb = t & 1;  // S buffer (split) / P buffer
      if (kSepP<kSplit>) {
        mbar_wait(&ctrl->s_full[0], t & 1);
      } else {
        mbar_wait(&ctrl->s_full[sb], (t >> 1) & 1);
      }
      tc_fence_after();
      const uint32_t s_col = kSepP<kSplit> ? 0u : (uint32_t)(sb * kBox);
      uint32_t x[kCols];                          // own keys c0 .. c0+kCols-1
      uint32_t y[kHalves > 1 ? kBox - kCols : 1];  // the other half (max only)
      if (kHalves == 1) {
        tmem_ld32x32b_x64(tmem + lane_off + s_col, x);
      } else {
        tmem_ld32x32b_x32(tmem + lane_off + s_col + c0, x);
        tmem_ld32x32b_x32(tmem + lane_off + s_col + (c0 ^ kCols), y);
      }
      // valid key slots for this row, [lo, hi), computed while the TMEM load is in flight
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);  // descriptor consumed (MMA read its kind earlier)
      tmem_wait_ld();
      if (kSepP<kSplit>) {  // S consumed: QK(t+1) may overwrite it while this step computes
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctrl->s_free[0]);
      }
      if (!__any_sync(0xffffffffu, hi > lo)) {
        // none of this warp's rows sees the step (the other row block's tile of a union
        // step, a block-sparse block of the other row): P = 0, softmax state unchanged
        uint32_t z[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = 0u;
        if (kSepP<kSplit>) {
          const uint32_t pcol = kBox + sb * (kBox / 2) + half * (kCols / 2);
          if (kCols == 32) tmem_st32x32b_x16(tmem + lane_off + pcol, z);
          else tmem_st32x32b_x32(tmem + lane_off + pcol, z);
        } else {
          tmem_st32x32b_x32(tmem + lane_off + sb * kBox, z);
          if (kSplit) tmem_st32x32b_x32(tmem + lane_off + sb * kBox + 32, z);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&ctrl->p_full[sb]);
        continue;
      }
      // branch-free masking: invalid slots become -inf (ex2(-inf) = +0)
      if (!(lo == 0 && hi == kBox)) {
        const int xl = lo - c0, xh = hi - c0;
#pragma unroll
        for (int j = 0; j < kCols; ++j) x[j] = (j >= xl && j < xh) ? x[j] : 0xff800000u;
        if (kHalves > 1) {
          const int yl = lo - (c0 ^ kCols), yh = hi - (c0 ^ kCols);
#pragma unroll
          for (int j = 0; j < kBox - kCols; ++j) y[j] = (j >= yl && j < yh) ? y[j] : 0xff800000u;
        }
      }
      // row max over all 64 keys: four independent 3-input max chains (FMNMX3)
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int j = 0; j < kCols; j += 8) {
        mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
        mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
        mx2 = fmax3(mx2, u2f(x[j + 4]), u2f(x[j + 5]));
        mx3 = fmax3(mx3, u2f(x[j + 6]), u2f(x[j + 7]));
      }
      if (kHalves > 1) {
#pragma unroll
        for (int j = 0; j < kBox - kCols; j += 8) {
          mx0 = fmax3(mx0, u2f(y[j]), u2f(y[j + 1]));
          mx1 = fmax3(mx1, u2f(y[j + 2]), u2f(y[j + 3]));
          mx2 = fmax3(mx2, u2f(y[j + 4]), u2f(y[j + 5]));
          mx3 = fmax3(mx3, u2f(y[j + 6]), u2f(y[j + 7]));
        }
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
      uint32_t ph[kCols / 2];
      uint32_t pl[kSplit ? kCols / 2 : 1];
      // p = 2^(x*c - m): packed FFMA2, MUFU ex2, packed FADD2 row sums
      const float neg_m = (m_run == -INFINITY) ? 0.f : -m_run;
      const uint64_t c2 = pack_f32x2(scale_log2, scale_log2);
      const uint64_t m2 = pack_f32x2(neg_m, neg_m);
      uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
      for (int j = 0; j < kCols; j += 2) {
        const uint64_t yv = ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, m2);
        float y0, y1;
        unpack_f32x2(yv, y0, y1);
        const float p0 = ex2_approx(y0);
        const float p1 = ex2_approx(y1);
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

      // O rescale needs PV(t-1) retired: the V slot it read is released by a commit behind
      // it (v_empty, phase (t-1)/kV).  S(t) being ready implies PV(t-2) retired (QK(t) is
      // issued after PV(t-2) and the commit behind s_full tracks every earlier MMA of the
      // issuing thread), so that slot's previous phase (PV(t-1-kV)) is complete and the
      // parity wait cannot alias.  The same fact frees P buffer t&1 (last read by PV(t-2)).
      // tcgen05.ld/st are warp-collective: decide per warp.
      if (t > 0 && __any_sync(0xffffffffu, rescale)) {
        mbar_wait(&ctrl->v_empty[(t - 1) % R::kV], ((t - 1) / R::kV) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kOCols; c += 32) {
          uint32_t o[32];
          tmem_ld32x32b_x32(tmem + lane_off + 128 + oc0 + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(u2f(o[j]) * alpha);
          tmem_st32x32b_x32(tmem + lane_off + 128 + oc0 + c, o);
        }
      }
      // P(t) -> TMEM: bf16 pairs, K-major (PV reads A from TMEM)
      if (kSepP<kSplit>) {
        const uint32_t pcol = kBox + sb * (kBox / 2) + half * (kCols / 2);
        if (kCols == 32) tmem_st32x32b_x16(tmem + lane_off + pcol, ph);
        else tmem_st32x32b_x32(tmem + lane_off + pcol, ph);
      } else {
        tmem_st32x32b_x32(tmem + lane_off + sb * kBox, ph);
        if (kSplit) tmem_st32x32b_x32(tmem + lane_off + sb * kBox + 32, pl);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctrl->p_full[sb]);
    }
    // ---- epilogue: O / l -> global ----
    if (t > 0) {
      mbar_wait(&ctrl->o_ready, 0);
      tc_fence_after();
    }
    float l_tot = l_run;
    if (kHalves > 1) {
      // sum the halves' l through TMEM columns 0..1 (S is dead once every PV retired)
      uint32_t lv = __float_as_uint(l_run);
      tmem_st32x32b_x1(tmem + lane_off + half, &lv);
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1, 32 * 4 * kHalves);
      tc_fence_after();
      uint32_t l2[2];
      tmem_ld32x32b_x2(tmem + lane_off, l2);
      tmem_wait_ld();
      l_tot = u2f(l2[0]) + u2f(l2[1]);
    }
    if (p.lse != nullptr && half == 0 && q < S)
      p.lse[(int64_t)h * S + q] = (t > 0 && l_tot > 0.f) ? (m_run + log2f(l_tot)) * 0.6931471805599453f : -INFINITY;
    if (!kSplit && kHalves == 1 && !p.out_f32 && p.d_out == kD) {
      // O / l as bf16 into the (now idle) K ring in the SW128 layout of a TMA tile -- 16-byte
      // chunk c of row r at c ^ (r & 7) -- then one tensor store per 64-column atom (rows
      // past S clipped by the map): coalesced, where per-row stores touch one sector per lane
      const float inv = (t > 0 && l_tot > 0.f) ? 1.f / l_tot : 0.f;
      uint8_t* ost = smem + L::kOffK;  // every MMA, load and gather into the rings has retired
#pragma unroll
      for (int c = 0; c < kD; c += 32) {
        uint32_t o[32];
        __syncwarp();
        if (t > 0) {
          tmem_ld32x32b_x32(tmem + lane_off + 128 + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0u;
        }
        const uint32_t rbase = smem_u32(ost) + (uint32_t)((c >> 6) * (kRows * 128) + row * 128);
        const int ch0 = (c & 63) >> 3;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int j = 8 * k4;
          st_shared_v4(rbase + ((((ch0 + k4) ^ (row & 7))) << 4), pack_bf16x2(u2f(o[j]) * inv, u2f(o[j + 1]) * inv),
                       pack_bf16x2(u2f(o[j + 2]) * inv, u2f(o[j + 3]) * inv),
                       pack_bf16x2(u2f(o[j + 4]) * inv, u2f(o[j + 5]) * inv),
                       pack_bf16x2(u2f(o[j + 6]) * inv, u2f(o[j + 7]) * inv));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(2, 128);
      if (threadIdx.x == 64) {
#pragma unroll
        for (int a = 0; a < L::kAtoms; ++a) tma_store_3d(&tm_o, ost + a * (kRows * 128), a * 64, R0, h);
        bulk_commit_group();
        bulk_wait_group_read0();
      }
    } else {
      const float inv = (t > 0 && l_tot > 0.f) ? 1.f / l_tot : 0.f;
      const int dout = p.d_out;
      const int64_t obase = ((int64_t)h * S + min(q, S - 1)) * dout + oc0;
      const int dmine = min(kOCols, dout - oc0);  // columns of this half that exist in the output
#pragma unroll
      for (int c = 0; c < kOCols; c += 32) {
        uint32_t o[32];
        __syncwarp();
        if (t > 0) {  // warp-uniform: every lane loads, only rows < S store
          tmem_ld32x32b_x32(tmem + lane_off + 128 + oc0 + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0u;
        }
        if (q >= S || dmine <= 0) {
        } else if (p.out_f32) {
          float* out = reinterpret_cast<float*>(p.out) + obase;
          if (dmine == kOCols) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(out + c + j) =
                  make_float4(u2f(o[j]) * inv, u2f(o[j + 1]) * inv, u2f(o[j + 2]) * inv, u2f(o[j + 3]) * inv);
          } else {
            for (int j = 0; j < 32; ++j)
              if (c + j < dmine) out[c + j] = u2f(o[j]) * inv;
          }
        } else {
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + obase;
          if (dmine == kOCols) {
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
              if (c + j < dmine) out[c + j] = __float2bfloat16_rn(u2f(o[j]) * inv);
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
  CUtensorMap tq, tk, tv, tq2, tk2, tv2, to;
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
  // bf16 output of the padded width: stored by tensor-map tiles (see the epilogue)
  if (!kSplit && !a.out_f32 && a.d_out == kD) {
    if ((rc = make_tmap_bf16_3d(&to, a.out, kD, a.S, a.Hq, kRows))) return rc;
  } else {
    to = tq;
  }
  auto kern = sparse_attn_fwd_kernel<kD, kSplit>;
  constexpr int kLaunchSmem = L::kSmem;
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kLaunchSmem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(attn smem)");
    attr_done = true;
  }
  const int n_ctile = (a.S + kRows - 1) / kRows;
  const long long grid = a.work_order != nullptr ? (long long)a.n_work : (long long)n_ctile * a.Hq;
  if (grid == 0) return 0;
  if (grid > 0x7fffffffLL) return set_error(2, "attention grid too large");
  const float scale_log2 = a.scale * 1.4426950408889634f;
  note_launches(1);
  kern<<<(unsigned)grid, kThreadsT<kSplit>, kLaunchSmem, stream>>>(tq, tk, tv, tq2, tk2, tv2, to, a, n_ctile, scale_log2);
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
