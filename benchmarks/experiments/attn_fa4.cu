// attn_fa4.cu -- sparse FlashAttention forward, bf16 I/O: two 128-row query tiles
// per CTA sharing 128-key K/V steps (the production kernel for bf16 heads;
// attn_fwd.cu keeps the fp32 split path and the LSE-free fallbacks).
//
// Same contract as attn_fwd.cu (the reference kernel _core.pyx:72-192 /
// _core_py.py:17-66: per B-row block, its tiles then its column chips, per-cell
// causal masks, one online-softmax state per row, zero rows without coverage).
//
// B200 structure:
//   * CTA = 256 query rows of one q-head = two 128-row tiles A and B, one CTA per
//     SM with all 512 TMEM columns: S_A, S_B (128 fp32 columns each; P is written
//     back over S as packed bf16) and O_A, O_B (128 columns each);
//   * step = 128 keys = two 64-key boxes of the union of the CTA's row blocks'
//     tiles (descending, the diagonal first) and then their column chips; each
//     box carries its own segment mask, so a row block never sees another
//     block's keys; K / V stages are shared by both tiles (half the loads of two
//     independent 128-row CTAs);
//   * MMA order per step t: PV_A(t), QK_A(t+1), PV_B(t), QK_B(t+1): while one
//     tile's softmax runs, the tensor pipe works on the other tile.  S = QK^T is
//     M128 x N128 x K=d (full rate: no N=64 shared-memory bound), O += PV is
//     M128 x N=d x K128 with A (= P) read from TMEM;
//   * the softmax chain per step is the critical path (QK(t+1) waits for PV(t),
//     which waits for P(t)), so it is kept short: S is loaded in two 64-column
//     halves with the first half's mask / max under the second load, P is stored
//     in 32-key chunks as its exponentials complete (one store wait per step),
//     and the row sum runs in packed f32x2 arithmetic.
#include "spf_internal.h"
#include "spf_ptx.cuh"

#include <math.h>

namespace spf {

namespace {

constexpr int kTRows = 128;    // rows per query tile (UMMA M)
constexpr int kCRows = 256;    // rows per CTA
constexpr int kBox = 64;       // keys per box
constexpr int kSKeys = 128;    // keys per step (two boxes)
constexpr int kKS = 2, kVS = 2, kDS = 3;
constexpr int kThreadsF = 384;  // warps 0-3 tile A, 4-7 tile B (softmax), 8 loader, 9/10 MMA A/B, 11 idle
constexpr int kWarpLoad = 8, kWarpMma = 9;  // kWarpMma issues tile A's MMAs, kWarpMma + 1 tile B's
// registers per thread after setmaxnreg: the two softmax warpgroups grow, the
// producer warpgroup shrinks (8*32*184 + 4*32*120 <= 65536; both spill-free)
constexpr int kRegsSoftmax = 184, kRegsProducer = 120;
// every kEmu-th pair of exponentials is computed by exp2_poly_x2 on the FMA pipe (the two
// softmax warpgroups share each SMSP's MUFU; the FA4 balance); 0 = all on MUFU
constexpr int kEmu = 0;

enum : int { kNone = 0, kTile = 1, kChip = 2, kEnd = 3 };

struct BoxDesc {
  unsigned long long segmask;
  int box;
  short kind;
  short width;
};

struct StepDescF {
  BoxDesc b[2];
  int pmax[2][kBox];
};

struct CtrlF {
  uint64_t q_full;
  uint64_t k_full[kKS], k_empty[kKS];
  uint64_t v_full[kVS], v_empty[kVS];
  uint64_t d_full[kDS], d_empty[kDS];
  uint64_t s_full[2];
  uint64_t p_full[2];
  uint64_t pv_done[2];
  uint64_t o_ready;
  uint32_t tmem_base;
  uint32_t pad;
  StepDescF desc[kDS];
};

template <int kD>
struct LayoutF {
  static constexpr int kAtoms = kD / 64;
  static constexpr int kQTile = kTRows * kD * 2;
  static constexpr int kStage = kSKeys * kD * 2;  // one K or V stage (two boxes)
  static constexpr int kAtomStage = kSKeys * 128;  // one 64-wide d atom of a stage
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = 2 * kQTile;
  static constexpr int kOffV = kOffK + kKS * kStage;
  static constexpr int kOffCtrl = kOffV + kVS * kStage;
  static constexpr int kSmem = kOffCtrl + (int)sizeof(CtrlF);
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

__device__ __forceinline__ void mma_bf16_ts_f(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

struct BoxInfo {
  int kind;
  int box, width;
  unsigned long long mask;
  int64_t s0;  // chip: first column index
  int n;       // chip: keys in this box
  bool first;  // chip: first box of a chip (prefix max restarts)
};

// valid key slots [lo, hi) of box `b` for query row q (segment seg of the CTA)
__device__ __forceinline__ void box_range(const BoxDesc& b, const int* pmax, int seg, int q, int S, int& lo,
                                          int& hi) {
  lo = 0;
  hi = 0;
  if (seg < 0 || !((b.segmask >> seg) & 1ull)) return;
  if (b.kind == kTile) {
    lo = max(0, -b.box);
    hi = min((int)b.width, min(S - b.box, q - b.box + 1));
  } else if (b.kind == kChip) {
    int a = 0, e = b.width;
    while (a < e) {
      const int m = (a + e) >> 1;
      if (pmax[m] <= q) a = m + 1; else e = m;
    }
    hi = a;
  }
}

template <int kD>
__global__ void __launch_bounds__(kThreadsF, 1)
    sparse_attn_fa4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                            const __grid_constant__ CUtensorMap tm_v, const AttnArgs p, int n_ctile,
                            float scale_log2) {
  using L = LayoutF<kD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  CtrlF* ctrl = reinterpret_cast<CtrlF*>(smem + L::kOffCtrl);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  int item = blockIdx.x;
  if (p.work_order != nullptr) item = p.work_order[item];
  const int ct = n_ctile - 1 - item / p.Hq;  // heavy (late) row tiles first, heads fastest
  const int h = item % p.Hq;
  for (int i = 0; i < p.n_pair; ++i)
    if (p.pair_heads[i] == h) {
      if (pair_preferred(p.pair_stats, i)) return;  // run by the paired-box kernel (attn_bs.cu)
      break;
    }
  const int kvh = h / (p.Hq / p.Hkv);
  const int S = p.S, B = p.B;
  const int n_rows = (S + B - 1) / B;
  const int R0 = ct * kCRows;
  const int r_first = R0 / B;
  const int r_last = min((R0 + kCRows - 1) / B, n_rows - 1);
  const int G = r_last - r_first + 1;  // <= 64 (host checks B >= 4)

  if (threadIdx.x == 0) {
    if ((sbase & 1023u) != 0) {
      printf("spf: dynamic smem not 1024-aligned\n");
      __trap();
    }
    mbar_init(&ctrl->q_full, 1);
    for (int s = 0; s < kKS; ++s) {
      mbar_init(&ctrl->k_full[s], 1);
      mbar_init(&ctrl->k_empty[s], 2);  // both tiles' QK
    }
    for (int s = 0; s < kVS; ++s) {
      mbar_init(&ctrl->v_full[s], 1);
      mbar_init(&ctrl->v_empty[s], 2);  // both tiles' PV
    }
    for (int s = 0; s < kDS; ++s) {
      mbar_init(&ctrl->d_full[s], 1);
      mbar_init(&ctrl->d_empty[s], 8);  // one arrival per softmax warp (both tiles)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ctrl->s_full[s], 1);
      mbar_init(&ctrl->p_full[s], 128);
      mbar_init(&ctrl->pv_done[s], 1);
    }
    mbar_init(&ctrl->o_ready, 2);
    fence_mbar_init();
  }
  if (warp == kWarpMma) tmem_alloc(&ctrl->tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ctrl->tmem_base;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegsProducer));
  if (warp == kWarpLoad) {
    // =============================== loader warp ===============================
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(&ctrl->q_full, 2u * L::kQTile);
#pragma unroll
      for (int tt = 0; tt < 2; ++tt)
#pragma unroll
        for (int a = 0; a < L::kAtoms; ++a)
          tma_load_3d(smem + L::kOffQ + tt * L::kQTile + a * (kTRows * 128), &tm_q, &ctrl->q_full, a * 64,
                      R0 + tt * kTRows, h);
    }
    const int64_t row0 = (int64_t)h * n_rows + r_first;
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_hi) + (int64_t)kvh * S * kD;
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_hi) + (int64_t)kvh * S * kD;

    // ---- box generator: union tiles (descending) then chips; warp-uniform ----
    constexpr int kBuf = 8;
    int cur[2], bn[2];
    int64_t nxt[2], beg[2];
    int buf[2][kBuf];
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int g = lane + 32 * sl;
      beg[sl] = g < G ? p.tile_offsets[row0 + g] : 0;
      nxt[sl] = (g < G ? p.tile_offsets[row0 + g + 1] : 0) - 1;
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
    int phase = 0;
    int tile_best = 0, tile_sub = 0;
    const int n_sub = (B + kBox - 1) / kBox;
    unsigned long long tile_mask = 0ull;
    bool tile_open = false;
    int cg = 0;
    int64_t c0 = 0, cend = 0, s0 = 0, chip_end = 0;
    bool chip_open = false, chip_first = false;
    if (G > 0) {
      c0 = p.col_offsets[row0];
      cend = p.col_offsets[row0 + 1];
    }
    auto next_box = [&](BoxInfo& st) {
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

    // gather 64 K or V rows by column index into half `half` of a 128-row SW128 stage
    auto gather = [&](uint8_t* stage, int half, const __nv_bfloat16* src, const BoxInfo& st) {
      constexpr int kChunksPerRow = kD / 8;
      for (int idx = lane; idx < kBox * kChunksPerRow; idx += 32) {
        const int j = idx / kChunksPerRow;
        const int c16 = idx % kChunksPerRow;
        const int atom = c16 >> 3, c = c16 & 7;
        const int jr = half * kBox + j;  // row within the stage
        const uint32_t off = atom * L::kAtomStage + (jr >> 3) * 1024 + (jr & 7) * 128 + ((c ^ (jr & 7)) << 4);
        int4 x = make_int4(0, 0, 0, 0);
        if (j < st.n) {
          const int key = p.col_indices[st.s0 + j];
          x = __ldg(reinterpret_cast<const int4*>(src + (int64_t)key * kD + c16 * 8));
        }
        *reinterpret_cast<int4*>(stage + off) = x;
      }
    };
    // TMA one 64-key box (all d atoms) into half `half` of a stage; an empty box loads
    // rows past the end of the sequence, which TMA fills with zeros
    auto tma_box = [&](uint8_t* stage, int half, const CUtensorMap* map, uint64_t* bar, int key) {
#pragma unroll
      for (int a = 0; a < L::kAtoms; ++a)
        tma_load_3d(stage + a * L::kAtomStage + half * (kBox * 128), map, bar, a * 64, key, kvh);
    };

    int running = INT_MIN;
    // one arrival per stage fill: chips are gathered first, then a single
    // arrive(.expect_tx for the TMA boxes) and the TMA issues
    auto fill_stage = [&](uint8_t* stage, uint64_t* bar, const CUtensorMap* map, const __nv_bfloat16* src,
                          const BoxInfo (&bx)[2]) {
      uint32_t tx = 0;
      bool gathered = false;
      for (int i = 0; i < 2; ++i) {
        if (bx[i].kind == kChip) {
          gather(stage, i, src, bx[i]);
          gathered = true;
        } else {
          tx += kBox * kD * 2;
        }
      }
      if (gathered) {
        fence_proxy_async_smem();
        __threadfence_block();
      }
      __syncwarp();
      if (lane == 0) {
        if (tx) {
          mbar_arrive_expect_tx(bar, tx);
          for (int i = 0; i < 2; ++i)
            if (bx[i].kind != kChip) tma_box(stage, i, map, bar, bx[i].kind == kTile ? bx[i].box : S);
        } else {
          mbar_arrive(bar);
        }
      }
      __syncwarp();
    };
    auto issue_k = [&](int t, const BoxInfo (&bx)[2]) {
      const int sk = t % kKS;
      if (lane == 0) mbar_wait(&ctrl->k_empty[sk], ((t / kKS) & 1) ^ 1);
      __syncwarp();
      fill_stage(smem + L::kOffK + sk * L::kStage, &ctrl->k_full[sk], &tm_k, kb, bx);
    };
    auto write_desc = [&](int t, const BoxInfo (&bx)[2], bool end) {
      const int sd = t % kDS;
      if (lane == 0) mbar_wait(&ctrl->d_empty[sd], ((t / kDS) & 1) ^ 1);
      __syncwarp();
      StepDescF& d = ctrl->desc[sd];
      for (int i = 0; i < 2; ++i) {
        if (!end && bx[i].kind == kChip) {
          if (bx[i].first) running = INT_MIN;
          int pa = lane < bx[i].n ? p.col_indices[bx[i].s0 + lane] : INT_MIN;
          int pb = lane + 32 < bx[i].n ? p.col_indices[bx[i].s0 + lane + 32] : INT_MIN;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int xa = __shfl_up_sync(0xffffffffu, pa, off);
            const int xb = __shfl_up_sync(0xffffffffu, pb, off);
            if (lane >= off) {
              pa = max(pa, xa);
              pb = max(pb, xb);
            }
          }
          pa = max(pa, running);
          pb = max(pb, __shfl_sync(0xffffffffu, pa, 31));
          d.pmax[i][lane] = pa;
          d.pmax[i][lane + 32] = pb;
          running = __shfl_sync(0xffffffffu, pb, 31);
        }
      }
      if (lane == 0) {
        for (int i = 0; i < 2; ++i) {
          const int kind = end ? kEnd : bx[i].kind;
          d.b[i].kind = (short)kind;
          d.b[i].box = (kind == kTile) ? bx[i].box : 0;
          d.b[i].width = (short)(kind == kTile ? bx[i].width : (kind == kChip ? bx[i].n : 0));
          d.b[i].segmask = (kind == kTile || kind == kChip) ? bx[i].mask : 0ull;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_full[sd]);
    };
    auto issue_v = [&](int t, const BoxInfo (&bx)[2]) {
      const int sv = t % kVS;
      if (lane == 0) mbar_wait(&ctrl->v_empty[sv], ((t / kVS) & 1) ^ 1);
      __syncwarp();
      fill_stage(smem + L::kOffV + sv * L::kStage, &ctrl->v_full[sv], &tm_v, vb, bx);
    };

    // schedule: K + descriptor of step t+1 before V of step t
    BoxInfo pend[2];
    bool have_pend = false;
    int t = 0;
    while (true) {
      BoxInfo bx[2];
      next_box(bx[0]);
      bool end = bx[0].kind == kEnd;
      if (!end) {
        next_box(bx[1]);
        if (bx[1].kind == kEnd) bx[1].kind = kNone;
      }
      const int tn = have_pend ? t + 1 : t;
      if (!end) {
        issue_k(tn, bx);
        write_desc(tn, bx, false);
      } else {
        write_desc(tn, bx, true);
      }
      if (have_pend) {
        issue_v(t, pend);
        ++t;
      }
      if (end) break;
      pend[0] = bx[0];
      pend[1] = bx[1];
      have_pend = true;
    }
  } else if (warp == kWarpMma || warp == kWarpMma + 1) {
    // ========================= MMA issuers (one per tile) =========================
    // Separate issuing warps: tcgen05.mma issue blocks at the pipe rate, so one issuer
    // serving both tiles would hold tile B's PV behind tile A's QK issue (and back).
    const int tile = warp - kWarpMma;
    if (lane == 0) {
      constexpr uint32_t idesc_qk = umma_idesc_bf16(128, kSKeys, 0, 0);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(128, kD, 0, 1);
      const uint32_t q_addr = sbase + L::kOffQ + tile * L::kQTile;
      const uint32_t tS = tmem + tile * 128;
      const uint32_t tO = tmem + 256 + tile * 128;
      mbar_wait(&ctrl->q_full, 0);
      tc_fence_after();
      auto qk = [&](int t) {
        const int sk = t % kKS;
        const uint32_t k_addr = sbase + L::kOffK + sk * L::kStage;
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const int atom = k >> 2;
          const uint32_t koff = (k & 3) * 32;
          const uint64_t ad = umma_desc_sw128(q_addr + atom * (kTRows * 128) + koff, 0, 1024);
          const uint64_t bd = umma_desc_sw128(k_addr + atom * L::kAtomStage + koff, 0, 1024);
          mma_bf16_ss(tS, ad, bd, idesc_qk, k > 0 ? 1u : 0u);
        }
        mma_commit(&ctrl->s_full[tile]);
        mma_commit(&ctrl->k_empty[sk]);
      };
      auto pv = [&](int t) {  // P: key k in packed column k / 2 over S
        const int sv = t % kVS;
        const uint32_t v_addr = sbase + L::kOffV + sv * L::kStage;
#pragma unroll
        for (int k = 0; k < kSKeys / 16; ++k) {
          const uint64_t bd = umma_desc_sw128(v_addr + k * 2048, L::kAtomStage, 1024);
          mma_bf16_ts_f(tO, tS + 8 * k, bd, idesc_pv, (t > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&ctrl->pv_done[tile]);
        mma_commit(&ctrl->v_empty[sv]);
      };
      auto step_kind = [&](int t) {
        const int sd = t % kDS;
        mbar_wait(&ctrl->d_full[sd], (t / kDS) & 1);
        return (int)*reinterpret_cast<volatile short*>(&ctrl->desc[sd].b[0].kind);
      };
      if (step_kind(0) != kEnd) {
        mbar_wait(&ctrl->k_full[0], 0);
        tc_fence_after();
        qk(0);
        for (int t = 0;; ++t) {
          const bool next = step_kind(t + 1) != kEnd;
          // PV(t), then QK(t+1) into the S/P columns PV(t) just consumed (in-order pipe)
          mbar_wait(&ctrl->p_full[tile], t & 1);
          mbar_wait(&ctrl->v_full[t % kVS], (t / kVS) & 1);
          tc_fence_after();
          pv(t);
          if (!next) break;
          mbar_wait(&ctrl->k_full[(t + 1) % kKS], ((t + 1) / kKS) & 1);
          tc_fence_after();
          qk(t + 1);
        }
      }
      mma_commit(&ctrl->o_ready);
    }
    __syncwarp();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegsSoftmax));
    // =============================== softmax warpgroups ========================
    const int tile = warp >> 2;  // 0: warps 0-3, 1: warps 4-7
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = R0 + tile * kTRows + row;
    const int seg = (q < S) ? (q / B - r_first) : -1;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + tile * 128;
    const uint32_t tO = tmem + lane_off + 256 + tile * 128;
    float m_run = -INFINITY, l_run = 0.f;
    const uint64_t c2 = pack_f32x2(scale_log2, scale_log2);
    // Exponential ping-pong: the two warps of a lane quarter (tile A warp q, tile B warp
    // q + 4) share one SMSP and its MUFU; a token passed through two named barriers lets
    // them exponentiate in turn (A, B, A, ...) instead of halving each other's rate.
    const uint32_t bar_a = 1 + quarter, bar_b = 5 + quarter;  // A waits on bar_a, B on bar_b
    if (tile == 1) named_bar_arrive(bar_a, 64);                 // A holds the first token
    int t = 0;
    for (;; ++t) {
      const int sd = t % kDS;
      mbar_wait(&ctrl->d_full[sd], (t / kDS) & 1);
      const StepDescF& d = ctrl->desc[sd];
      if (d.b[0].kind == kEnd) break;
      int lo0, hi0, lo1, hi1;  // this row's valid key slots of the two boxes (before S is ready)
      box_range(d.b[0], d.pmax[0], seg, q, S, lo0, hi0);
      box_range(d.b[1], d.pmax[1], seg, q, S, lo1, hi1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctrl->d_empty[sd]);
      const bool any0 = __any_sync(0xffffffffu, hi0 > lo0), any1 = __any_sync(0xffffffffu, hi1 > lo1);
      mbar_wait(&ctrl->s_full[tile], t & 1);
      tc_fence_after();
      float alpha = 1.f;
      bool rescale = false;
      if (!any0 && !any1) {
        // no row of this warp sees the step (the other tile's boxes): P = 0
        uint32_t z[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = 0u;
        tmem_st32x32b_x32(tS, z);
        tmem_st32x32b_x32(tS + 32, z);
        named_bar_sync(tile == 0 ? bar_a : bar_b, 64);
        named_bar_arrive(tile == 0 ? bar_b : bar_a, 64);
      } else {
        uint32_t x0[kBox], x1[kBox];
        tmem_ld32x32b_x64(tS, x0);
        tmem_ld32x32b_x64(tS + 64, x1);
        tmem_wait_ld();
        if (!(lo0 == 0 && hi0 == kBox)) {
#pragma unroll
          for (int j = 0; j < kBox; ++j) x0[j] = (j >= lo0 && j < hi0) ? x0[j] : 0xff800000u;
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int j = 0; j < kBox; j += 4) {
          mx0 = fmax3(mx0, u2f(x0[j]), u2f(x0[j + 1]));
          mx1 = fmax3(mx1, u2f(x0[j + 2]), u2f(x0[j + 3]));
        }
        if (!(lo1 == 0 && hi1 == kBox)) {
#pragma unroll
          for (int j = 0; j < kBox; ++j) x1[j] = (j >= lo1 && j < hi1) ? x1[j] : 0xff800000u;
        }
#pragma unroll
        for (int j = 0; j < kBox; j += 4) {
          mx2 = fmax3(mx2, u2f(x1[j]), u2f(x1[j + 1]));
          mx3 = fmax3(mx3, u2f(x1[j + 2]), u2f(x1[j + 3]));
        }
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        if (hi0 > lo0 || hi1 > lo1) {
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
        const uint64_t m2 = pack_f32x2(neg_m, neg_m);
        uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        named_bar_sync(tile == 0 ? bar_a : bar_b, 64);  // this warp's turn on the MUFU
        // P in 32-key chunks, each stored as soon as its exponentials are done: keys
        // 32c..32c+31 -> packed bf16 columns [16c, 16c+16) over S (already in registers)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t* xs = c < 2 ? x0 + 32 * c : x1 + 32 * (c - 2);
          uint32_t ph[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const uint64_t y = ffma2(pack_f32x2(u2f(xs[j]), u2f(xs[j + 1])), c2, m2);
            float p0, p1;
            if (kEmu > 0 && ((j >> 1) % (kEmu > 0 ? kEmu : 1)) == kEmu - 1) {
              unpack_f32x2(exp2_poly_x2(y), p0, p1);
            } else {
              float y0, y1;
              unpack_f32x2(y, y0, y1);
              p0 = ex2_approx(y0);
              p1 = ex2_approx(y1);
            }
            const uint64_t pp = pack_f32x2(p0, p1);
            switch ((j >> 1) & 3) {
              case 0: s0 = fadd2(s0, pp); break;
              case 1: s1 = fadd2(s1, pp); break;
              case 2: s2 = fadd2(s2, pp); break;
              default: s3 = fadd2(s3, pp); break;
            }
            ph[j >> 1] = pack_bf16x2(p0, p1);
          }
          tmem_st32x32b_x16(tS + 16 * c, ph);
        }
        named_bar_arrive(tile == 0 ? bar_b : bar_a, 64);  // pass the token
        float sa, sb;
        unpack_f32x2(fadd2(fadd2(s0, s1), fadd2(s2, s3)), sa, sb);
        l_run = l_run * alpha + (sa + sb);
      }
      // O rescale: S(t) ready implies PV(t-1) retired (QK(t) is issued after PV(t-1) in the
      // in-order pipe and s_full tracks all earlier MMAs).  Warp-collective: decide per warp.
      if (t > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
        for (int c = 0; c < kD; c += 32) {
          uint32_t o[32];
          tmem_ld32x32b_x32(tO + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(u2f(o[j]) * alpha);
          tmem_st32x32b_x32(tO + c, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&ctrl->p_full[tile]);
    }
    if (tile == 0) named_bar_sync(bar_a, 64);  // B's last token: every arrive is matched
    // ---- epilogue: O / l -> global ----
    if (t > 0) {
      mbar_wait(&ctrl->o_ready, 0);
      tc_fence_after();
    }
    if (p.lse != nullptr && q < S)
      p.lse[(int64_t)h * S + q] = (t > 0 && l_run > 0.f) ? (m_run + log2f(l_run)) * 0.6931471805599453f : -INFINITY;
    const float inv = (t > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
    const int dout = p.d_out;
    const int64_t obase = ((int64_t)h * S + min(q, S - 1)) * dout;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + obase;
#pragma unroll
    for (int c = 0; c < kD; c += 32) {
      uint32_t o[32];
      __syncwarp();
      if (t > 0) {
        tmem_ld32x32b_x32(tO + c, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = 0u;
      }
      if (q < S) {
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

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int kD>
int launch_fa4_impl(const AttnArgs& a, cudaStream_t stream) {
  using L = LayoutF<kD>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_tmap_bf16_3d(&tq, a.q_hi, kD, a.S, a.Hq, kTRows))) return rc;
  if ((rc = make_tmap_bf16_3d(&tk, a.k_hi, kD, a.S, a.Hkv, kBox))) return rc;
  if ((rc = make_tmap_bf16_3d(&tv, a.v_hi, kD, a.S, a.Hkv, kBox))) return rc;
  auto kern = sparse_attn_fa4_kernel<kD>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmem);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute(attn fa4 smem)");
    attr_done = true;
  }
  const int n_ctile = (a.S + kCRows - 1) / kCRows;
  const long long grid = a.work_order != nullptr ? (long long)a.n_work : (long long)n_ctile * a.Hq;
  if (grid == 0) return 0;
  if (grid > 0x7fffffffLL) return set_error(2, "attention grid too large");
  note_launches(1);
  kern<<<(unsigned)grid, kThreadsF, L::kSmem, stream>>>(tq, tk, tv, a, n_ctile, a.scale * 1.4426950408889634f);
  return check_cuda(cudaGetLastError(), "sparse_attn_fwd2 launch");
}

}  // namespace

bool attn_fa4_supported(const AttnArgs& a) {
  return !a.split && !a.out_f32 && a.B >= 4 && (a.kD == 128 || a.kD == 64) && a.work_order == nullptr;
}

int launch_sparse_attn_fa4(const AttnArgs& a, cudaStream_t stream) {
  if (a.kD == 128) return launch_fa4_impl<128>(a, stream);
  return launch_fa4_impl<64>(a, stream);
}

}  // namespace spf
