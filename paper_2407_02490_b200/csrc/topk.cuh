// topk.cuh -- deterministic block-wide top-k (radix select) with the reference's
// tie rule and force-include, estimator.py:59-79:
//   * order = descending value, ties broken toward the LOWER index
//     (np.argsort(-x, kind="stable"));
//   * if `force_idx` is not selected it replaces the weakest pick, i.e. the
//     smallest selected value, and among equal values the highest index;
//   * the result is written sorted by index (ascending, or descending when
//     `descending` is set, as estimator.py:114 does for slashes).
//
// Keys: monotone unsigned images of the float/double values.  Radix select in
// 8-bit digits finds the exact k-th largest key T and how many T-valued
// elements are taken (the lowest-index ones); once the boundary bucket fits in
// shared memory its keys are gathered and the remaining rounds count only them.
// When every T-valued element is taken (no tie straddles the boundary) one
// ordered pass writes the selection; otherwise warp-cooperative ordered passes
// rank the T-valued elements by index.
#pragma once
#include <cub/block/block_scan.cuh>
#include <stdint.h>

namespace spf {

__device__ __forceinline__ uint64_t mono_key(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__device__ __forceinline__ uint32_t mono_key(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b >> 31) ? ~b : (b | (1u << 31));
}

template <int kThreads, typename T>
struct BlockTopK {
  using Key = typename std::conditional<sizeof(T) == 8, uint64_t, uint32_t>::type;
  // 8-bit digits: a 256-bin histogram is zeroed and scanned with one bin per thread (rows
  // of a few thousand candidates pay more for 2048-bin rounds than for one extra round)
  static constexpr int kBits = 8;  // 11-bit digits for fp32 keys (3 rounds) measured 1 % slower on C4
  static constexpr int kBins = 1 << kBits;
  static constexpr int kKeyBits = sizeof(Key) * 8;
  using Scan = cub::BlockScan<int, kThreads>;

  static constexpr int kWarps = kThreads / 32;
  static constexpr int kCap = 2048;
  struct Storage {
    int hist[kBins];
    typename Scan::TempStorage scan;
    Key prefix;
    int krem;
    int bcount;  // elements in the bucket chosen by the last radix round
    int ncand;
    int force_pos;
    int force_sel;
    int wcnt[2][kWarps];  // per-warp T-valued / selected counts (index-ordered passes)
    int wdrop[kWarps];
    Key cand[kCap];  // keys of the boundary bucket once it fits (later rounds only count)
  };

  // vals: n candidates (global or shared).  Writes k_eff = min(k, n) indices to out.
  static __device__ void run(Storage& sm, const T* vals, int n, int k, int force_idx, bool descending,
                             int32_t* out, int32_t out_scale) {
    const int tid = threadIdx.x;
    if (k > n) k = n;
    if (k <= 0) return;
    Key prefix = 0, pmask = 0;
    int krem = k, bcount = 0;
    bool listed = false;
    for (int shift = kKeyBits - kBits; shift > -kBits; shift -= kBits) {
      const int sh = shift < 0 ? 0 : shift;
      const int width = shift < 0 ? kBits + shift : kBits;
      const Key dmask = (Key)((1u << width) - 1);
      for (int i = tid; i < kBins; i += kThreads) sm.hist[i] = 0;
      __syncthreads();
      if (listed) {  // the boundary bucket's keys are in sm.cand
        const int nc = sm.ncand;
        for (int j = tid; j < nc; j += kThreads) {
          const Key key = sm.cand[j];
          if ((key & pmask) == prefix) atomicAdd(&sm.hist[(int)((key >> sh) & dmask)], 1);
        }
      } else
      // warp-aggregated histogram: the leading digits are highly concentrated (values of one
      // exponent), so lanes with equal digits are merged before the shared-memory atomic
      for (int base = 0; base < n; base += kThreads) {
        const int i = base + tid;
        bool hit = false;
        int dig = 0;
        if (i < n) {
          const Key key = mono_key(vals[i]);
          hit = (key & pmask) == prefix;
          dig = (int)((key >> sh) & dmask);
        }
        // lanes sharing the first active lane's digit add once; the rest add singly
        const unsigned act = __ballot_sync(0xffffffffu, hit);
        if (act) {
          const int lead = __ffs(act) - 1;
          const int ldig = __shfl_sync(0xffffffffu, dig, lead);
          const unsigned same = __ballot_sync(0xffffffffu, hit && dig == ldig);
          if ((threadIdx.x & 31) == lead) atomicAdd(&sm.hist[ldig], __popc(same));
          else if (hit && dig != ldig) atomicAdd(&sm.hist[dig], 1);
        }
      }
      __syncthreads();
      // suffix counts: reverse-order inclusive scan over bins (each thread owns kBins/kThreads bins)
      constexpr int kPer = kBins / kThreads;
      int local[kPer];
      int tot = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        local[j] = sm.hist[kBins - 1 - (tid * kPer + j)];  // descending digit order
        tot += local[j];
      }
      int excl;
      Scan(sm.scan).ExclusiveSum(tot, excl);
      // the digit where the running (descending) count first reaches krem
      int run = excl;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int before = run;
        run += local[j];
        if (before < krem && run >= krem) {
          const int digit = kBins - 1 - (tid * kPer + j);
          sm.prefix = prefix | ((Key)digit << sh);
          sm.krem = krem - before;
          sm.bcount = local[j];
        }
      }
      __syncthreads();
      prefix = sm.prefix;
      krem = sm.krem;
      bcount = sm.bcount;
      pmask |= dmask << sh;
      __syncthreads();
      if (!listed && shift - kBits > -kBits && bcount <= kCap) {
        // one pass gathers the bucket's keys; the remaining rounds scan only them
        if (tid == 0) sm.ncand = 0;
        __syncthreads();
        const int lane = tid & 31;
        for (int base = 0; base < n; base += kThreads) {
          const int i = base + tid;
          Key key = 0;
          bool hit = false;
          if (i < n) {
            key = mono_key(vals[i]);
            hit = (key & pmask) == prefix;
          }
          const unsigned hm = __ballot_sync(0xffffffffu, hit);
          if (hm) {
            const int lead = __ffs(hm) - 1;
            int wb = 0;
            if (lane == lead) wb = atomicAdd(&sm.ncand, __popc(hm));
            wb = __shfl_sync(0xffffffffu, wb, lead);
            if (hit) sm.cand[wb + __popc(hm & ((1u << lane) - 1u))] = key;
          }
        }
        __syncthreads();
        listed = true;
      }
    }
    const Key thr = prefix;  // exact k-th largest key; krem T-valued elements are taken
    // Index-ordered passes, warp-cooperative: warp w owns a contiguous range of 32-element
    // groups, lanes read consecutive elements (coalesced, no bank conflicts) and the
    // in-order ranks come from ballots; per-warp totals are prefixed over the warps.
    const int lane = tid & 31, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int wchunk = (((n + kWarps - 1) / kWarps) + 31) & ~31;
    const int w0 = min(n, w * wchunk), w1 = min(n, w0 + wchunk);
    if (bcount == krem) {
      // Every T-valued element is taken (no tie straddles the boundary): selected = key >= T.
      // If force_idx is not among them it replaces the weakest pick, the T-valued element of
      // highest index; the selection is then written in index order in one pass.
      const bool need_force = force_idx >= 0 && force_idx < n && mono_key(vals[force_idx]) < thr;
      int selc = 0, drop = -1;
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const Key key = i < w1 ? mono_key(vals[i]) : (Key)0;
        selc += __popc(__ballot_sync(0xffffffffu, i < w1 && key >= thr));
        if (need_force) {
          const unsigned em = __ballot_sync(0xffffffffu, i < w1 && key == thr);
          if (em) drop = base + 31 - __clz(em);
        }
      }
      if (lane == 0) {
        sm.wcnt[1][w] = selc;
        sm.wdrop[w] = drop;
      }
      __syncthreads();
      int pos = 0;
      for (int x = 0; x < w; ++x) pos += sm.wcnt[1][x];
      int idx_drop = -1;
      if (need_force) {
        for (int x = 0; x < kWarps; ++x) idx_drop = max(idx_drop, sm.wdrop[x]);
        pos += (force_idx < w0 ? 1 : 0) - (idx_drop < w0 ? 1 : 0);
      }
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const Key key = i < w1 ? mono_key(vals[i]) : (Key)0;
        bool s = i < w1 && key >= thr;
        if (need_force) s = (s && i != idx_drop) || (i < w1 && i == force_idx);
        const unsigned smask = __ballot_sync(0xffffffffu, s);
        if (s) {
          const int slot = pos + __popc(smask & lt);
          out[descending ? (k - 1 - slot) : slot] = i * out_scale;
        }
        pos += __popc(smask);
      }
      __syncthreads();
      return;
    }
    // pass A: T-valued count per warp
    int eqc = 0;
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      eqc += __popc(__ballot_sync(0xffffffffu, i < w1 && mono_key(vals[i]) == thr));
    }
    if (lane == 0) sm.wcnt[0][w] = eqc;
    if (tid == 0) sm.force_sel = (force_idx < 0 || force_idx >= n) ? 1 : 0;
    __syncthreads();
    int eq_base = 0;
    for (int x = 0; x < w; ++x) eq_base += sm.wcnt[0][x];
    // is force_idx selected?  (the warp owning it ranks it among the T-valued keys)
    if (force_idx >= w0 && force_idx < w1) {
      int r = eq_base;
      for (int base = w0; base <= force_idx; base += 32) {
        const int i = base + lane;
        const unsigned em = __ballot_sync(0xffffffffu, i < w1 && mono_key(vals[i]) == thr);
        if (force_idx < base + 32) {
          const Key kf = mono_key(vals[force_idx]);
          const int rf = r + __popc(em & ((1u << (force_idx - base)) - 1u));
          if (lane == 0) sm.force_sel = (kf > thr) || (kf == thr && rf < krem);
        }
        r += __popc(em);
      }
    }
    __syncthreads();
    const bool need_force = !sm.force_sel;
    const int quota = need_force ? krem - 1 : krem;  // the weakest (rank krem-1) makes room
    auto selected = [&](int i, int base, int r, unsigned em, Key key) {
      const bool is_eq = i < w1 && key == thr;
      const bool s = i < w1 && ((key > thr) || (is_eq && r + __popc(em & lt) < quota));
      return s && !(need_force && i == force_idx);
    };
    // pass B: selected count per warp (force_idx, when forced, is placed separately)
    int selc = 0;
    {
      int r = eq_base;
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const Key key = i < w1 ? mono_key(vals[i]) : (Key)0;
        const unsigned em = __ballot_sync(0xffffffffu, i < w1 && key == thr);
        selc += __popc(__ballot_sync(0xffffffffu, selected(i, base, r, em, key)));
        r += __popc(em);
      }
    }
    if (lane == 0) sm.wcnt[1][w] = selc;
    __syncthreads();
    int sel_base = 0;
    for (int x = 0; x < w; ++x) sel_base += sm.wcnt[1][x];
    // forced index: its slot = selected elements before it in index order
    if (need_force && force_idx >= w0 && force_idx < w1) {
      int r = eq_base, before = sel_base;
      for (int base = w0; base <= force_idx; base += 32) {
        const int i = base + lane;
        const Key key = i < w1 ? mono_key(vals[i]) : (Key)0;
        const unsigned em = __ballot_sync(0xffffffffu, i < w1 && key == thr);
        const unsigned sm_ = __ballot_sync(0xffffffffu, selected(i, base, r, em, key));
        before += __popc(force_idx < base + 32 ? (sm_ & ((1u << (force_idx - base)) - 1u)) : sm_);
        r += __popc(em);
      }
      if (lane == 0) sm.force_pos = before;
    }
    __syncthreads();
    const int fpos = need_force ? sm.force_pos : -1;
    // pass C: write in index order
    {
      int r = eq_base, pos = sel_base;
      for (int base = w0; base < w1; base += 32) {
        const int i = base + lane;
        const Key key = i < w1 ? mono_key(vals[i]) : (Key)0;
        const unsigned em = __ballot_sync(0xffffffffu, i < w1 && key == thr);
        const bool s = selected(i, base, r, em, key);
        const unsigned smask = __ballot_sync(0xffffffffu, s);
        if (s) {
          const int p0 = pos + __popc(smask & lt);
          const int slot = p0 + ((need_force && p0 >= fpos) ? 1 : 0);
          out[descending ? (k - 1 - slot) : slot] = i * out_scale;
        }
        pos += __popc(smask);
        r += __popc(em);
      }
    }
    if (need_force && tid == 0) out[descending ? (k - 1 - fpos) : fpos] = force_idx * out_scale;
    __syncthreads();
  }
};

}  // namespace spf
