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
// 11-bit digits finds the exact k-th largest key T and how many T-valued
// elements are taken (the lowest-index ones); one ordered pass then compacts
// the selection in index order with block scans.
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
  static constexpr int kBits = 11;
  static constexpr int kBins = 1 << kBits;
  static constexpr int kKeyBits = sizeof(Key) * 8;
  using Scan = cub::BlockScan<int, kThreads>;

  struct Storage {
    int hist[kBins];
    typename Scan::TempStorage scan;
    Key prefix;
    int krem;
    int force_pos;
    int force_sel;
  };

  // vals: n candidates (global or shared).  Writes k_eff = min(k, n) indices to out.
  static __device__ void run(Storage& sm, const T* vals, int n, int k, int force_idx, bool descending,
                             int32_t* out, int32_t out_scale) {
    const int tid = threadIdx.x;
    if (k > n) k = n;
    if (k <= 0) return;
    Key prefix = 0, pmask = 0;
    int krem = k;
    for (int shift = kKeyBits - kBits; shift > -kBits; shift -= kBits) {
      const int sh = shift < 0 ? 0 : shift;
      const int width = shift < 0 ? kBits + shift : kBits;
      const Key dmask = (Key)((1u << width) - 1);
      for (int i = tid; i < kBins; i += kThreads) sm.hist[i] = 0;
      __syncthreads();
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
        const unsigned act = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const unsigned peers = __match_any_sync(act, dig);
          if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sm.hist[dig], __popc(peers));
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
        }
      }
      __syncthreads();
      prefix = sm.prefix;
      krem = sm.krem;
      pmask |= dmask << sh;
      __syncthreads();
    }
    const Key thr = prefix;  // exact k-th largest key; krem T-valued elements are taken
    // force-include bookkeeping: is force_idx selected?  (its equal-rank is
    // irrelevant unless key == thr; we compute it in the ordered pass.)
    const int chunk = (n + kThreads - 1) / kThreads;
    const int b0 = min(n, tid * chunk), b1 = min(n, b0 + chunk);
    int eq = 0;
    for (int i = b0; i < b1; ++i) eq += (mono_key(vals[i]) == thr);
    int eq_base;
    Scan(sm.scan).ExclusiveSum(eq, eq_base);
    __syncthreads();
    // pass 1: is force_idx selected?
    if (force_idx >= b0 && force_idx < b1) {
      const Key kf = mono_key(vals[force_idx]);
      int r = eq_base;
      for (int i = b0; i < force_idx; ++i) r += (mono_key(vals[i]) == thr);
      sm.force_sel = (kf > thr) || (kf == thr && r < krem);
    }
    if (force_idx < 0 || force_idx >= n) {
      if (tid == 0) sm.force_sel = 1;
    }
    __syncthreads();
    const bool need_force = !sm.force_sel;
    const int quota = need_force ? krem - 1 : krem;  // the weakest (rank krem-1) makes room
    // pass 2: count selected per chunk, excluding force_idx (placed separately)
    int sel = 0;
    {
      int r = eq_base;
      for (int i = b0; i < b1; ++i) {
        const Key key = mono_key(vals[i]);
        const bool is_eq = key == thr;
        const bool s = (key > thr) || (is_eq && r < quota);
        r += is_eq;
        sel += (s && !(need_force && i == force_idx)) ? 1 : 0;
      }
    }
    int sel_base;
    Scan(sm.scan).ExclusiveSum(sel, sel_base);
    __syncthreads();
    if (need_force && force_idx >= b0 && force_idx < b1) {
      int before = sel_base;
      int r = eq_base;
      for (int i = b0; i < force_idx; ++i) {
        const Key key = mono_key(vals[i]);
        const bool is_eq = key == thr;
        before += ((key > thr) || (is_eq && r < quota)) ? 1 : 0;
        r += is_eq;
      }
      sm.force_pos = before;
    }
    __syncthreads();
    const int fpos = need_force ? sm.force_pos : -1;
    // pass 3: write in index order
    {
      int r = eq_base;
      int pos = sel_base;
      for (int i = b0; i < b1; ++i) {
        const Key key = mono_key(vals[i]);
        const bool is_eq = key == thr;
        const bool s = ((key > thr) || (is_eq && r < quota)) && !(need_force && i == force_idx);
        r += is_eq;
        if (s) {
          const int slot = pos + ((need_force && pos >= fpos) ? 1 : 0);
          out[descending ? (k - 1 - slot) : slot] = i * out_scale;
          ++pos;
        }
      }
    }
    if (need_force && tid == 0) out[descending ? (k - 1 - fpos) : fpos] = force_idx * out_scale;
    __syncthreads();
  }
};

}  // namespace spf
