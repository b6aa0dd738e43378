// cluster_topk.cuh -- deterministic top-k of one fp64 vector by a cluster of
// kCl CTAs (distributed shared memory), with the reference's tie rule and
// index-0 force-include (estimator.py:59-79):
//   * order = descending value, ties to the LOWER index;
//   * if index 0 is not selected it replaces the weakest pick (the k-th: the
//     smallest value, highest index among equal values);
//   * output sorted by index, ascending or descending (estimator.py:114).
// Each CTA owns a contiguous slice of the vector.  Radix select in 11-bit
// digits of the monotone 64-bit key: per round every CTA histograms its slice
// (warp-aggregated shared atomics), pushes the non-zero bins into CTA 0 over
// DSMEM, CTA 0 picks the digit and broadcasts (prefix, remaining k).  The
// ordered output pass exchanges per-CTA counts so every CTA writes its picks
// at their global, index-ordered positions.  Optionally certifies the
// boundary against a relative error threshold (see estimate_vs_tc.cu).
#pragma once
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <stdint.h>

#include "topk.cuh"

namespace spf {

// certification: absolute uncertainty of a vector entry from flushed exponentials
// (<= 64 probabilities below 2^-126 each, set to 0 by ex2.approx.ftz)
constexpr double kFlushAbs = 64.0 * 0x1p-126;

template <int kThreads, int kCl>
struct ClusterTopK {
  static constexpr int kBits = 11;
  static constexpr int kBins = 1 << kBits;
  static constexpr int kPer = kBins / kThreads;
  static constexpr int kU = 8;  // loads in flight per thread
  // Once a CTA's share of the boundary bucket fits here, its remaining radix rounds
  // histogram this list instead of re-reading the whole slice.
  static constexpr int kCap = 2048;
  using Scan = cub::BlockScan<int, kThreads>;

  struct Storage {
    int hist[kBins];
    int tot[2][kBins];  // CTA 0: cluster totals, double-buffered by round parity
    typename Scan::TempStorage scan;
    unsigned long long prefix;
    int krem;
    int cnt[2][kCl];    // exchanged per-CTA counts (T-valued, selected)
    double lo[kCl], hi[kCl];
    int eq[kCl];
    int ncand;
    uint64_t cand[kCap];  // keys of this CTA's slice inside the current boundary bucket
  };

  // Aggregated increment: lanes whose digit equals lane-leader's digit add once.
  static __device__ __forceinline__ void hist_add(int* hist, bool hit, int dig) {
    const unsigned act = __ballot_sync(0xffffffffu, hit);
    if (act == 0u) return;
    const int lead = __ffs(act) - 1;
    const int ldig = __shfl_sync(0xffffffffu, dig, lead);
    const unsigned same = __ballot_sync(0xffffffffu, hit && dig == ldig);
    const int lane = threadIdx.x & 31;
    if (lane == lead) atomicAdd(&hist[ldig], __popc(same));
    else if (hit && dig != ldig) atomicAdd(&hist[dig], 1);
  }

  // vals: n values in global memory (the whole vector); writes min(k, n) indices.
  // tau != nullptr: certification; sets *flag |= 1 when the selection is too close to call.
  // [lo, hi) (optional, hi > lo): every value outside is known to be +0 (the fp64 fallback's
  // support); the selection then scans only [lo, hi) when at least k values there are
  // positive -- the k-th largest is then positive, so nothing outside is selected -- and the
  // whole vector otherwise (zeros are then taken by lowest index over all of it).
  static __device__ void run(Storage& sm, const double* __restrict__ vals, int n, int k, bool descending,
                             int32_t* out, const float* tau, int32_t* flag, int lo = 0, int hi = -1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x;
    if (k > n) k = n;
    int dlo = 0, dhi = n;
    if (hi > lo && (lo > 0 || hi < n) && hi - lo >= k) {
      const int c = (hi - lo + kCl - 1) / kCl;
      const int a0 = min(hi, lo + rank * c), a1 = min(hi, a0 + c);
      int pos = 0;
      for (int i = a0 + tid; i < a1; i += kThreads) pos += vals[i] > 0.0 ? 1 : 0;
      int excl, pos_cta;
      Scan(sm.scan).ExclusiveSum(pos, excl, pos_cta);
      if (tid == 0) *cl.map_shared_rank(&sm.cnt[0][rank], 0) = pos_cta;
      cl.sync();
      if (rank == 0 && tid == 0) {
        int total = 0;
        for (int r = 0; r < kCl; ++r) total += sm.cnt[0][r];
        for (int r = 0; r < kCl; ++r) *cl.map_shared_rank(&sm.ncand, r) = total >= k ? 1 : 0;
      }
      cl.sync();
      if (sm.ncand) {  // cluster-uniform
        dlo = lo;
        dhi = hi;
      }
      __syncthreads();
    }
    const int chunk = (dhi - dlo + kCl - 1) / kCl;
    const int s0 = min(dhi, dlo + rank * chunk), s1 = min(dhi, s0 + chunk);
    if (rank == 0)
      for (int b = tid; b < 2 * kBins; b += kThreads) (&sm.tot[0][0])[b] = 0;
    cl.sync();
    uint64_t prefix = 0, pmask = 0;
    int krem = k;
    int round = 0;
    int ncand = -1;  // >= 0: the slice's boundary-bucket keys are in sm.cand[0, ncand)
    for (int shift = 64 - kBits; shift > -kBits; shift -= kBits, ++round) {
      const int sh = shift < 0 ? 0 : shift;
      const int width = shift < 0 ? kBits + shift : kBits;
      const uint64_t dmask = (uint64_t)((1u << width) - 1);
      for (int b = tid; b < kBins; b += kThreads) sm.hist[b] = 0;
      __syncthreads();
      if (ncand >= 0) {
        for (int i0 = 0; i0 < ncand; i0 += kThreads) {  // warp-uniform trip count
          const int i = i0 + tid;
          const uint64_t key = i < ncand ? sm.cand[i] : 0ull;
          hist_add(sm.hist, i < ncand && (key & pmask) == prefix, (int)((key >> sh) & dmask));
        }
      }
      for (int base = ncand >= 0 ? s1 : s0; base < s1; base += kThreads * kU) {
        double v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {  // kU independent loads in flight per thread
          const int i = base + u * kThreads + tid;
          v[u] = i < s1 ? vals[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = base + u * kThreads + tid;
          const uint64_t key = mono_key(v[u]);
          const bool hit = i < s1 && (key & pmask) == prefix;
          hist_add(sm.hist, hit, (int)((key >> sh) & dmask));
        }
      }
      __syncthreads();
      int* tot0 = cl.map_shared_rank(&sm.tot[round & 1][0], 0);
      for (int b = tid; b < kBins; b += kThreads)
        if (sm.hist[b]) atomicAdd(tot0 + b, sm.hist[b]);
      cl.sync();
      if (rank == 0) {
        const int* tot = sm.tot[round & 1];
        int local[kPer];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          local[j] = tot[kBins - 1 - (tid * kPer + j)];  // descending digits
          cnt += local[j];
        }
        int excl;
        Scan(sm.scan).ExclusiveSum(cnt, excl);
        int run = excl;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int before = run;
          run += local[j];
          if (before < krem && run >= krem) {
            const int digit = kBins - 1 - (tid * kPer + j);
            sm.prefix = prefix | ((uint64_t)digit << sh);
            sm.krem = krem - before;
          }
        }
        for (int b = tid; b < kBins; b += kThreads) sm.tot[(round + 1) & 1][b] = 0;
        __syncthreads();
        if (tid < kCl && tid > 0) {
          *cl.map_shared_rank(&sm.prefix, tid) = sm.prefix;
          *cl.map_shared_rank(&sm.krem, tid) = sm.krem;
        }
      }
      cl.sync();
      prefix = sm.prefix;
      krem = sm.krem;
      pmask |= dmask << sh;
      if (ncand < 0 && shift > 0) {
        const int mine = sm.hist[(int)((prefix >> sh) & dmask)];  // this CTA's keys in the new bucket
        __syncthreads();
        if (mine <= kCap) {  // one more pass over the slice, then lists only
          if (tid == 0) sm.ncand = 0;
          __syncthreads();
          for (int base = s0; base < s1; base += kThreads * kU) {
            double v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int i = base + u * kThreads + tid;
              v[u] = i < s1 ? vals[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int i = base + u * kThreads + tid;
              const uint64_t key = mono_key(v[u]);
              const bool hit = i < s1 && (key & pmask) == prefix;
              const unsigned m = __ballot_sync(0xffffffffu, hit);
              if (m) {
                const int lane = tid & 31;
                int at = 0;
                if (lane == __ffs(m) - 1) at = atomicAdd(&sm.ncand, __popc(m));
                at = __shfl_sync(0xffffffffu, at, __ffs(m) - 1);
                if (hit) sm.cand[at + __popc(m & ((1u << lane) - 1))] = key;
              }
            }
          }
          __syncthreads();
          ncand = sm.ncand;
        }
      }
    }
    const uint64_t thr = prefix;
    const uint64_t key0 = mono_key(vals[0]);
    const bool need_force = key0 < thr;  // index 0 is the first T-valued element if key0 == thr
    const int quota = need_force ? krem - 1 : krem;

    // per-thread contiguous sub-slices, index order
    const int per = (s1 - s0 + kThreads - 1) / kThreads;
    const int b0 = min(s1, s0 + tid * per), b1 = min(s1, b0 + per);
    int eq = 0, gt = 0;
    double below = -INFINITY, above = INFINITY;
    for (int i0 = b0; i0 < b1; i0 += kU) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = i0 + u < b1 ? vals[i0 + u] : -INFINITY;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (i0 + u >= b1) break;
        const uint64_t key = mono_key(v[u]);
        if (key == thr) ++eq;
        else if (key < thr) below = fmax(below, v[u]);
        else {
          above = fmin(above, v[u]);
          ++gt;
        }
      }
    }
    int eq_base, eq_cta;
    Scan(sm.scan).ExclusiveSum(eq, eq_base, eq_cta);
    __syncthreads();
    if (tau != nullptr) {
      for (int o = 16; o > 0; o >>= 1) {
        below = fmax(below, __shfl_xor_sync(0xffffffffu, below, o));
        above = fmin(above, __shfl_xor_sync(0xffffffffu, above, o));
      }
      // reduce over warps through the hist array (reused as scratch)
      double* wr = reinterpret_cast<double*>(sm.hist);
      if ((tid & 31) == 0) {
        wr[2 * (tid >> 5)] = below;
        wr[2 * (tid >> 5) + 1] = above;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kThreads / 32; ++w) {
          below = fmax(below, wr[2 * w]);
          above = fmin(above, wr[2 * w + 1]);
        }
        *cl.map_shared_rank(&sm.lo[rank], 0) = below;
        *cl.map_shared_rank(&sm.hi[rank], 0) = above;
        *cl.map_shared_rank(&sm.eq[rank], 0) = eq_cta;
      }
    }
    if (tid < kCl) *cl.map_shared_rank(&sm.cnt[0][rank], tid) = eq_cta;
    cl.sync();
    if (tau != nullptr && rank == 0 && tid == 0 && k < n) {
      double lo = -INFINITY, hi = INFINITY;
      int eqs = 0;
      for (int r = 0; r < kCl; ++r) {
        lo = fmax(lo, sm.lo[r]);
        hi = fmin(hi, sm.hi[r]);
        eqs += sm.eq[r];
      }
      const double T = __longlong_as_double((long long)((thr >> 63) ? (thr & ~(1ull << 63)) : ~thr));
      // every entry x of the vector is within x * eta + kFlushAbs of its exact value
      // (eta: vs_tc_combine_kernel; kFlushAbs: <= 64 terms flushed to zero below 2^-126
      // by ex2.approx.ftz), so an order is certain when the intervals do not overlap
      const double eta = (double)(*tau);
      const double v0 = vals[0];
      auto apart = [&](double big, double small) {  // exact big > exact small, guaranteed
        return big * (1.0 - eta) - kFlushAbs > small * (1.0 + eta) + kFlushAbs;
      };
      bool f = eqs > krem;                                   // the k-th value ties with an unselected one
      f |= !apart(T, lo);                                    // k-th vs (k+1)-th
      f |= !(v0 > T ? apart(v0, T) : apart(T, v0));          // index 0 sits on the boundary
      if (v0 < T) f |= krem >= 2 || !apart(hi, T);           // forced 0 drops the k-th: k-th vs (k-1)-th
      if (f) atomicOr(flag, 1);
    }
    int eq_glob = 0;
    for (int r = 0; r < rank; ++r) eq_glob += sm.cnt[0][r];
    // selected count: every key above the threshold, plus this thread's T-valued keys
    // whose global rank among the T-valued ones (index order) is below the quota
    const int sel = gt + min(eq, max(0, quota - (eq_glob + eq_base)));
    int sel_base, sel_cta;
    Scan(sm.scan).ExclusiveSum(sel, sel_base, sel_cta);
    if (tid < kCl) *cl.map_shared_rank(&sm.cnt[1][rank], tid) = sel_cta;
    cl.sync();
    int sel_glob = need_force ? 1 : 0;  // forced index 0 is the smallest index: slot 0
    for (int r = 0; r < rank; ++r) sel_glob += sm.cnt[1][r];
    {
      int r = eq_glob + eq_base;
      int pos = sel_glob + sel_base;
      for (int i0 = b0; i0 < b1; i0 += kU) {
        double v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = i0 + u < b1 ? vals[i0 + u] : -INFINITY;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (i0 + u >= b1) break;
          const uint64_t key = mono_key(v[u]);
          const bool is_eq = key == thr;
          if ((key > thr) || (is_eq && r < quota)) {
            out[descending ? (k - 1 - pos) : pos] = i0 + u;
            ++pos;
          }
          r += is_eq;
        }
      }
    }
    if (need_force && rank == 0 && tid == 0) out[descending ? (k - 1) : 0] = 0;
    cl.sync();  // no CTA leaves while others may still address its shared memory
  }
};

}  // namespace spf
