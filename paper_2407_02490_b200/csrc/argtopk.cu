// argtopk.cu -- spf_argtopk: estimator.argtopk (estimator.py:59-67) on the device.
//
// Indices of the k largest values in descending-value order, ties toward the lower
// index (np.argsort(-x, kind="stable")[:k]).  Two launches on one vector:
//   1. select: block radix select (topk.cuh, BlockTopK) -> the k indices, index order;
//   2. order:  one CTA bitonic-sorts the k (value, index) pairs in shared memory by
//              value descending, index ascending (k <= kMaxSort).
// -0.0 is folded to +0.0 first (argsort(-x) treats them as equal).
#include <algorithm>

#include "spf.h"
#include "spf_internal.h"
#include "topk.cuh"

namespace spf {
namespace {

constexpr int kSelThreads = 256;
constexpr int kMaxSort = 16384;  // 16384 x 12 B of shared memory

__global__ void fold_zero_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] + 0.0;  // -0.0 + 0.0 = +0.0
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const double* __restrict__ vals, int n, int k,
                                                             int32_t* __restrict__ out) {
  using TK = BlockTopK<kSelThreads, double>;
  __shared__ typename TK::Storage sm;
  TK::run(sm, vals, n, k, -1, false, out, 1);
}

// Bitonic sort of m (<= kMaxSort) selected indices by (value desc, index asc).
__global__ void __launch_bounds__(1024) order_kernel(const double* __restrict__ vals, int32_t* __restrict__ idx,
                                                     int m) {
  extern __shared__ uint64_t sk[];  // keys [P2], then indices as int32 [P2]
  int P2 = 1;
  while (P2 < m) P2 <<= 1;
  int32_t* si = reinterpret_cast<int32_t*>(sk + P2);
  for (int i = threadIdx.x; i < P2; i += blockDim.x) {
    if (i < m) {
      const int j = idx[i];
      sk[i] = mono_key(vals[j]);
      si[i] = j;
    } else {
      sk[i] = 0;  // below every real key: sorts last
      si[i] = 0x7fffffff;
    }
  }
  __syncthreads();
  // "a before b" = larger key, or equal key and smaller index
  auto before = [&](int a, int b) { return sk[a] > sk[b] || (sk[a] == sk[b] && si[a] < si[b]); };
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;  // this run is ordered "before"-first
          if (up ? before(j, i) : before(i, j)) {
            const uint64_t tk = sk[i];
            sk[i] = sk[j];
            sk[j] = tk;
            const int32_t ti = si[i];
            si[i] = si[j];
            si[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) idx[i] = si[i];
}

}  // namespace
}  // namespace spf

using namespace spf;

extern "C" {

size_t spf_argtopk_workspace_size(int64_t n) { return (size_t)(n > 0 ? n : 0) * sizeof(double); }

int spf_argtopk(const double* values, int64_t n, int k, int32_t* out, void* workspace, size_t workspace_bytes,
                void* stream) {
  if (k < 1) return set_error(SPF_ERR_INVALID, "k must be >= 1");
  if (n < 0 || n > 0x7fffffff) return set_error(SPF_ERR_INVALID, "bad length %lld", (long long)n);
  if (n == 0) return SPF_OK;
  const int m = (int)std::min<int64_t>(k, n);
  if (m > kMaxSort) return set_error(SPF_ERR_INVALID, "argtopk supports k <= %d (got %d)", kMaxSort, m);
  if (values == nullptr || out == nullptr) return set_error(SPF_ERR_INVALID, "null pointer");
  if (workspace == nullptr || workspace_bytes < spf_argtopk_workspace_size(n))
    return set_error(SPF_ERR_INVALID, "workspace too small");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double* folded = reinterpret_cast<double*>(workspace);
  note_launches(3);
  fold_zero_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(values, folded, n);
  select_kernel<<<1, kSelThreads, 0, st>>>(folded, (int)n, m, out);
  int P2 = 1;
  while (P2 < m) P2 <<= 1;
  const size_t smem = (size_t)P2 * (sizeof(uint64_t) + sizeof(int32_t));
  int rc = check_cuda(cudaFuncSetAttribute(order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "argtopk smem attr");
  if (rc) return rc;
  order_kernel<<<1, 1024, smem, st>>>(folded, out, m);
  return check_cuda(cudaGetLastError(), "argtopk");
}

}  // extern "C"
