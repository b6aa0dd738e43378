// micro-benchmark: tcgen05.mma.cta_group::2 (CTA pair, M = 256, B split over the pair)
// back-to-back issue / completion rate for the QK (SS) shapes of a 128-row-per-CTA
// attention step, against cta_group::1 M = 128 (mb_mma_issue.cu).  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_02490_b200/csrc \
//        -o mb_mma_pair benchmarks/mb_mma_pair.cu && ./mb_mma_pair
#include <cstdio>
#include <cuda_runtime.h>
#include "spf_ptx.cuh"
using namespace spf;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) k_pair(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {  // one warp of EACH CTA of the pair, same warp id
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sb = smem_u32(smem);
  constexpr uint32_t idesc = umma_idesc_bf16(256, N, 0, 0);
  if (warp == 0 && rank == 0) {  // the leader issues for the pair
    const uint32_t alo = sw128_lo(sb, 0), blo = sw128_lo(sb + 32768, 0);
    constexpr uint32_t hi = sw128_hi(1024);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile(
          "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
          "mov.b64 da, {%1, %2};\n\t"
          "mov.b64 db, {%3, %4};\n\t"
          "elect.sync _|e, 0xffffffff;\n\t"
          "setp.ne.b32 p, %6, 0;\n\t"
          "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(tmem),
          "r"(alo + (i & 3) * 2), "r"(hi), "r"(blo + (i & 3) * 2), "r"(hi), "r"(idesc), "r"(i > 0 ? 1 : 0)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(&bar)),
        "h"((unsigned short)3)
        : "memory");
    const long long t1 = clock64();
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  } else if (warp == 0) {
    mbar_wait(&bar, 0);  // the peer's barrier is signalled by the multicast commit
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
  }
}

template <int N>
__global__ void k_single(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sb = smem_u32(smem);
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
  if (warp == 0) {
    const uint32_t alo = sw128_lo(sb, 0), blo = sw128_lo(sb + 32768, 0);
    constexpr uint32_t hi = sw128_hi(1024);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mma_bf16_ss_w2(tmem, alo + (i & 3) * 2, hi, blo + (i & 3) * 2, hi, idesc, i > 0);
    mma_commit_w(&bar);
    const long long t1 = clock64();
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 16);
  long long h[2];
  const int iters = 4096;
  auto run = [&](auto kern, const char* name, int blocks, double flop_per_mma_per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<<<blocks, 128, 65536>>>(d, iters);
    cudaDeviceSynchronize();
    kern<<<blocks, 128, 65536>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double cyc = (double)h[1] / iters;
    printf("%-34s issue %6.1f  complete %6.1f cyc/mma  -> %6.0f FLOP/cyc/SM (%s)\n", name, (double)h[0] / iters, cyc,
           flop_per_mma_per_sm / cyc, cudaGetErrorString(e));
  };
  run(k_single<64>, "1-CTA M128 N64 K16 (SS)", 148, 2.0 * 128 * 64 * 16);
  run(k_single<128>, "1-CTA M128 N128 K16 (SS)", 148, 2.0 * 128 * 128 * 16);
  run(k_pair<64>, "pair  M256 N64 K16 (SS, B split)", 148, 2.0 * 128 * 64 * 16);
  run(k_pair<128>, "pair  M256 N128 K16 (SS, B split)", 148, 2.0 * 128 * 128 * 16);
  run(k_pair<256>, "pair  M256 N256 K16 (SS, B split)", 148, 2.0 * 128 * 256 * 16);
  return 0;
}
