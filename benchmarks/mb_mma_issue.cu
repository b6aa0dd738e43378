// micro-benchmark: back-to-back tcgen05.mma issue rate (M128 N64/N128 K16, bf16, SS)
#include <cstdio>
#include <cuda_runtime.h>
#include "spf_ptx.cuh"
using namespace spf;
template <int N, int kWarpWide>
__global__ void k_issue(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t sb = smem_u32(smem);
  constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
  if (warp == 0) {
    const uint32_t alo = sw128_lo(sb, 0), blo = sw128_lo(sb + 32768, 0);
    constexpr uint32_t hi = sw128_hi(1024);
    long long t0 = clock64();
    if (kWarpWide) {
      for (int i = 0; i < iters; ++i)
        mma_bf16_ss_w2(tmem, alo + (i & 3) * 2, hi, blo + (i & 3) * 2, hi, idesc, i > 0);
      mma_commit_w(&bar);
    } else if (lane == 0) {
      for (int i = 0; i < iters; ++i) {
        const uint64_t ad = umma_desc_sw128(sb + (i & 3) * 32, 0, 1024), bd = umma_desc_sw128(sb + 32768 + (i & 3) * 32, 0, 1024);
        mma_bf16_ss(tmem, ad, bd, idesc, i > 0);
      }
      mma_commit(&bar);
    }
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}
int main() {
  long long* d; cudaMalloc(&d, 1024 * 16);
  long long h[2];
  const int iters = 4096;
  auto run = [&](auto kern, const char* name, int blocks) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<<<blocks, 128, 65536>>>(d, iters); cudaDeviceSynchronize();
    kern<<<blocks, 128, 65536>>>(d, iters); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-28s blocks=%3d  issue %.1f cyc/mma   complete %.1f cyc/mma  (%s)\n", name, blocks, (double)h[0] / iters, (double)h[1] / iters, cudaGetErrorString(e));
  };
  run(k_issue<64, 0>, "N64 lane0", 148);
  run(k_issue<64, 1>, "N64 warp-wide elect", 148);
  run(k_issue<128, 0>, "N128 lane0", 148);
  run(k_issue<128, 1>, "N128 warp-wide elect", 148);
  run(k_issue<256, 1>, "N256 warp-wide elect", 148);
  run(k_issue<64, 1>, "N64 warp-wide 2 CTA/SM", 296);
  return 0;
}
