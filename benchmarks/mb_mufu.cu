// MUFU.EX2 throughput on one SM: warps x independent ex2.approx chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mufu benchmarks/mb_mufu.cu && ./mb_mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int kChains>
__global__ void ex2_kernel(float* out, int iters, long long* cyc) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = -0.001f * (threadIdx.x + c);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// packed half-precision ex2 (two exponentials per instruction): bf16x2 / f16x2
template <int kMode>
__global__ void ex2x2_kernel(float* out, int iters, long long* cyc) {
  unsigned x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 0xbc00bc00u + threadIdx.x + c;  // small negative values
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (kMode == 0) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[c]));
      else asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[c]));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  unsigned s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// packed FFMA2 throughput for comparison
__global__ void ffma2_kernel(float* out, int iters, long long* cyc) {
  unsigned long long x[8];
  for (int c = 0; c < 8; ++c) x[c] = 0x3f8000003f800000ull + c;
  const unsigned long long m = 0x3f7fffff3f7fffffull, a = 0x3c0000003c000000ull;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(m), "l"(a));
  }
  __syncthreads();
  const long long t1 = clock64();
  unsigned long long s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 4096 * 8);
  const int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    ex2_kernel<8><<<1, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)warps * 32 * 8 * iters;
    printf("ex2   warps=%2d  %.2f lanes/clk/SM  (%.2f cyc per warp-instr per SMSP)\n", warps, ops / c,
           (double)c / ((double)warps * 8 * iters) * (warps >= 4 ? 4 : warps));
  }
  for (int mode : {0, 1}) {
    for (int warps : {4, 8, 16}) {
      if (mode == 0) ex2x2_kernel<0><<<1, warps * 32>>>(out, iters, cyc);
      else ex2x2_kernel<1><<<1, warps * 32>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)warps * 32 * 8 * iters * 2;  // two exponentials per instruction
      printf("ex2 %s warps=%2d  %.2f exponentials/clk/SM\n", mode == 0 ? "bf16x2" : "f16x2 ", warps, ops / c);
    }
  }
  for (int warps : {4, 8, 16}) {
    ffma2_kernel<<<1, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)warps * 32 * 8 * iters;
    printf("ffma2 warps=%2d  %.2f packed-lanes/clk/SM\n", warps, ops / c);
  }
  return 0;
}
