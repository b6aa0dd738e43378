// Softmax step micro-benchmark: the per-row work of one 64-key attention step
// (row max, p = 2^(x*c - m) on MUFU or partly on the FMA pipe, packed row sums,
// bf16 pack), registers only, no TMEM / barriers.  Measures the cycles one step
// costs a warp when W warps share each SMSP, i.e. the softmax floor of the
// attention kernel's period.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_02490_b200/csrc \
//        -o mb_softmax benchmarks/mb_softmax.cu && ./mb_softmax
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "spf_ptx.cuh"

using namespace spf;

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }

template <int kEmu, int kCols>
__global__ void softmax_steps(int steps, float c, uint32_t* sink, long long* cyc) {
  uint32_t x[kCols];
#pragma unroll
  for (int j = 0; j < kCols; ++j) x[j] = __float_as_uint(0.01f * (threadIdx.x * 7 + j * 13) - 3.f);
  float m_run = -INFINITY, l_run = 0.f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int t = 0; t < steps; ++t) {
    // perturb the inputs so nothing is loop-invariant
#pragma unroll
    for (int j = 0; j < kCols; ++j) x[j] ^= (uint32_t)(t & 1);
    float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
    for (int j = 0; j < kCols; j += 8) {
      mx0 = fmax3(mx0, u2f(x[j]), u2f(x[j + 1]));
      mx1 = fmax3(mx1, u2f(x[j + 2]), u2f(x[j + 3]));
      mx2 = fmax3(mx2, u2f(x[j + 4]), u2f(x[j + 5]));
      mx3 = fmax3(mx3, u2f(x[j + 6]), u2f(x[j + 7]));
    }
    const float m_tile = fmax3(mx0, mx1, fmaxf(mx2, mx3)) * c;
    float alpha = 1.f;
    if (m_run == -INFINITY) m_run = m_tile;
    else if (m_tile > m_run + 8.f) { alpha = exp2f(m_run - m_tile); m_run = m_tile; }
    const uint64_t c2 = pack_f32x2(c, c);
    const uint64_t m2 = pack_f32x2(-m_run, -m_run);
    uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    uint32_t ph[kCols / 2];
#pragma unroll
    for (int j = 0; j < kCols; j += 2) {
      const uint64_t y = ffma2(pack_f32x2(u2f(x[j]), u2f(x[j + 1])), c2, m2);
      float p0, p1;
      if (kEmu > 0 && ((j >> 1) % kEmu) == kEmu - 1) {
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
    float sa, sb;
    unpack_f32x2(fadd2(fadd2(s0, s1), fadd2(s2, s3)), sa, sb);
    l_run = l_run * alpha + sa + sb;
#pragma unroll
    for (int j = 0; j < kCols / 2; ++j) acc ^= ph[j];
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(l_run);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kEmu, int kCols>
void run(const char* name, int ctas_per_sm, int warps_per_cta) {
  uint32_t* sink;
  long long* cyc;
  const int blocks = 148 * ctas_per_sm, threads = 32 * warps_per_cta, steps = 2000;
  cudaMalloc(&sink, (size_t)blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  softmax_steps<kEmu, kCols><<<blocks, threads>>>(steps, 0.12f, sink, cyc);
  softmax_steps<kEmu, kCols><<<blocks, threads>>>(steps, 0.12f, sink, cyc);
  cudaDeviceSynchronize();
  long long c[1];
  cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
  const int warps_per_smsp = ctas_per_sm * warps_per_cta / 4;
  printf("%-22s cols=%d  warps/SMSP=%d  %7.1f cyc per step per warp  (%6.1f cyc per SMSP per warp-step)\n", name,
         kCols, warps_per_smsp, (double)c[0] / steps, (double)c[0] / steps / warps_per_smsp);
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 3, 4}) run<0, 64>("mufu only", w, 4);
  for (int w : {2, 4}) run<8, 64>("1/8 pairs on FMA", w, 4);
  for (int w : {2, 4}) run<4, 64>("1/4 pairs on FMA", w, 4);
  for (int w : {2, 4}) run<2, 64>("1/2 pairs on FMA", w, 4);
  for (int w : {2, 4}) run<0, 32>("mufu only", w, 4);
  return 0;
}
