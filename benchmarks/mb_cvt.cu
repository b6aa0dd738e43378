// mb_cvt.cu -- issue rate of the softmax's per-element instructions on sm_100a:
// MUFU.EX2, F2FP (cvt.rn.bf16x2.f32) and an integer-pipe bf16x2 pack (IADD + PRMT).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_cvt benchmarks/mb_cvt.cu && ./mb_cvt
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int kMode>
__global__ void loop(uint32_t* out, int iters) {
  float a[8];
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; r[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kMode == 0) {  // MUFU ex2
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
        a[i] = __uint_as_float(__float_as_uint(y) ^ 0x80000000u);  // dependent chain, no other pipe
      } else if (kMode == 1) {  // F2FP pack
        uint32_t y;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(a[i]), "f"(a[i]));
        a[i] = __uint_as_float(y);  // dependent chain
      } else {  // integer pack: round-half-up via IADD, then PRMT of the high halves
        const uint32_t u0 = __float_as_uint(a[i]) + 0x8000u;
        uint32_t y;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(y) : "r"(u0), "r"(u0));
        a[i] = __uint_as_float(y);  // dependent chain
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= r[i] ^ __float_as_uint(a[i]);
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192;
  const char* names[3] = {"MUFU.EX2", "F2FP.BF16 (cvt.rn.bf16x2.f32)", "IADD+PRMT bf16x2 pack"};
  for (int m = 0; m < 3; ++m) {
    auto k = m == 0 ? loop<0> : (m == 1 ? loop<1> : loop<2>);
    k<<<sms, 512>>>(out, 16);
    cudaEventRecord(e0);
    k<<<sms, 512>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int mhz = 0;
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    const double ops = (double)sms * 512 * iters * 8;
    printf("%-32s %.1f thread-ops/clk/SM (at %d MHz nominal)\n", names[m], ops / (ms * 1e-3) / sms / (mhz * 1e3), mhz / 1000);
  }
  return 0;
}
