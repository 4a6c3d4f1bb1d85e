// Micro-benchmark: cost of the NS epilogue store pattern (per CTA one 128x128
// tile, 128 threads, half-warp per row) -- bf16 pairs and fp32 pairs.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
__global__ void st_pattern(float* F, uint32_t* B, int ld, int mode, unsigned long long* tt) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  const int rr0 = lane >> 4, cc = 2 * (lane & 15);
  const size_t base = (size_t)blockIdx.x * 128 * ld;
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int i = warp * 32 + 2 * it + rr0, j = c * 32 + cc;
      const float o0 = i * 0.5f + j, o1 = o0 + 1.f;
      if (mode & 1) *reinterpret_cast<float2*>(F + base + (size_t)i * ld + j) = make_float2(o0, o1);
      if (mode & 2) B[(base + (size_t)i * ld + j) / 2] = __float_as_uint(o0) ^ __float_as_uint(o1);
    }
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (tid == 0) tt[blockIdx.x] = t1 - t0;
}
int main() {
  const int ld = 512, ctas = 148;
  float* F; uint32_t* B; unsigned long long* tt;
  cudaMalloc(&F, (size_t)ctas * 128 * ld * 4);
  cudaMalloc(&B, (size_t)ctas * 128 * ld * 2);
  cudaMalloc(&tt, ctas * 8);
  unsigned long long h[148];
  for (int mode = 1; mode <= 3; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      st_pattern<<<ctas, 128>>>(F, B, ld, mode, tt);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, tt, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
      printf("mode %d rep %d: kernel %.2f us, in-kernel avg %.2f us\n", mode, rep, ms * 1e3, avg * 1e-3);
    }
  return 0;
}
