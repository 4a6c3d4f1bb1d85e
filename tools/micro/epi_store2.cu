// Store-pattern micro-benchmark: one 128x128 fp32 tile per CTA (64 KB) written
// (1) float2 by 128 threads, (2) float4 by 128 threads, (3) float4 by 256
// threads, (4) smem staging + cp.async.bulk (one 512 B row per bulk op).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void k(float* F, int ld, int mode, unsigned long long* tt) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int tid = threadIdx.x, nt = blockDim.x;
  const size_t base = (size_t)blockIdx.x * 128 * ld;
  __syncthreads();
  unsigned long long t0 = gt();
  if (mode == 1) {
    for (int e = tid; e < 128 * 64; e += nt) { const int i = e >> 6, j = (e & 63) * 2;
      *reinterpret_cast<float2*>(F + base + (size_t)i * ld + j) = make_float2(i, j); }
  } else if (mode == 2) {
#pragma unroll 4
    for (int e = tid; e < 128 * 32; e += nt) { const int i = e >> 5, j = (e & 31) * 4;
      *reinterpret_cast<float4*>(F + base + (size_t)i * ld + j) = make_float4(i, j, 0, 1); }
  } else if (mode == 4) {   // thread = row, 32 float4 stores along its row
    if (tid < 128) {
      float* row = F + base + (size_t)tid * ld;
#pragma unroll 8
      for (int c = 0; c < 32; ++c) *reinterpret_cast<float4*>(row + 4 * c) = make_float4(tid, c, 0, 1);
    }
  } else if (mode == 5) {   // thread = row, bf16 row (256 B) as 16 x 16 B
    if (tid < 128) {
      uint4* row = reinterpret_cast<uint4*>(reinterpret_cast<char*>(F) + (base + (size_t)tid * ld) * 2);
#pragma unroll 8
      for (int c = 0; c < 16; ++c) row[c] = make_uint4(tid, c, 0, 1);
    }
  } else if (mode == 3) {
    for (int e = tid; e < 128 * 32; e += nt) { const int i = e >> 5, j = (e & 31) * 4;
      sm4[e] = make_float4(i, j, 0, 1); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < 128) {
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm + tid * 128);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(F + base + (size_t)tid * ld), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  __syncthreads();
  unsigned long long t1 = gt();
  if (tid == 0) tt[blockIdx.x] = t1 - t0;
}
int main() {
  const int ld = 512, ctas = 148;
  float* F; unsigned long long* tt;
  cudaMalloc(&F, (size_t)ctas * 128 * ld * 4);
  cudaMalloc(&tt, ctas * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  unsigned long long h[148];
  const int cfgs[][2] = {{1, 128}, {1, 256}, {2, 128}, {2, 256}, {2, 512}, {3, 128}, {3, 256}, {4, 128}, {5, 128}};
  for (auto& c : cfgs)
    for (int rep = 0; rep < 3; ++rep) {
      k<<<ctas, c[1], 65536>>>(F, ld, c[0], tt);
      cudaDeviceSynchronize();
      cudaMemcpy(h, tt, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
      if (rep == 2) printf("mode %d threads %d: in-kernel avg %.2f us (%s)\n", c[0], c[1], avg * 1e-3, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
