// Per-SM throughput of 16-byte cp.async (L2-resident source) vs TMA 2-D loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;

template <int LAG, int FENCE>
__global__ void __launch_bounds__(256, 1) cpasync_kernel(const uint8_t* src, int iters, long long* out) {
  extern __shared__ uint8_t sm[];
  const uint32_t s0 = umma::smem_u32(sm);
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int st = it % 8;
    // 16 KB per stage: 256 threads x 4 x 16 B, source spread over 4 MB (L2 resident)
    const uint8_t* base = src + ((size_t)(blockIdx.x * 131 + it * 7919) % 256) * 16384;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      umma::cp_async16(s0 + st * 16384 + (tid + 256 * i) * 16, base + (tid + 256 * i) * 16, true);
    umma::cp_async_commit();
    umma::cp_async_wait<LAG>();
    if (FENCE == 1) umma::fence_proxy_async_smem();
    if (FENCE == 2) { umma::fence_proxy_async_smem(); __syncthreads(); }
  }
  umma::cp_async_wait<0>();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  uint8_t* src; cudaMalloc(&src, 8 << 20); cudaMemset(src, 1, 8 << 20);
  long long* d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int iters = 2000;
  cudaFuncSetAttribute(cpasync_kernel<6, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(cpasync_kernel<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(cpasync_kernel<6, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  for (int rep = 0; rep < 2; ++rep) {
    cpasync_kernel<6, 0><<<148, 256, 8 * 16384>>>(src, iters, d);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("cp.async no fence     : %.1f B/cycle/SM\n", 16384.0 * iters / h[0]);
    cpasync_kernel<6, 1><<<148, 256, 8 * 16384>>>(src, iters, d);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("cp.async + proxy fence: %.1f B/cycle/SM\n", 16384.0 * iters / h[0]);
    cpasync_kernel<6, 2><<<148, 256, 8 * 16384>>>(src, iters, d);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("cp.async + fence+sync : %.1f B/cycle/SM\n", 16384.0 * iters / h[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
