// tcgen05.mma kind::f16 issue/throughput micro-benchmark: one CTA per SM,
// one thread issues NMMA MMAs (M=128, N given, K=16) from smem operands
// (SWIZZLE_128B K-major, zero data), commit + wait; reports cycles per MMA.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
template <int N>
__global__ void __launch_bounds__(128, 1) k(int nmma, int astride, unsigned long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); umma::fence_mbar_init(); }
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = umma::smem_u32(sm), b = a + 32768;
    constexpr uint32_t ID = umma::idesc_bf16(128, N);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t aa = a + (uint32_t)((i % 9) * astride) * 128u;
      umma::mma_bf16(tbase, umma::sdesc_sw128(aa + 32 * (i & 3)), umma::sdesc_sw128(b + 32 * (i & 3)), ID, i > 0);
    }
    umma::mma_commit(&bar);
    umma::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 256);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  unsigned long long h;
  auto run = [&](auto kern, int n, int stride, int ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    kern<<<ctas, 128, 70000>>>(4096, stride, d);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d astride=%2d ctas=%3d: %.1f cycles/MMA (%s)\n", n, stride, ctas, h / 4096.0, cudaGetErrorString(cudaGetLastError()));
  };
  for (int ctas : {1, 148}) {
    run(k<64>, 64, 0, ctas); run(k<64>, 64, 8, ctas); run(k<64>, 64, 1, ctas); run(k<64>, 64, 3, ctas);
    run(k<128>, 128, 0, ctas); run(k<128>, 128, 8, ctas); run(k<256>, 256, 0, ctas);
  }
}
