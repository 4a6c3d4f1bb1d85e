// tcgen05.mma kind::f16 issue/throughput micro-benchmark: one CTA per SM,
// one thread issues NMMA MMAs (M=128, N given, K=16) from smem operands
// (SWIZZLE_128B K-major, zero data), commit + wait; reports cycles per MMA.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
template <int M, int N>
__global__ void __launch_bounds__(128, 1) k(int nmma, int astride, int bstride, unsigned long long* out, int zero_data) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 98304 / 4; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // two bf16 values in (-1, 1): sign random, exponent 120..126, mantissa random
    const uint32_t lo = ((h & 1u) << 15) | ((120u + (h >> 1) % 7u) << 7) | ((h >> 4) & 0x7fu);
    const uint32_t hi = ((h >> 11 & 1u) << 15) | ((120u + (h >> 12) % 7u) << 7) | ((h >> 16) & 0x7fu);
    reinterpret_cast<uint32_t*>(sm)[i] = zero_data ? 0u : (lo | (hi << 16));
  }
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); umma::fence_mbar_init(); }
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = umma::smem_u32(sm), b = a + 32768;
    constexpr uint32_t ID = umma::idesc_bf16(M, N);
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t aa = a + (uint32_t)((i % 9) * astride) * 128u;
      const uint32_t bb = b + (uint32_t)((i % 9) * bstride) * 128u;
      umma::mma_bf16(tbase, umma::sdesc_sw128(aa + 32 * (i & 3)), umma::sdesc_sw128(bb + 32 * (i & 3)), ID, i > 0);
    }
    umma::mma_commit(&bar);
    umma::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 256);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  unsigned long long h, hg[2];
  int zero = 0;
  auto run = [&](auto kern, int m, int n, int as, int bs, int ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int nm = ctas > 1 ? 262144 : 4096;
    kern<<<ctas, 128, 100000>>>(nm, as, bs, d, zero);
    cudaDeviceSynchronize();
    cudaMemcpy(hg, d, 16, cudaMemcpyDeviceToHost);
    h = hg[0];
    printf("zero=%d M=%3d N=%3d astride=%2d bstride=%2d ctas=%3d: %.1f cycles/MMA, %.1f ns/MMA, clock %.0f MHz (%s)\n", zero, m, n, as,
           bs, ctas, h / (double)nm, hg[1] / (double)nm, 1e3 * h / (double)hg[1], cudaGetErrorString(cudaGetLastError()));
  };
  for (zero = 0; zero < 2; ++zero) {
    run(k<128, 128>, 128, 128, 0, 0, 148); run(k<128, 256>, 128, 256, 0, 0, 148); run(k<64, 256>, 64, 256, 0, 3, 148);
  }
}
