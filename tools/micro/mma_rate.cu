// tcgen05.mma kind::f16 issue/throughput micro-benchmark: one CTA per SM,
// one thread issues NMMA MMAs (M=128, N given, K=16) from smem operands
// (SWIZZLE_128B K-major, zero data), commit + wait; reports cycles per MMA.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
template <int M, int N, int NACC = 1>
__global__ void __launch_bounds__(128, 1) k(int nmma, int astride, int bstride, unsigned long long* out, int zero_data) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 200704 / 4; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // two bf16 values in (-1, 1): sign random, exponent 120..126, mantissa random
    const uint32_t lo = ((h & 1u) << 15) | ((120u + (h >> 1) % 7u) << 7) | ((h >> 4) & 0x7fu);
    const uint32_t hi = ((h >> 11 & 1u) << 15) | ((120u + (h >> 12) % 7u) << 7) | ((h >> 16) & 0x7fu);
    reinterpret_cast<uint32_t*>(sm)[i] = zero_data == 1 ? 0u : (lo | (hi << 16));
  }
  if (threadIdx.x == 0) *reinterpret_cast<int*>(sm + 200704 - 16) = 0;
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) { umma::mbar_init(&bar, 1); umma::fence_mbar_init(); }
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  if (zero_data >= 2 && threadIdx.x >= 32) {   // concurrent shared-memory writers (96 threads)
    volatile int* stop = reinterpret_cast<volatile int*>(sm + 200704 - 16);
    float4* w = reinterpret_cast<float4*>(sm + 180224);   // 16 KB region past the MMA operands
    int it = 0;
    while (!*stop) {
      for (int e = threadIdx.x - 32; e < 1024; e += 96) w[e] = make_float4(it, e, 1.f, 2.f);
      ++it;
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t a = umma::smem_u32(sm), b = a + 32768;
    constexpr uint32_t ID = umma::idesc_bf16(M, N);
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t aa = a + (uint32_t)((i % 9) * astride) * 128u;
      const uint32_t bb = b + (uint32_t)((i % 9) * bstride) * 128u;
      if (astride < 0) {   // ring mode: every 4 MMAs (one 64-deep K block) move to the next of 5 stages
        const uint32_t st = a + (uint32_t)(((i >> 2) % 4) * (16384 + N * 128));
        umma::mma_bf16(tbase, umma::sdesc_sw128(st + 32 * (i & 3)), umma::sdesc_sw128(st + 16384 + 32 * (i & 3)), ID,
                       i > 0);
        continue;
      }
      umma::mma_bf16(tbase + (uint32_t)((i % NACC) * N), umma::sdesc_sw128(aa + 32 * (i & 3)), umma::sdesc_sw128(bb + 32 * (i & 3)), ID, i >= NACC);
    }
    umma::mma_commit(&bar);
    umma::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = g1 - g0;
    if (zero_data >= 2) *reinterpret_cast<volatile int*>(sm + 200704 - 16) = 1;
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 512);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 148);
  unsigned long long h, hg[2];
  int zero = 0;
  auto run = [&](auto kern, int m, int n, int as, int bs, int ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 210000);
    const int nm = ctas > 1 ? 262144 : 4096;
    kern<<<ctas, 128, 210000>>>(nm, as, bs, d, zero);
    cudaDeviceSynchronize();
    static unsigned long long all[2 * 148];
    cudaMemcpy(all, d, 16 * ctas, cudaMemcpyDeviceToHost);
    hg[0] = hg[1] = 0;
    for (int c = 0; c < ctas; ++c) { hg[0] += all[2 * c] / ctas; hg[1] += all[2 * c + 1] / ctas; }
    h = hg[0];
    printf("zero=%d M=%3d N=%3d astride=%2d bstride=%2d ctas=%3d: %.1f cycles/MMA, %.1f ns/MMA, clock %.0f MHz (%s)\n", zero, m, n, as,
           bs, ctas, h / (double)nm, hg[1] / (double)nm, 1e3 * h / (double)hg[1], cudaGetErrorString(cudaGetLastError()));
  };
  // independent accumulators interleaved (NACC D regions, round robin): does a second accumulator
  // overlap the per-MMA latency?
  run(k<128, 64, 1>, 128, 64, 0, 0, 148);
  run(k<128, 64, 2>, 128, 64, 0, 0, 148);
  run(k<128, 64, 4>, 128, 64, 0, 0, 148);
  run(k<128, 128, 1>, 128, 128, 0, 0, 148);
  run(k<128, 128, 2>, 128, 128, 0, 0, 148);
  run(k<128, 192, 1>, 128, 192, 0, 0, 148);
  run(k<128, 192, 2>, 128, 192, 0, 0, 148);
  run(k<128, 256, 1>, 128, 256, 0, 0, 148);
  run(k<128, 256, 2>, 128, 256, 0, 0, 148);
  run(k<64, 256, 1>, 64, 256, 0, 0, 148);
  run(k<64, 256, 2>, 64, 256, 0, 0, 148);
}
