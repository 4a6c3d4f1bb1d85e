// mbarrier arrival throughput: P producer threads per stage arrive on a stage's "full" barrier
// (cp.async.mbarrier.arrive.noinc with 4 16-byte cp.async each, or none), one consumer thread waits
// full and arrives "empty"; a ring of S stages.  Reports cycles per stage.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;

template <int P, int COPY>
__global__ void __launch_bounds__(288, 1) k(const uint4* __restrict__ g, int iters, unsigned long long* out) {
  constexpr int S = 4;
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { umma::mbar_init(&full[i], P); umma::mbar_init(&empty[i], 1); }
    umma::fence_mbar_init();
  }
  __syncthreads();
  const int tid = threadIdx.x;
  const unsigned long long t0 = clock64();
  if (tid < P) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      if (it >= S) umma::mbar_wait(&empty[s], ((it / S) - 1) & 1);
      if (COPY)
        for (int i = 0; i < 4 * 256 / P; ++i)
          umma::cp_async16(umma::smem_u32(sm) + s * 16384 + (tid + i * P) * 16, g + ((it * 1024 + tid + i * P) & 65535), true);
      umma::cp_async_mbar_arrive(&full[s]);
    }
  } else if (tid == 256) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      umma::mbar_wait(&full[s], (it / S) & 1);
      umma::mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  umma::cp_async_wait<0>();
}

int main() {
  uint4* g;
  cudaMalloc(&g, 65536 * 16);
  cudaMemset(g, 0, 65536 * 16);
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const int iters = 8192;
    kern<<<148, 288, 70000>>>(g, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += (double)h[i] / 148;
    printf("%-40s %.0f cycles/stage (%s)\n", name, c / iters, cudaGetErrorString(e));
  };
  run(k<256, 0>, "256 arrivals, no copies");
  run(k<128, 0>, "128 arrivals, no copies");
  run(k<32, 0>, "32 arrivals, no copies");
  run(k<8, 0>, "8 arrivals, no copies");
  run(k<256, 1>, "256 threads x 4 cp.async (16 KB), L2");
  run(k<128, 1>, "128 threads x 8 cp.async (16 KB), L2");
  run(k<64, 1>, "64 threads x 16 cp.async (16 KB), L2");
}
