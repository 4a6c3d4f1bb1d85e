// Micro-benchmark of the producer/MMA mbarrier skeleton (no data, no MMA):
// cycles per stage for variants of the empty-barrier signal.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;

template <int S, int MODE>
__global__ void __launch_bounds__(288, 1) skel(int iters, long long* out) {
  __shared__ uint64_t full_bar[S], empty_bar[S];
  __shared__ uint32_t tm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 4) umma::tmem_alloc(&tm, 64);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { umma::mbar_init(&full_bar[i], 128); umma::mbar_init(&empty_bar[i], 1); }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  long long t0 = clock64();
  if (warp < 4) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      umma::mbar_wait(&empty_bar[st], ((it / S) & 1) ^ 1);
      umma::mbar_arrive(&full_bar[st]);
    }
  } else if (warp == 4 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      umma::mbar_wait(&full_bar[st], (it / S) & 1);
      umma::tc_fence_after();
      if (MODE == 0) umma::mma_commit(&empty_bar[st]);
      else umma::mbar_arrive(&empty_bar[st]);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 4) umma::tmem_dealloc(tm, 64);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int iters = 10000;
  skel<8, 0><<<148, 288>>>(iters, d); cudaDeviceSynchronize();
  skel<8, 0><<<148, 288>>>(iters, d); cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  printf("commit-signal : %.1f cycles/stage (err %s)\n", (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
  skel<8, 1><<<148, 288>>>(iters, d); cudaDeviceSynchronize();
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  printf("arrive-signal : %.1f cycles/stage\n", (double)h[0] / iters);
  return 0;
}
