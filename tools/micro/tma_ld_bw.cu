// Per-SM TMA load throughput from L2: `ctas` CTAs (one per SM), each streams 128 x 64 BF16 boxes
// (16 KB, SWIZZLE_128B) of an L2-resident matrix through a ring of `S` 32 KB stages (two boxes per
// stage, like one K block of a 128 x 128 tile: A + B), one producer thread, one consumer thread that
// only waits and releases.  Reports GB/s per SM and in total.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
#include "../../paper_2601_13776_b200/csrc/tma_host.h"
using namespace orth;

template <int S, int BR>   // BR: box rows (64 / 128 / 256): 32 KB per stage = 32768 / (BR * 128) TMAs
__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap tm, int rows, int iters,
                                           unsigned long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { umma::mbar_init(&full[i], 1); umma::mbar_init(&empty[i], 1); }
    umma::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t base = umma::smem_u32(sm);
  const int nbox = rows / 128;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      if (it >= S) umma::mbar_wait(&empty[s], ((it / S) - 1) & 1);
      umma::mbar_arrive_expect_tx(&full[s], 32768);
      constexpr int NB = 32768 / (BR * 128);
#pragma unroll
      for (int j = 0; j < NB; ++j)
        umma::tma_load_2d(base + s * 32768 + j * BR * 128, &tm, &full[s], (it & 7) * 64,
                          ((blockIdx.x * 7 + it * NB + j) & (nbox - 1)) * 128);
    }
    umma::mbar_wait(&empty[(iters - 1) % S], ((iters - 1) / S) & 1);
    out[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      umma::mbar_wait(&full[s], (it / S) & 1);
      umma::mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  const int rows = 8192, cols = 512;   // 8 MB BF16: L2 resident after the first pass
  void* x;
  cudaMalloc(&x, (size_t)rows * cols * 2);
  cudaMemset(x, 0, (size_t)rows * cols * 2);
  CUtensorMap tm;
  auto enc = tensor_map_encoder();
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  CUtensorMap tms[3];
  const cuuint32_t es[2] = {1, 1};
  for (int i = 0; i < 3; ++i) {
    const cuuint32_t box[2] = {64, (cuuint32_t)(64 << i)};
    enc(&tms[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto run = [&](auto kern, int S, int ctas, const CUtensorMap& tm, int br) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 32768 + 1024);
    const int iters = 4096;
    kern<<<ctas, 64, S * 32768 + 1024>>>(tm, rows, 64, d);   // warm L2
    kern<<<ctas, 64, S * 32768 + 1024>>>(tm, rows, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 8 * ctas, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int c = 0; c < ctas; ++c) cyc += (double)h[c] / ctas;
    const double bpc = (double)iters * 32768 / cyc;   // bytes per cycle per SM
    printf("box rows %3d S=%d ctas=%3d: %.1f B/cycle/SM = %.0f GB/s/SM at %.0f MHz, total %.0f GB/s (%s)\n", br, S, ctas, bpc,
           bpc * clk * 1e-6, clk * 1e-3, bpc * clk * 1e-6 * ctas, cudaGetErrorString(e));

  };
  for (int ctas : {1, 148}) {
    run(k<4, 64>, 4, ctas, tms[0], 64);
    run(k<4, 128>, 4, ctas, tms[1], 128);
    run(k<4, 256>, 4, ctas, tms[2], 256);
    run(k<6, 64>, 6, ctas, tms[0], 64);
    run(k<6, 256>, 6, ctas, tms[2], 256);
  }
}
