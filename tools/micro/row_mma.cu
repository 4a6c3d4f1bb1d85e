// The kernel-row conv tile (conv_pad ROW) in isolation: one CTA per SM issues tiles of 3 rows x 4 K
// steps of M=128 N=192 K=16 bf16 MMAs (A in one of 4 window buffers at row offsets 0/58/116, B = 3
// stacked 8 KB tap tiles per row), accumulator alternating per tile.  Bisects why the conv kernel's
// MMAs run slower than this pattern: operand VALUES (positive narrow-range vs signed wide-range vs
// zeros), number of tiles per CTA, block size (idle warps), whole-warp elected issue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o row_mma row_mma.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
__device__ __forceinline__ bool try_wait_once(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
               : "=r"(ok) : "r"(umma::smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// data: 0 = positive, exponents 2^-7..2^-1 (mma_ts's fill); 1 = random sign, exponents 2^-20..2^4;
//       2 = zeros; 3 = random sign, exponents 2^-3..2^1 (normal-like activations)
template <bool WARP_ISSUE, int NCOMMIT = 1, int IWARP = 0, int SPIN = 0>
__global__ void __launch_bounds__(384, 1) k(int ntiles, int data, unsigned long long* out, uint32_t sa, uint32_t sbo, unsigned long long* ns) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, emp[4], emp2[4][4];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 200704 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 0x9e3779b9u * blockIdx.x;
    h ^= h >> 13;
    h *= 0x85ebca6bu;
    h ^= h >> 16;
    uint32_t v;
    if (data == 0) v = (((120u + h % 7u) << 7) | ((h >> 4) & 0x7fu)) * 0x10001u;
    else if (data == 1) v = (((h & 1u) << 15) | ((107u + (h >> 1) % 24u) << 7) | ((h >> 8) & 0x7fu)) |
                            ((((h >> 16) & 1u) << 15) | ((107u + (h >> 17) % 24u) << 7) | ((h >> 24) & 0x7fu)) << 16;
    else if (data == 2) v = 0;
    else v = (((h & 1u) << 15) | ((124u + (h >> 1) % 5u) << 7) | ((h >> 8) & 0x7fu)) |
             ((((h >> 16) & 1u) << 15) | ((124u + (h >> 17) % 5u) << 7) | ((h >> 24) & 0x7fu)) << 16;
    reinterpret_cast<uint32_t*>(sm)[i] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) { umma::mbar_init(&emp[i], 1); for (int j = 0; j < 4; ++j) umma::mbar_init(&emp2[i][j], 1); }
    umma::fence_mbar_init();
  }
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const bool issuer = WARP_ISSUE ? (threadIdx.x >> 5) == IWARP : threadIdx.x == 32 * IWARP;
  // SPIN: warps 4.. wait (try_wait loop) on the final barrier while the MMAs run (1: mbar_wait,
  // 2: mbar_wait with __nanosleep backoff)
  if (SPIN && (threadIdx.x >> 5) >= 4) {
    if (SPIN == 1) umma::mbar_wait(&bar, 0);
    else while (!try_wait_once(&bar, 0)) __nanosleep(200);
  }
  if (issuer) {
    const uint32_t a = umma::smem_u32(sm);
    const unsigned long long t0 = clock64();
    unsigned long long g0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    const uint32_t ID = umma::idesc_bf16(128, 192);
    for (int t = 0; t < ntiles; ++t) {
      umma::tc_fence_after();
      const uint32_t abuf = a + (uint32_t)(t & 3) * sa, d = tbase + (uint32_t)(t & 1) * 256u;
      for (int ra = 0; ra < 3; ++ra) {
        const uint32_t aa = abuf + (uint32_t)(ra * 58) * 128u, bb = a + sbo + (uint32_t)ra * 24576u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (WARP_ISSUE)
            umma::mma_bf16_warp(d, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), ID, (ra | q) != 0);
          else
            umma::mma_bf16(d, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), ID, (ra | q) != 0);
        }
      }
      if (WARP_ISSUE) umma::mma_commit_warp(&emp[t & 3]);
      else umma::mma_commit(&emp[t & 3]);
      for (int c = 1; c < NCOMMIT; ++c) {
        if (WARP_ISSUE) umma::mma_commit_warp(&emp2[c][t & 3]);
        else umma::mma_commit(&emp2[c][t & 3]);
      }
    }
    if (WARP_ISSUE) umma::mma_commit_warp(&bar);
    else umma::mma_commit(&bar);
    umma::mbar_wait(&bar, 0);
    unsigned long long g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    if (threadIdx.x == 32 * IWARP) { out[blockIdx.x] = clock64() - t0; ns[blockIdx.x] = g1 - g0; }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 512);
}

extern "C" int row_mma_main() {
  unsigned long long *d, *dn_;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&dn_, 8 * 148);
  uint32_t SA = 30720, SBO = 126976;
  int GRID = 148, SMEM = 202000, PDL = 0;
  auto run = [&](auto kern, int threads, int ntiles, int data, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    for (int rep = 0; rep < 2; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(GRID);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = SMEM;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = PDL;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, ntiles, data, d, SA, SBO, dn_);
    }
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    unsigned long long hn[148];
    cudaMemcpy(hn, dn_, 8 * 148, cudaMemcpyDeviceToHost);
    double s = 0, sn = 0;
    for (int c = 0; c < GRID; ++c) { s += (double)h[c] / GRID; sn += (double)hn[c] / GRID; }
    const double flops = 2.0 * 128 * 192 * 16 * 12.0 * ntiles * GRID;
    printf("%-52s %.1f cycles/MMA, %.1f ns/MMA, %.0f MHz, %.0f TFLOP/s (%s)\n", name, s / (12.0 * ntiles),
           sn / (12.0 * ntiles), 1e3 * s / sn, flops / sn * 1e-3, cudaGetErrorString(e));
  };
  SA = 29696; SBO = 118784;
  GRID = 147; SMEM = 205824;
  run(k<false, 2, 2>, 384, 49, 3, "thread issue (warp 2), 2 commits, others idle");
  run(k<false, 2, 2, 1>, 384, 49, 3, "... 8 warps spinning in mbar_wait");
  run(k<false, 2, 2, 2>, 384, 49, 3, "... 8 warps polling with nanosleep");
  fflush(stdout);
  return 0;
}

#ifndef ROW_MMA_LIB
int main() { return row_mma_main(); }
#endif
