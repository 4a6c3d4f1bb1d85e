// Per-SM store throughput: a 128x128 fp32 tile (64 KB) + its bf16 copy (32 KB) written
// (a) by TMA tensor stores from shared memory with box (bw cols x bh rows), or
// (b) by 256 threads with float4 / 8-byte stores (the NS epilogue pattern).
// Output matrix ld = 1024 floats (tiles side by side), 8 tiles per CTA, 1 or 148 CTAs.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
#include "../../paper_2601_13776_b200/csrc/tma_host.h"
using namespace orth;
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap mf, const __grid_constant__ CUtensorMap mh,
                                         float* F, __nv_bfloat16* H, int ld, int mode, int bw, int bh, int reps,
                                         unsigned long long* tt) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = umma::align1024_smem(raw);
  float* S = reinterpret_cast<float*>(sm);                       // 128 x 128 fp32, row-major within boxes
  __nv_bfloat16* SH = reinterpret_cast<__nv_bfloat16*>(sm + 65536);
  for (int e = threadIdx.x; e < 16384; e += 256) { S[e] = e * 1e-3f; SH[e] = __float2bfloat16(e * 1e-3f); }
  umma::fence_proxy_async_smem();
  __syncthreads();
  const unsigned long long t0 = gt();
  for (int rep = 0; rep < reps; ++rep) {
    const int t_id = blockIdx.x * reps + rep, per_row = ld / 128;
    const int r0 = (t_id / per_row) * 128, c0 = (t_id % per_row) * 128;
    if (mode == 0) {
      if (threadIdx.x == 0) {
        const int nbx = 128 / bw, nby = 128 / bh;
        for (int by = 0; by < nby; ++by)
          for (int bx = 0; bx < nbx; ++bx) {
            const int box = by * nbx + bx;
            umma::tma_store_2d(&mf, umma::smem_u32(S + box * bw * bh), c0 + bx * bw, r0 + by * bh);
            umma::tma_store_2d(&mh, umma::smem_u32(SH + box * bw * bh), c0 + bx * bw, r0 + by * bh);
          }
        umma::bulk_commit();
        umma::bulk_wait_read0();
      }
      __syncthreads();
    } else {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row0 = (warp & 3) * 32, ch = warp >> 2;
      for (int c = 0; c < 2; ++c)
#pragma unroll 4
        for (int it = 0; it < 8; ++it) {
          const int rr = 4 * it + (lane >> 3), i = r0 + row0 + rr, j = c0 + ch * 64 + c * 32 + (lane & 7) * 4;
          const float4 v = *reinterpret_cast<const float4*>(S + ((rr * 32 + (lane & 7) * 4) & 16383));
          *reinterpret_cast<float4*>(F + (size_t)i * ld + j) = v;
          __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
          *reinterpret_cast<uint2*>(H + (size_t)i * ld + j) = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
        }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) { umma::bulk_wait0(); tt[blockIdx.x] = gt() - t0; }
}
int main(int argc, char** argv) {
  const int ld = 1024, reps = 8;
  float* F; __nv_bfloat16* H; unsigned long long* tt;
  const size_t n = (size_t)148 * reps * 128 * 128;
  cudaMalloc(&F, n * 4); cudaMalloc(&H, n * 2); cudaMalloc(&tt, 148 * 8);
  const size_t rows = n / ld;
  auto enc = tensor_map_encoder();
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024 + 1024);
  int shapes[][2] = {{32, 128}, {32, 32}, {32, 8}, {16, 128}, {8, 128}, {32, 256}};
  for (int ctas : {1, 148})
    for (auto& sh : shapes) {
      const int bw = sh[0], bh = sh[1] > 128 ? 128 : sh[1];
      CUtensorMap mf, mh;
      const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
      const cuuint64_t sf[1] = {(cuuint64_t)ld * 4}, shh[1] = {(cuuint64_t)ld * 2};
      const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
      enc(&mf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, F, dims, sf, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      enc(&mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, dims, shh, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int mode : {0, 1}) {
        if (mode == 1 && bw != 32) continue;
        unsigned long long h[148] = {};
        for (int rep = 0; rep < 3; ++rep) {
          k<<<ctas, 256, 100 * 1024 + 1024>>>(mf, mh, F, H, ld, mode, bw, bh, reps, tt);
          cudaDeviceSynchronize();
        }
        cudaMemcpy(h, tt, ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
        printf("ctas %3d %s box %3dx%3d: %.2f us per tile (96 KB) = %.0f GB/s per SM (%s)\n", ctas,
               mode ? "threads" : "TMA    ", bw, bh, avg * 1e-3 / reps, 98304.0 * reps / avg,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
}
