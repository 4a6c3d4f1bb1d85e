// Replica of the persistent-NS epilogue row pass: 148 CTAs x 8 warps, warp =
// 32 rows x 64 cols of a 128x128 tile; per 4-group: float4 smem acc + C,
// float4 fp32 store, 8-byte bf16 hi (+lo) stores.  mode bit0: fp32 store,
// bit1: lo store, bit2: C from smem; reps tiles per CTA.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t pk(float a, float b) { __nv_bfloat162 v = __floats2bfloat162_rn(a, b); return *reinterpret_cast<uint32_t*>(&v); }
__global__ void __launch_bounds__(288) k(float* F, __nv_bfloat16* H, __nv_bfloat16* L, int ld, int mode, int reps, unsigned long long* tt) {
  __shared__ float S[8][2][512];
  __shared__ volatile int done_flag;
  __shared__ uint32_t tbase;
  __shared__ uint64_t mbar;
  extern __shared__ uint8_t dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { done_flag = 0; umma::mbar_init(&mbar, 1); umma::fence_mbar_init(); }
  if (warp == 8) {   // tensor-core hog: M128 N128 K16 MMAs from shared memory until the row pass ends
    umma::tmem_alloc(&tbase, 128);
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    if (lane == 0 && (mode & 8)) {
      const uint32_t a = (umma::smem_u32(dyn) + 1023) & ~1023u, b = a + 16384;
      const uint32_t ID = umma::idesc_bf16(128, 128);
      for (int i = 0; ; ++i) {
        umma::mma_bf16(tbase, umma::sdesc_sw128(a + 32 * (i & 3)), umma::sdesc_sw128(b + 32 * (i & 3)), ID, i > 0);
        if ((i & 63) == 63 && done_flag) break;
      }
      umma::mma_commit(&mbar);
      umma::mbar_wait(&mbar, 0);
    }
    __syncwarp();
    umma::tc_fence_before();
    __syncthreads();
    umma::tmem_dealloc(tbase, 128);
    return;
  }
  umma::tc_fence_before();
  __syncthreads();
  const int row0 = (warp & 3) * 32, ch = warp >> 2, rsub = lane >> 3, q4 = lane & 7, c4 = q4 * 4;
  for (int e = lane; e < 1024; e += 32) S[warp][e >> 9][e & 511] = e * 0.001f;
  asm volatile("bar.sync 1, 256;");
  const unsigned long long t0 = gt();
  for (int rep = 0; rep < reps; ++rep) {
    const size_t t_id = (size_t)blockIdx.x * reps + rep, per_row = (size_t)ld / 128;   // tiles side by side
    const size_t base = (t_id / per_row) * 128 * (size_t)ld + (t_id % per_row) * 128;
    for (int c = 0; c < 2; ++c) {
#pragma unroll 4
      for (int it = 0; it < 8; ++it) {
        const int rr = 4 * it + rsub, i = row0 + rr, j = ch * 64 + c * 32 + c4;
        const int sw = 4 * (q4 ^ (rr & 7));
        const float4 a = *reinterpret_cast<const float4*>(&S[warp][0][(rr & 15) * 32 + sw]);
        const float4 cv = (mode & 4) ? *reinterpret_cast<const float4*>(&S[warp][1][(rr & 15) * 32 + sw]) : make_float4(0, 0, 0, 0);
        const float o0 = fmaf(0.5f, a.x, cv.x), o1 = fmaf(0.5f, a.y, cv.y), o2 = fmaf(0.5f, a.z, cv.z), o3 = fmaf(0.5f, a.w, cv.w);
        const size_t off = base + (size_t)i * ld + j;
        if (mode & 1) *reinterpret_cast<float4*>(F + off) = make_float4(o0, o1, o2, o3);
        const uint32_t h01 = pk(o0, o1), h23 = pk(o2, o3);
        *reinterpret_cast<uint2*>(H + off) = make_uint2(h01, h23);
        if (mode & 2) *reinterpret_cast<uint2*>(L + off) = make_uint2(pk(o0 - 1.f, o1), pk(o2, o3 - 1.f));
      }
      __syncwarp();
    }
  }
  asm volatile("bar.sync 1, 256;");
  if (threadIdx.x == 0) { tt[blockIdx.x] = gt() - t0; done_flag = 1; }
  umma::tc_fence_before();
  __syncthreads();
}
int main(int argc, char** argv) {
  const int ld = argc > 1 ? atoi(argv[1]) : 128, ctas = argc > 2 ? atoi(argv[2]) : 148, reps = 8;
  float* F; __nv_bfloat16 *H, *L; unsigned long long* tt;
  const size_t n = (size_t)ctas * reps * 128 * ld;
  cudaMalloc(&F, n * 4); cudaMalloc(&H, n * 2); cudaMalloc(&L, n * 2); cudaMalloc(&tt, ctas * 8);
  unsigned long long h[148] = {};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int mode : {0, 1, 3, 5, 7, 8 + 1, 8 + 5, 8 + 7})
    for (int rep = 0; rep < 3; ++rep) {
      k<<<ctas, 288, 40000>>>(F, H, L, ld, mode, reps, tt);
      cudaDeviceSynchronize();
      cudaMemcpy(h, tt, ctas * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < ctas; ++i) avg += h[i]; avg /= ctas;
      if (rep == 2) printf("ctas %d ld %d mode %d: %.2f us per 128x128 tile (%s)\n", ctas, ld, mode, avg * 1e-3 / reps, cudaGetErrorString(cudaGetLastError()));
    }
}
