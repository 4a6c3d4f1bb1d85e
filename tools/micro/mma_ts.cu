// tcgen05.mma issue cost with the A operand in TMEM (ts form) vs shared memory (ss form): one CTA per
// SM, one thread issues NMMA MMAs (M=128, N given, K=16) into one accumulator; optionally each MMA is
// preceded by a tcgen05.cp of its 128 x 256-bit A slice from shared memory (the operand streamed
// through TMEM).  Reports cycles per MMA.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void cp_128x256(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

#include "../../paper_2601_13776_b200/csrc/tma_host.h"
template <int N, int MODE>   // MODE 0: ss; 1: ts, A resident in TMEM; 2: ts + tcgen05.cp per MMA;
                             // 3: ss with both operands MN-major (the NS Gram's column operands);
                             // 4: ss in conv_ws's K-block loop shape: per 4 MMAs an mbarrier wait on an
                             //    already-completed barrier, proxy + tcgen05 fences, a commit to a barrier;
                             // 5: as 4 without the proxy fence; 6: as 4 without the wait;
                             // 7: as 6 while warps 1-3 continuously read the other TMEM half (an epilogue);
                             // 8: as 6 while warps 1-3 continuously write shared memory (st.shared.v4);
                             // 9: as 6 with the operands cycling through 4 distinct 48 KB stages (conv_ws);
                             // 10: as 9 with both operands MN-major (the NS Gram: 2 x 8 KB blocks per operand);
                             // 11: A rows starting at 0 / 58 / 116 (an unaligned window row offset, the kernel-row
                             //     conv), B fixed; 12: as 11 with aligned offsets 0 / 64 / 128;
                             // 13: the kernel-row conv's tile: 3 rows x 4 K steps, A in one of 4 window
                             //     buffers (30 KB apart) at row offsets 0 / 58 / 116, B = 3 stacked 8 KB tap
                             //     tiles per row (24 KB apart), accumulator alternating per tile (256 cols);
                             // 14: as 13 with the epilogue handshake: commit -> tfull[acc], warp 1 waits
                             //     tfull and arrives tempty[acc], the MMA thread waits tempty before a tile;
                             // 15: as 13 while warp 2 streams TMA loads (L2-resident, 16 KB boxes) into a
                             //     separate shared-memory region (a producer's window / weight traffic)
__global__ void __launch_bounds__(128, 1) k(int nmma, unsigned long long* out, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, done_bar, emp[4], tfull[2], tempty[2];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 200704 / 4; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(sm)[i] = (((120u + h % 7u) << 7) | ((h >> 4) & 0x7fu)) * 0x10001u;
  }
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(sm + 200704 - 16) = 0;   // the streamer's stop flag
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_init(&done_bar, 1);
    for (int i = 0; i < 4; ++i) umma::mbar_init(&emp[i], 1);
    for (int i = 0; i < 2; ++i) { umma::mbar_init(&tfull[i], 1); umma::mbar_init(&tempty[i], 1); }
    umma::fence_mbar_init();
  }
  umma::fence_proxy_async_smem();
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  __shared__ uint64_t tbar[2];
  if (MODE == 15 && threadIdx.x == 64) {   // TMA streamer: 2 x 16 KB boxes in flight, until the MMAs finish
    umma::mbar_init(&tbar[0], 1); umma::mbar_init(&tbar[1], 1); umma::fence_mbar_init();
    const uint32_t dst = umma::smem_u32(sm) + 163840;   // 2 x 16 KB past the MMA operands
    for (int it = 0; it < (1 << 20); ++it) {
      const int b = it & 1;
      if (it >= 2) umma::mbar_wait(&tbar[b], ((it >> 1) - 1) & 1);
      if (*reinterpret_cast<volatile int*>(sm + 200704 - 16)) break;
      umma::mbar_arrive_expect_tx(&tbar[b], 16384);
      umma::tma_load_2d(dst + b * 16384, &tm, &tbar[b], 0, (it * 128) & 8191);
    }
  }
  if (MODE == 14 && threadIdx.x == 32) {   // the epilogue stand-in: release each accumulator once full
    for (int t = 0; t < nmma / 12; ++t) {
      umma::mbar_wait(&tfull[t & 1], (t >> 1) & 1);
      umma::tc_fence_after();
      umma::mbar_arrive(&tempty[t & 1]);
    }
  }
  if ((MODE == 7 || MODE == 8) && threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5;
    float acc = 0.f;
    if (MODE == 7) {
      while (!stop) {
        float v[32];
        umma::tmem_ld32(tbase + ((uint32_t)(w * 32) << 16) + 256 + 64 * (w - 1), v);
        acc += v[0];
      }
    } else {
      float4* p = reinterpret_cast<float4*>(sm + 184320);
      int it = 0;
      while (!stop) {
        for (int e = threadIdx.x - 32; e < 1024; e += 96) p[e] = make_float4(it, e, 1.f, 2.f);
        ++it;
      }
    }
    if (acc == 12345.f) out[0] = 1;
  }
  if (threadIdx.x == 0) {
    const uint32_t a = umma::smem_u32(sm), b = a + 65536;
    constexpr uint32_t ID = umma::idesc_bf16(128, N) | (MODE == 3 ? (1u << 15) | (1u << 16) : 0u);
    const uint32_t at = tbase + 256;   // A slices: 8 columns each, 4 of them (one 64-deep K block)
    if (MODE == 1)
      for (int q = 0; q < 4; ++q) cp_128x256(at + 8 * q, umma::sdesc_sw128(a + 32 * q));
    const unsigned long long t0 = clock64();
    if (MODE == 13 || MODE == 14 || MODE == 15) {
      const uint32_t ID13 = umma::idesc_bf16(128, 192);
      for (int t = 0; t < nmma / 12; ++t) {
        if (MODE == 14 && t >= 2) umma::mbar_wait(&tempty[t & 1], ((t >> 1) - 1) & 1);
        umma::tc_fence_after();
        const uint32_t abuf = a + (uint32_t)(t & 3) * 30720u, d = tbase + (uint32_t)(t & 1) * 256u;
        for (int ra = 0; ra < 3; ++ra) {
          const uint32_t aa = abuf + (uint32_t)(ra * 58) * 128u, bb = a + 126976u + (uint32_t)ra * 24576u;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            umma::mma_bf16(d, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), ID13, (ra | q) != 0);
        }
        if (MODE == 14) umma::mma_commit(&tfull[t & 1]);
        else umma::mma_commit(&emp[t & 3]);
      }
    } else if (MODE >= 4) {
      umma::mbar_arrive(&done_bar);   // phase 0 completes: every wait below hits the already-complete path
      for (int kb = 0; kb < nmma / 4; ++kb) {
        if (MODE == 4 || MODE == 5) umma::mbar_wait(&done_bar, 0);
        if (MODE != 5) umma::fence_proxy_async_smem();
        umma::tc_fence_after();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t sa = MODE == 11 ? a + (uint32_t)((kb % 3) * 58) * 128u
                              : MODE == 12 ? a + (uint32_t)((kb % 3) * 64) * 128u
                              : MODE >= 9 ? a + (uint32_t)(kb & 3) * 49152u : a;
          const uint32_t sb = MODE >= 11 ? a + 65536u : MODE >= 9 ? sa + 16384u : b;
          if (MODE == 10)
            umma::mma_bf16(tbase, umma::sdesc_sw128_mn(sa + 2048 * q, 8192), umma::sdesc_sw128_mn(sb + 2048 * q, 8192),
                           ID | (1u << 15) | (1u << 16), (kb | q) != 0);
          else
            umma::mma_bf16(tbase, umma::sdesc_sw128(sa + 32 * q), umma::sdesc_sw128(sb + 32 * q), ID, (kb | q) != 0);
        }
        umma::mma_commit(&emp[kb & 3]);
      }
    }
    for (int i = 0; i < (MODE >= 4 ? 0 : nmma); ++i) {   // (modes >= 4 ran above)
      const int q = i & 3;
      if (MODE == 3) {
        umma::mma_bf16(tbase, umma::sdesc_sw128_mn(a + 2048 * q, 8192), umma::sdesc_sw128_mn(b + 2048 * q, 8192), ID,
                       i > 0);
      } else if (MODE == 0) {
        umma::mma_bf16(tbase, umma::sdesc_sw128(a + 32 * q), umma::sdesc_sw128(b + 32 * q), ID, i > 0);
      } else {
        if (MODE == 2) cp_128x256(at + 8 * q, umma::sdesc_sw128(a + 16384 * ((i >> 2) & 1) + 32 * q));
        mma_ts(tbase, at + 8 * q, umma::sdesc_sw128(b + 32 * q), ID, i > 0);
      }
    }
    umma::mma_commit(&bar);
    umma::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
    *reinterpret_cast<volatile int*>(sm + 200704 - 16) = 1;
  }
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  void* gx;
  cudaMalloc(&gx, 8192 * 512 * 2);
  cudaMemset(gx, 0, 8192 * 512 * 2);
  CUtensorMap tm;
  {
    const cuuint64_t dims[2] = {512, 8192};
    const cuuint64_t strides[1] = {1024};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, gx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 202000);
    const int nm = 65536;
    kern<<<148, 128, 202000>>>(nm, d, tm);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int c = 0; c < 148; ++c) s += (double)h[c] / 148;
    printf("%-28s %.1f cycles/MMA (%s)\n", name, s / nm, cudaGetErrorString(e));
  };
  run(k<192, 13>, "ss  kernel-row conv tile pattern");
  run(k<192, 15>, "ss  ... + concurrent TMA loads");
  run(k<192, 14>, "ss  ... + epilogue handshake");
  run(k<192, 11>, "ss  N=192 A at rows 0/58/116");
  run(k<192, 12>, "ss  N=192 A at rows 0/64/128");
  run(k<128, 11>, "ss  N=128 A at rows 0/58/116");
  run(k<128, 10>, "ss  N=128 4-stage ring MN-major");
  run(k<256, 10>, "ss  N=256 4-stage ring MN-major");
  run(k<256, 9>, "ss  N=256 4-stage ring");
  run(k<128, 9>, "ss  N=128 4-stage ring");
  run(k<256, 7>, "ss  N=256 + TMEM readers");
  run(k<128, 7>, "ss  N=128 + TMEM readers");
  run(k<256, 8>, "ss  N=256 + smem writers");
  run(k<256, 4>, "ss  N=256 conv_ws loop");
  run(k<256, 5>, "ss  N=256 conv_ws loop, no proxy fence");
  run(k<256, 6>, "ss  N=256 conv_ws loop, no wait");
  run(k<128, 3>, "ss  N=128 MN-major A, B");
  run(k<256, 3>, "ss  N=256 MN-major A, B");
  run(k<64, 0>, "ss  N=64");
  run(k<64, 1>, "ts  N=64 (A resident)");
  run(k<64, 2>, "ts  N=64 (+cp per MMA)");
  run(k<128, 0>, "ss  N=128");
  run(k<128, 1>, "ts  N=128 (A resident)");
  run(k<128, 2>, "ts  N=128 (+cp per MMA)");
  run(k<192, 0>, "ss  N=192");
  run(k<192, 1>, "ts  N=192 (A resident)");
  run(k<192, 2>, "ts  N=192 (+cp per MMA)");
  run(k<256, 0>, "ss  N=256");
  run(k<256, 1>, "ts  N=256 (A resident)");
  run(k<256, 2>, "ts  N=256 (+cp per MMA)");
}
