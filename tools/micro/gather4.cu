// TMA tile::gather4 (sm_100a) as the conv_ws A-operand gather: 128 rows of 64 bf16 channels picked by
// row index from a 2-D [pixels, C] tensor, 32 gather4 instructions per 16 KB stage, SWIZZLE_128B.
// (1) correctness: the stage bytes equal the K-major SW128 layout the UMMA descriptors expect (row r,
//     16-byte chunk j at r*128 + ((j ^ (r & 7)) << 4)), rows with a negative index zero-filled;
// (2) rate: 148 CTAs x NST stages of random rows (L2-resident tensor), bytes per cycle per SM, with the
//     32 gathers of a stage issued by one thread or spread over 8 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather4 gather4.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
#include "../../paper_2601_13776_b200/csrc/tma_host.h"
using namespace orth;

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int col, int r0, int r1,
                                        int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(umma::smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

constexpr int NSLOT = 4;
template <int MODE>   // 0: one thread issues gather4; 1: 8 warps issue gather4; 2: cp.async by 256 threads
__global__ void __launch_bounds__(288, 1) k(const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* __restrict__ gsrc, const int* __restrict__ rows,
                                             int nst, int nrows_tab, uint8_t* dump, unsigned long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = umma::align1024_smem(sm_raw);
  __shared__ uint64_t full[NSLOT], empty[NSLOT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) { umma::mbar_init(&full[i], MODE == 2 ? 256 : 1); umma::mbar_init(&empty[i], 1); }
    umma::fence_mbar_init();
  }
  __syncthreads();
  const uint32_t base = umma::smem_u32(sm);
  const unsigned long long t0 = clock64();
  if (warp < 8) {   // producers
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NSLOT;
      if (s >= NSLOT) umma::mbar_wait(&empty[slot], ((s / NSLOT) - 1) & 1);
      const uint32_t dst = base + slot * 16384;
      const int* rr = rows + ((size_t)(blockIdx.x * 131 + s) * 128) % (size_t)(nrows_tab - 128);
      if (MODE == 2) {   // conv_ws-style: thread = (row group, 16-byte chunk), 4 rows each
        const int c = tid & 7, rb = tid >> 3;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i, idx = rr[r];
          umma::cp_async16(dst + r * 128 + ((c ^ (r & 7)) << 4), gsrc + (size_t)(idx < 0 ? 0 : idx) * 64 + c * 8, idx >= 0);
        }
        umma::cp_async_mbar_arrive(&full[slot]);
      } else if (MODE == 1) {   // warp w issues gathers 4w .. 4w + 3 (lanes 0..3)
        if (tid == 0) umma::mbar_arrive_expect_tx(&full[slot], 16384);
        __syncwarp();
        asm volatile("bar.sync 1, 256;");
        if (lane < 4) {
          const int g = warp * 4 + lane;
          gather4(dst + g * 512, &tm, &full[slot], 0, rr[4 * g], rr[4 * g + 1], rr[4 * g + 2], rr[4 * g + 3]);
        }
      } else if (tid == 0) {
        umma::mbar_arrive_expect_tx(&full[slot], 16384);
        for (int g = 0; g < 32; ++g)
          gather4(dst + g * 512, &tm, &full[slot], 0, rr[4 * g], rr[4 * g + 1], rr[4 * g + 2], rr[4 * g + 3]);
      }
    }
  } else {   // consumer: wait full, (first stage of CTA 0: dump), release
    for (int s = 0; s < nst; ++s) {
      const int slot = s % NSLOT;
      umma::mbar_wait(&full[slot], (s / NSLOT) & 1);
      if (s == 0 && blockIdx.x == 0)
        for (int i = lane; i < 16384 / 16; i += 32)
          reinterpret_cast<uint4*>(dump)[i] = reinterpret_cast<const uint4*>(sm + slot * 16384)[i];
      __syncwarp();
      if (lane == 0) umma::mbar_arrive(&empty[slot]);
    }
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const int R = 1 << 20, C = 64;   // 1M pixels x 64 channels bf16 = 128 MB (L2-resident share: random rows)
  std::vector<uint16_t> h((size_t)R * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  uint16_t* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  const int NT = 1 << 20;
  std::vector<int> rows(NT);
  srand(7);
  for (int i = 0; i < NT; ++i) rows[i] = (i % 37 == 5) ? -1 : (rand() % (R / 16));   // 1/16 of the tensor: L2
  int* drows;
  cudaMalloc(&drows, NT * 4);
  cudaMemcpy(drows, rows.data(), NT * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  const cuuint32_t box[2] = {64, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = tensor_map_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  uint8_t* dump;
  cudaMalloc(&dump, 16384);
  unsigned long long* out;
  cudaMalloc(&out, 8 * 148);
  auto run = [&](auto kern, const char* name, int nst) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, NSLOT * 16384 + 1024);
    kern<<<148, 288, NSLOT * 16384 + 1024>>>(tm, (const __nv_bfloat16*)d, drows, nst, NT, dump, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long ho[148];
    cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int c = 0; c < 148; ++c) s += (double)ho[c] / 148;
    printf("%-28s %d stages: %.0f cycles/stage, %.1f B/cycle/SM (%s)\n", name, nst, s / nst, 16384.0 * nst / s,
           cudaGetErrorString(e));
    return e;
  };
  if (run(k<0>, "gather4, one thread", 1) != cudaSuccess) return 1;
  // check stage 0 of CTA 0
  std::vector<uint8_t> hd(16384);
  cudaMemcpy(hd.data(), dump, 16384, cudaMemcpyDeviceToHost);
  int bad = 0;
  const int* rr = rows.data();   // CTA 0, stage 0: offset 0
  for (int r = 0; r < 128; ++r)
    for (int j = 0; j < 8; ++j) {
      const uint8_t* got = hd.data() + r * 128 + ((j ^ (r & 7)) << 4);
      for (int b = 0; b < 16; ++b) {
        const int idx = rr[r];
        uint8_t want = 0;
        if (idx >= 0) want = reinterpret_cast<const uint8_t*>(h.data() + (size_t)idx * C + j * 8)[b];
        if (got[b] != want) ++bad;
      }
    }
  printf("layout check: %d bad bytes of 16384 (%s)\n", bad, bad ? "FAIL" : "ok");
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {   // conv-like: consecutive pixels (rows of neighbouring outputs), 1/37 padding rows
      for (int i = 0; i < NT; ++i) rows[i] = (i % 37 == 5) ? -1 : (i % (R / 16));
      cudaMemcpy(drows, rows.data(), NT * 4, cudaMemcpyHostToDevice);
    }
    printf("== %s rows\n", pass ? "consecutive" : "random");
    run(k<0>, "gather4, one thread", 4000);
    run(k<1>, "gather4, 8 warps", 4000);
    run(k<2>, "cp.async, 256 threads", 4000);
  }
  return bad ? 1 : 0;
}
