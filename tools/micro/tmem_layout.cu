// Probe: register layout of tcgen05.ld.16x256b.x4 (thread -> TMEM lane/column) and stmatrix .trans.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
__global__ void k(uint32_t* out, uint16_t* out2) {
  __shared__ uint32_t tbase;
  __shared__ __align__(1024) uint16_t sm[64 * 64];
  if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 64);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t t = tbase;
  const int lane = threadIdx.x;
  // lane L of TMEM, column c := (L << 8) | c, written with 32x32b.x1 per column
  for (int c = 0; c < 64; ++c) {
    uint32_t v = ((uint32_t)lane << 8) | (uint32_t)c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) out[lane * 16 + i] = r[i];
  // stmatrix x4 trans: register i of thread t = (i << 12) | t ; row addresses: matrix t/8 row t%8 -> sm row (t) * 64
  uint32_t a = umma::smem_u32(&sm[lane * 64]);
  uint32_t v0 = (0u << 12) | lane, v1 = (1u << 12) | lane, v2 = (2u << 12) | lane, v3 = (3u << 12) | lane;
  // each 32-bit register holds two b16: low = 2*reg id, high = 2*reg id + 1 (tag them)
  v0 = (v0 & 0xFFF) | ((0u) << 12); 
  uint32_t p0 = ((uint32_t)(0 * 64 + lane * 2)) | ((uint32_t)(0 * 64 + lane * 2 + 1) << 16);
  uint32_t p1 = ((uint32_t)(1 * 64 + lane * 2)) | ((uint32_t)(1 * 64 + lane * 2 + 1) << 16);
  uint32_t p2 = ((uint32_t)(2 * 64 + lane * 2)) | ((uint32_t)(2 * 64 + lane * 2 + 1) << 16);
  uint32_t p3 = ((uint32_t)(3 * 64 + lane * 2)) | ((uint32_t)(3 * 64 + lane * 2 + 1) << 16);
  (void)v0; (void)v1; (void)v2; (void)v3;
  for (int i = lane; i < 64 * 64; i += 32) sm[i] = 0xFFFF;
  __syncwarp();
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(p0), "r"(p1),
               "r"(p2), "r"(p3) : "memory");
  __syncwarp();
  for (int i = lane; i < 32 * 8; i += 32) out2[i] = sm[(i / 8) * 64 + (i % 8)];
  umma::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tbase, 64);
}
int main() {
  uint32_t* d; uint16_t* d2;
  cudaMalloc(&d, 32 * 16 * 4); cudaMalloc(&d2, 256 * 2);
  k<<<1, 32>>>(d, d2);
  uint32_t h[512]; uint16_t h2[256];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 32; t += 1) {
    printf("t%2d:", t);
    for (int i = 0; i < 16; ++i) printf(" L%d/c%d", h[t * 16 + i] >> 8, h[t * 16 + i] & 255);
    printf("\n");
  }
  printf("stmatrix.trans: smem row (addr thread) -> 8 b16 values (tag = reg*64 + thread*2 + half)\n");
  for (int row = 0; row < 32; ++row) {
    printf("row%2d:", row);
    for (int j = 0; j < 8; ++j) { int v = h2[row * 8 + j]; printf(" r%d.t%d.%d", v / 64, (v % 64) / 2, v % 2); }
    printf("\n");
  }
}
