// conv_pad's kernel-row MMA issue loop (ROW branch), copied with its runtime parameters, its ring
// counters, its waits and commits, in isolation: a fake producer warp arrives on a_full, 8 fake
// epilogue warps wait tfull and arrive tempty.  Measures cycles per tile against the 12-MMA floor
// (1160) and bisects which part of the loop costs time (VARIANT).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o row_mma2 row_mma2.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2601_13776_b200/csrc/umma.cuh"
using namespace orth;
__device__ __forceinline__ uint32_t test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
               : "=r"(ok) : "r"(umma::smem_u32(bar)), "r"(parity) : "memory");
  return ok;
}

struct Args {
  int k, d, P, cr_g, nabuf, abuf_bytes, bres, tiles_m, num_tiles, tiles_per_cta, sb, delay;
};

// V: feature bits -- 1 no waits (producer + epilogue idle); 2 kernel rows compile-time 3; 4 no bres
// checks (resident weights assumed); 8 one tcgen05 fence per tile; 16 compile-time idesc; 32 descriptors
// rebuilt per MMA from byte addresses; 64 one commit per tile (a_empty only)
template <int V>
__global__ void __launch_bounds__(384, 1) k(const __grid_constant__ Args a, unsigned long long* out, unsigned long long* wt) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t a_full[4], a_empty[4], b_full[16], b_empty[16], tfull_bar[2], tempty_bar[2], done, done2;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int SB = a.sb, NA = a.nabuf;
  constexpr int B_BYTES = 64 * 128, ACC_COLS = 256;
  const int bst_bytes = a.k * B_BYTES;
  if (warp == 2) umma::tmem_alloc(&tmem_base_sh, 512);
  if (tid == 0) {
    for (int i = 0; i < NA; ++i) { umma::mbar_init(&a_full[i], 1); umma::mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < SB; ++i) { umma::mbar_init(&b_full[i], 1); umma::mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { umma::mbar_init(&tfull_bar[i], 1); umma::mbar_init(&tempty_bar[i], 256); }
    umma::mbar_init(&done, 1);
    umma::mbar_init(&done2, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t abase = (umma::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bbase = abase + NA * a.abuf_bytes;
  const int kk2 = a.k * a.k;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int t_end = min(a.num_tiles, t_begin + a.tiles_per_cta);
  constexpr bool NOWAIT = V & 1;
  if (warp == 0 && !NOWAIT) {   // fake A producer
    if (lane == 0) {
      int u = 0;
      for (int tile = t_begin; tile < t_end; ++tile, ++u) {
        const int ab = u % NA;
        if (u >= NA) umma::mbar_wait(&a_empty[ab], ((u / NA) - 1) & 1);
        umma::mbar_arrive(&a_full[ab]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) umma::mbar_arrive(&b_full[0]);
  } else if (warp >= 4 && !NOWAIT) {   // fake epilogue
    int tcount = 0;
    for (int tile = t_begin; tile < t_end; ++tile, ++tcount) {
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
    }
  } else if (warp == 2 || ((V & 512) && warp == 3)) {
    if (lane == 0) {
      const int wi = (V & 512) ? warp - 2 : 0, nw = (V & 512) ? 2 : 1;   // issuer index, issuers
      const unsigned long long c0_ = clock64();
      const uint64_t a_desc0 = umma::sdesc_sw128(abase), b_desc0 = umma::sdesc_sw128(bbase);
      const uint32_t a_buf16 = (uint32_t)a.abuf_bytes >> 4, a_row16 = (uint32_t)(a.d * a.P) * 8u;
      const uint32_t b_row16 = (uint32_t)(a.k * B_BYTES) >> 4, b_set16 = (uint32_t)(kk2 * B_BYTES) >> 4;
      const uint32_t b_st16 = (uint32_t)bst_bytes >> 4;
      const uint32_t idesc_row = (V & 16) ? umma::idesc_bf16(128, 192) : umma::idesc_bf16(128, a.k * 64);
      const int KR = (V & 2) ? 3 : a.k;
      const bool BRES = (V & 4) ? true : (bool)a.bres;
      int ab = 0, aph = 0, st = 0, bph = 0, tcount = 0, cur = -1, loads = 0;
      unsigned long long wt_t = 0, wt_a = 0;
      uint32_t ready_next = 0, look_t = 0, look_a = 0;
      const int tb = a.bres ? blockIdx.x * a.tiles_per_cta : blockIdx.x;
      const int te = a.bres ? min(a.num_tiles, tb + a.tiles_per_cta) : a.num_tiles;
      const int ts = a.bres ? 1 : gridDim.x;
      tcount = wi;
      if (V & 512) { ab = wi % NA; aph = 0; }
      for (int tile = tb + wi * ts; tile < te; tile += nw * ts, tcount += nw) {
        if (V & 512) { ab = tcount % NA; aph = (tcount / NA) & 1; }
        if (!(V & 4) && a.bres) {
          const int set = tile / a.tiles_m;
          if (set != cur) {
            if (loads > 0) umma::mma_commit(&b_empty[0]);
            umma::mbar_wait_uni(&b_full[0], loads & 1);
            cur = set;
            ++loads;
          }
        }
        const int acc = tcount & 1;
        unsigned long long w0 = clock64();
        const bool skip = (V & 128) && ready_next;
        if (!NOWAIT && !skip) {
          if (V & 1024) { if (!test_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1)) umma::mbar_wait_uni(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1); }
          else umma::mbar_wait_uni(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
        }
        wt_t += clock64() - w0;
        if (!(V & 8)) umma::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * ACC_COLS;
        uint64_t bset = b_desc0;
        for (int c0 = 0; c0 < a.cr_g; c0 += 64, bset += b_set16) {
          w0 = clock64();
          if (!NOWAIT && !(skip && c0 == 0)) {
            if (V & 1024) { if (!test_wait(&a_full[ab], aph)) umma::mbar_wait_uni(&a_full[ab], aph); }
            else umma::mbar_wait_uni(&a_full[ab], aph);
          }
          wt_a += clock64() - w0;
          umma::tc_fence_after();
          uint64_t ad = a_desc0 + ab * a_buf16;
          for (int ra = 0; ra < KR; ++ra, ad += a_row16) {
            uint64_t bd = bset + ra * b_row16;
            if (!BRES) {
              umma::mbar_wait_uni(&b_full[st], bph);
              umma::tc_fence_after();
              bd = b_desc0 + st * b_st16;
            }
            const uint32_t acc0 = (c0 | ra) != 0;
            if (V & 32) {
              const uint32_t aa = abase + ab * a.abuf_bytes + (uint32_t)(a.d * ra * a.P) * 128u, bb = bbase + ra * 24576u;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                umma::mma_bf16(d_tmem, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), idesc_row, acc0 | (q != 0));
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) umma::mma_bf16(d_tmem, ad + 2 * q, bd + 2 * q, idesc_row, acc0 | (q != 0));
            }
            if ((V & 128) && ra == 0 && c0 + 64 >= a.cr_g) {   // look ahead: the next tile's barriers
              const int acc_n = (tcount + 1) & 1;
              look_t = test_wait(&tempty_bar[acc_n], (((tcount + 1) >> 1) & 1) ^ 1);
              const int ab_n = ab + 1 == NA ? 0 : ab + 1;
              look_a = test_wait(&a_full[ab_n], ab + 1 == NA ? aph ^ 1 : aph);
            }
            if (!BRES) {
              umma::mma_commit(&b_empty[st]);
              if (++st == SB) { st = 0; bph ^= 1; }
            }
          }
          umma::mma_commit(&a_empty[ab]);
          if (++ab == NA) { ab = 0; aph ^= 1; }
        }
        if (!(V & 64) || !NOWAIT) umma::mma_commit(&tfull_bar[acc]);
        if (V & 256) {   // a fixed stall of the issuing thread per tile (calibrates the MMA queue depth)
          const long long e0 = clock64();
          while (clock64() - e0 < a.delay) {
          }
        }
        ready_next = look_t & look_a;
      }
      umma::mma_commit(wi ? &done2 : &done);
      umma::mbar_wait(wi ? &done2 : &done, 0);
      if (wi == 0) {
        out[blockIdx.x] = (clock64() - c0_) / (unsigned long long)(te - tb);
        wt[2 * blockIdx.x] = wt_t / (te - tb);
        wt[2 * blockIdx.x + 1] = wt_a / (te - tb);
      }
    }
    __syncwarp();
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 2) umma::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long *d, *w;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&w, 16 * 148);
  Args a{3, 1, 58, 64, 4, 29696, 1, 7168, 7168, 49, 1, 0};
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 205824);
    for (int rep = 0; rep < 2; ++rep) kern<<<147, 384, 205824>>>(a, d, w);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[147];
    cudaMemcpy(h, d, 8 * 147, cudaMemcpyDeviceToHost);
    unsigned long long hw[2 * 147];
    cudaMemcpy(hw, w, 16 * 147, cudaMemcpyDeviceToHost);
    double s = 0, s1 = 0, s2 = 0;
    for (int c = 0; c < 147; ++c) { s += (double)h[c] / 147; s1 += (double)hw[2 * c] / 147; s2 += (double)hw[2 * c + 1] / 147; }
    printf("%-48s %.0f cycles/tile (floor 1160), waits: tempty %.0f, a_full %.0f (%s)\n", name, s, s1, s2, cudaGetErrorString(e));
  };
  run(k<4 | 2>, "waits, k=3, one issuer");
  run(k<4 | 2 | 1024>, "waits, k=3, one issuer, test_wait first");
  run(k<4 | 2 | 512>, "waits, k=3, two issuers");
  run(k<4 | 2 | 512 | 1024>, "waits, k=3, two issuers, test_wait first");
  run(k<1 | 2 | 4>, "no waits, k=3");
  return 0;
}
