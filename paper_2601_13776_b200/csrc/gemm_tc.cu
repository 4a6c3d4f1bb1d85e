// Batched ragged GEMM on the 5th-generation tensor cores for the Bjorck / NS
// iteration (a3) and, FP32-accurately, the composition chain
// (a4/a5).  Same problem descriptors as the SIMT kernel (plan.cpp):
//   D = alpha * sum_seg opA(seg) opB(seg) + beta * C + diag * I
// with FP32 operands in global memory at arbitrary (row, k) strides.
//
// Loader: 256 threads read FP32 (float4 when aligned), optionally subtract
// the A2 operand, convert to BF16 (RNE) -- and for npass = 3 also the
// residual lo = bf16(x - hi) -- and store K-major SWIZZLE_128B tiles
// (K-contiguous sources directly, MN-contiguous sources via 8x4 register
// transposes).  MMA: one thread issues tcgen05.mma M=128, N=128, K=16 (x4 per
// 64-wide K block; x3 for the split passes hi*hi + hi*lo + lo*hi, which makes
// the product accurate to ~2^-16, reading R16), committing to the stage's
// mbarrier; the FP32 accumulator lives in TMEM (128 columns).  Epilogue:
// 8 warps (lane quarter x column half) apply alpha/beta/diag and store FP32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"
#include "umma.cuh"

namespace orth {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 64;

__device__ __forceinline__ int find_problem_tc(const GemmDesc* __restrict__ d, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tc_tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// hi/lo split of a pair: hi = bf16(x), lo = bf16(x - hi)
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const float2 hf = __bfloat1622float2(h);
  __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}

// Load a ROWS x 64 tile of operand X(r, k) = base[r*sr + k*sk] (- base2[...])
// for rows [r0, r0 + ROWS) and k in [k0, k0 + 64), zero outside [0,R) x [0,K).
template <int ROWS, bool SPLIT>
__device__ __forceinline__ void load_tile(const float* __restrict__ base, const float* __restrict__ base2, int64_t sr,
                                          int64_t sk, int r0, int R, int k0, int K, uint8_t* hi_tile,
                                          uint8_t* lo_tile) {
  const int tid = threadIdx.x;
  if (sk == 1) {
    // K-contiguous: ROWS/... threads per row, each 64*ROWS/256 consecutive floats
    constexpr int TPR = 256 / ROWS;          // threads per row: 2 (ROWS=128)
    constexpr int PER = 64 / TPR;            // floats per thread: 32
    const int r = tid / TPR, part = tid % TPR;
    const int gr = r0 + r, kb = k0 + part * PER;
    float v[PER];
    const float* src = base + (int64_t)gr * sr + kb;
    const float* src2 = base2 ? base2 + (int64_t)gr * sr + kb : nullptr;
    const bool full = gr < R && kb + PER <= K && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                      (!src2 || (reinterpret_cast<uintptr_t>(src2) & 15) == 0);
    if (full) {
#pragma unroll
      for (int i = 0; i < PER / 4; ++i) {
        float4 t = reinterpret_cast<const float4*>(src)[i];
        if (src2) {
          const float4 u = reinterpret_cast<const float4*>(src2)[i];
          t.x -= u.x; t.y -= u.y; t.z -= u.z; t.w -= u.w;
        }
        v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const bool ok = gr < R && kb + i < K;
        v[i] = ok ? src[i] - (src2 ? src2[i] : 0.f) : 0.f;
      }
    }
    const int c0 = part * (PER / 8);
#pragma unroll
    for (int c = 0; c < PER / 8; ++c) {
      uint32_t h[4], l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (SPLIT) split_pair(v[8 * c + 2 * j], v[8 * c + 2 * j + 1], h[j], l[j]);
        else h[j] = pack_bf16(v[8 * c + 2 * j], v[8 * c + 2 * j + 1]);
      }
      const uint32_t off = umma::sw128_off(r, c0 + c);
      *reinterpret_cast<uint4*>(hi_tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
      if (SPLIT) *reinterpret_cast<uint4*>(lo_tile + off) = make_uint4(l[0], l[1], l[2], l[3]);
    }
  } else {
    // row-contiguous (sr == 1) or generic: 8 rows x 4 k per block
    constexpr int NB = (ROWS / 8) * 16;
    for (int b = tid; b < NB; b += 256) {
      const int rb = b % (ROWS / 8), kq = b / (ROWS / 8);
      const int rr = rb * 8, kk = kq * 4;
      float v[4][8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gk = k0 + kk + j, gr = r0 + rr;
        const float* src = base + (int64_t)gk * sk + (int64_t)gr * sr;
        const float* src2 = base2 ? base2 + (int64_t)gk * sk + (int64_t)gr * sr : nullptr;
        const bool full = sr == 1 && gk < K && gr + 8 <= R && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                          (!src2 || (reinterpret_cast<uintptr_t>(src2) & 15) == 0);
        if (full) {
          float4 t0 = reinterpret_cast<const float4*>(src)[0], t1 = reinterpret_cast<const float4*>(src)[1];
          if (src2) {
            const float4 u0 = reinterpret_cast<const float4*>(src2)[0], u1 = reinterpret_cast<const float4*>(src2)[1];
            t0.x -= u0.x; t0.y -= u0.y; t0.z -= u0.z; t0.w -= u0.w;
            t1.x -= u1.x; t1.y -= u1.y; t1.z -= u1.z; t1.w -= u1.w;
          }
          v[j][0] = t0.x; v[j][1] = t0.y; v[j][2] = t0.z; v[j][3] = t0.w;
          v[j][4] = t1.x; v[j][5] = t1.y; v[j][6] = t1.z; v[j][7] = t1.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool ok = gk < K && gr + i < R;
            const int64_t o = (int64_t)gk * sk + (int64_t)(gr + i) * sr;
            v[j][i] = ok ? base[o] - (base2 ? base2[o] : 0.f) : 0.f;
          }
        }
      }
      const uint32_t chunk = kk >> 3, sub = (kk & 7) * 2;   // byte offset inside the 16-byte chunk: 0 or 8
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t off = umma::sw128_off(rr + i, chunk) + sub;
        uint32_t h0, h1, l0, l1;
        if (SPLIT) {
          split_pair(v[0][i], v[1][i], h0, l0);
          split_pair(v[2][i], v[3][i], h1, l1);
          *reinterpret_cast<uint2*>(lo_tile + off) = make_uint2(l0, l1);
        } else {
          h0 = pack_bf16(v[0][i], v[1][i]);
          h1 = pack_bf16(v[2][i], v[3][i]);
        }
        *reinterpret_cast<uint2*>(hi_tile + off) = make_uint2(h0, h1);
      }
    }
  }
}

template <int NPASS, int S>
__global__ void __launch_bounds__(256, (NPASS == 1 ? 2 : 1))
    gemm_tc_kernel(const GemmDesc* __restrict__ descs, int ndesc, const GemmSeg* __restrict__ segs, float* b0,
                   float* b1, float* b2, float* b3) {
  constexpr bool SPLIT = NPASS == 3;
  constexpr int TILE = 128 * 128;                     // bytes of one 128 x 64 bf16 tile
  constexpr int STAGE = (SPLIT ? 4 : 2) * TILE;       // A_hi, B_hi (, A_lo, B_lo)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const GemmDesc d = descs[find_problem_tc(descs, ndesc, blockIdx.x)];
  float* bufs[4] = {b0, b1, b2, b3};
  const int local = blockIdx.x - d.tc_tile_begin;
  const int m0 = (local / d.tc_tiles_n) * TBM, n0 = (local % d.tc_tiles_n) * TBN;

  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, TBN);
  if (tid == 32) {
    for (int i = 0; i < S; ++i) umma::mbar_init(&empty_bar[i], 1);
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  constexpr uint32_t IDESC = umma::idesc_bf16(TBM, TBN);

  const int nkb = (d.K + TBK - 1) / TBK;
  const int nk = nkb * d.seg_count;
  for (int kb = 0; kb < nk; ++kb) {
    const int st = kb % S;
    if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
    const GemmSeg sg = segs[d.seg_begin + kb / nkb];
    const int k0 = (kb % nkb) * TBK;
    uint8_t* stage = smem + st * STAGE;
    const float* A = bufs[d.a_buf] + sg.a_off;
    const float* A2 = sg.a2_off >= 0 ? bufs[d.a_buf] + sg.a2_off : nullptr;
    const float* B = bufs[d.b_buf] + sg.b_off;
    load_tile<TBM, SPLIT>(A, A2, d.sa_m, d.sa_k, m0, d.M, k0, d.K, stage, stage + 2 * TILE);
    load_tile<TBN, SPLIT>(B, nullptr, d.sb_n, d.sb_k, n0, d.N, k0, d.K, stage + TILE, stage + 3 * TILE);
    umma::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      umma::tc_fence_after();
      const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t acc = (kb | q) != 0;
        umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, acc);
        if (SPLIT) {
          umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
          umma::mma_bf16(tmem, umma::sdesc_sw128(al + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, 1);
        }
      }
      umma::mma_commit(&empty_bar[st]);
    }
  }
  if (tid == 0) umma::mma_commit(&done_bar);
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();

  const int q = warp & 3, half = warp >> 2;
  const int gi = m0 + q * 32 + lane;
  const float* C = d.c_off >= 0 ? bufs[d.c_buf] + d.c_off : nullptr;
  float* D = bufs[d.d_buf] + d.d_off;
#pragma unroll
  for (int cc = 0; cc < TBN / 2; cc += 32) {
    const int col = half * (TBN / 2) + cc;
    float v[32];
    umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
    if (gi < d.M) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int gj = n0 + col + j;
        if (gj < d.N) {
          float o = d.alpha * v[j];
          if (C) o = fmaf(d.beta, C[(int64_t)gi * d.ldc + gj], o);
          if (gi == gj) o += d.diag;
          D[(int64_t)gi * d.ldd + gj] = o;
        }
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, TBN);
}

template <int NPASS, int S>
int launch_tc_impl(const GemmPhase& ph, float* const bufs[BUF_COUNT], cudaStream_t stream) {
  constexpr int STAGE = (NPASS == 3 ? 4 : 2) * 128 * 128;
  const size_t smem = 1024 + (size_t)S * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<NPASS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  gemm_tc_kernel<NPASS, S><<<ph.tc_total_tiles, 256, smem, stream>>>(ph.d_descs, (int)ph.descs.size(), ph.d_segs,
                                                                     bufs[0], bufs[1], bufs[2], bufs[3]);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_gemm_tc(const GemmPhase& ph, float* const bufs[BUF_COUNT], int npass, void* stream) {
  if (ph.tc_total_tiles == 0) return 0;
  if (npass == 3) return launch_tc_impl<3, 3>(ph, bufs, (cudaStream_t)stream);
  return launch_tc_impl<1, 3>(ph, bufs, (cudaStream_t)stream);
}

}  // namespace orth
