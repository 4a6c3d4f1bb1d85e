// Bjorck / Newton-Schulz on the 5th-generation tensor cores (a3),
// residual form (reading R16):
//     R  = I - X^T X          (Gram on the short side, R4)
//     X' = X + beta * X R      (tall; wide: X + beta * R X)
// X is the FP32 master.  Every phase's epilogue also writes the BF16 (hi, and
// for the 3-pass split lo = bf16(x - hi)) copies the NEXT phase consumes:
// the Gram writes R (symmetric, so its rows are both operands' rows), the
// update writes X' row-major and transposed.  The mainloop therefore only
// moves BF16 K-major rows: 16-byte cp.async into a SWIZZLE_128B ring, one
// thread issuing tcgen05.mma M=128 N=128 K=16 (x4 per 64-wide K block, x3 for
// the hi/lo split), FP32 accumulation in TMEM.  Ragged batch: one flat tile
// list over all matrices of all layers (descriptors from plan.cpp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"
#include "umma.cuh"

namespace orth {
namespace {

struct NsBufs {
  float* X[2];
  float* R;
  __nv_bfloat16 *xh[2], *xl[2], *th[2], *tl[2], *rh, *rl;
};

__device__ __forceinline__ const __nv_bfloat16* operand(const NsBufs& b, int kind, int par, bool lo) {
  if (kind == 0) return lo ? b.xl[par] : b.xh[par];
  if (kind == 1) return lo ? b.tl[par] : b.th[par];
  return lo ? b.rl : b.rh;
}

__device__ __forceinline__ int find_ns(const NsDesc* __restrict__ d, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void split(float x, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  l = __float2bfloat16_rn(x - __bfloat162float(h));
}

template <int NPASS, int S>
__global__ void __launch_bounds__(256, (NPASS == 1 ? 2 : 1))
    ns_tc_kernel(const NsDesc* __restrict__ descs, int ndesc, NsBufs bufs, int par, int write_lo) {
  constexpr bool SPLIT = NPASS == 3;
  constexpr int TILE = 128 * 128;
  constexpr int STAGE = (SPLIT ? 4 : 2) * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const NsDesc d = descs[find_ns(descs, ndesc, blockIdx.x)];
  const int local = blockIdx.x - d.tile_begin;
  const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;

  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, 128);
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
  constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);

  const __nv_bfloat16* Ah = operand(bufs, d.a_kind, par, false) + d.a_off;
  const __nv_bfloat16* Bh = operand(bufs, d.b_kind, par, false) + d.b_off;
  const __nv_bfloat16* Al = operand(bufs, d.a_kind, par, true) + d.a_off;
  const __nv_bfloat16* Bl = operand(bufs, d.b_kind, par, true) + d.b_off;
  const int nk = (d.K + 63) / 64;
  const int c = tid & 7;

  for (int kb = 0; kb < nk + S - 1; ++kb) {
    if (kb < nk) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const int kc = kb * 64 + c * 8;
      const bool kok = kc < d.K;
      const uint32_t sa = s0 + st * STAGE;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i;
        const uint32_t off = umma::sw128_off(r, c);
        const bool aok = kok && m0 + r < d.M, bok = kok && n0 + r < d.N;
        const int64_t ao = (int64_t)(m0 + r) * d.lda + kc, bo = (int64_t)(n0 + r) * d.ldb + kc;
        umma::cp_async16(sa + off, aok ? Ah + ao : Ah, aok);
        umma::cp_async16(sa + TILE + off, bok ? Bh + bo : Bh, bok);
        if (SPLIT) {
          umma::cp_async16(sa + 2 * TILE + off, aok ? Al + ao : Al, aok);
          umma::cp_async16(sa + 3 * TILE + off, bok ? Bl + bo : Bl, bok);
        }
      }
    }
    umma::cp_async_commit();
    const int j = kb - (S - 1);
    if (j >= 0) {
      umma::cp_async_wait<S - 1>();
      umma::fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        umma::tc_fence_after();
        const int st = j % S;
        const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, (j | q) != 0);
          if (SPLIT) {
            umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
            umma::mma_bf16(tmem, umma::sdesc_sw128(al + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, 1);
          }
        }
        umma::mma_commit(&empty_bar[st]);
      }
    }
  }
  if (tid == 0) umma::mma_commit(&done_bar);
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();

  // ---------------------------------------------------------------- epilogue
  // TMEM -> smem tile (fp32, row stride 129: conflict-free), then coalesced
  // passes over the tile: fp32 D (+ C), row-major bf16 copies, transposed copies.
  float* St = reinterpret_cast<float*>(smem);       // the operand ring is free now (done_bar passed)
  constexpr int LDS = 129;
  {
    const int q = warp & 3, half = warp >> 2;
    const int r = q * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < 64; cc += 32) {
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * 64 + cc), v);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) St[r * LDS + half * 64 + cc + jj] = v[jj];
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  const bool upd = d.epi == 1;
  const int ldb16 = upd ? d.ldx : d.ldr;   // padded row length of the row-major bf16 output
  __nv_bfloat16* oh = upd ? bufs.xh[par ^ 1] + d.bx_off : bufs.rh + d.br_off;
  __nv_bfloat16* ol = upd ? bufs.xl[par ^ 1] + d.bx_off : bufs.rl + d.br_off;
  float* F = upd ? bufs.X[par ^ 1] + d.f_off : bufs.R + d.f_off;
  const float* Cm = bufs.X[par] + d.f_off;
  // pass 1: rows (threads along columns); value outside the matrix = 0 (keeps bf16 padding zero).
  // C (the previous X, never written by this kernel) is loaded 32 elements at a time
  // through the read-only path so the loads overlap instead of serialising behind stores.
  constexpr int BATCH = 32;
#pragma unroll 1
  for (int e0 = tid; e0 < 128 * 128; e0 += 256 * BATCH) {
    float cv[BATCH];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int e = e0 + u * 256, r = e >> 7, cl = e & 127;
      const int i = m0 + r, j = n0 + cl;
      cv[u] = (upd && i < d.M && j < d.N) ? __ldg(Cm + (int64_t)i * d.ldf + j) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int e = e0 + u * 256, r = e >> 7, cl = e & 127;
      const int i = m0 + r, j = n0 + cl;
      float o = 0.f;
      if (i < d.M && j < d.N) {
        o = fmaf(d.alpha, St[r * LDS + cl], d.beta * cv[u]);
        if (i == j) o += d.diag;
        F[(int64_t)i * d.ldf + j] = o;
      }
      St[r * LDS + cl] = o;
      if (i < d.M && j < ldb16) {
        __nv_bfloat16 h, l;
        split(o, h, l);
        oh[(int64_t)i * ldb16 + j] = h;
        if (write_lo) ol[(int64_t)i * ldb16 + j] = l;
      }
    }
  }
  if (upd) {  // pass 2: transposed copy X'^T (threads along i)
    __syncthreads();
    __nv_bfloat16* th = bufs.th[par ^ 1] + d.bx_off;
    __nv_bfloat16* tl = bufs.tl[par ^ 1] + d.bx_off;
    for (int e = tid; e < 128 * 128; e += 256) {
      const int cl = e >> 7, r = e & 127;
      const int i = m0 + r, j = n0 + cl;
      if (j < d.N && i < d.ldxt) {
        __nv_bfloat16 h, l;
        split(St[r * LDS + cl], h, l);
        th[(int64_t)j * d.ldxt + i] = h;
        if (write_lo) tl[(int64_t)j * d.ldxt + i] = l;
      }
    }
  }
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 128);
}

// X0 = W / sigma and its BF16 copies (row-major and transposed)
__global__ void __launch_bounds__(256) scale_bf16_kernel(const PowerItem* __restrict__ items,
                                                         const float* __restrict__ W, const float* __restrict__ sigma,
                                                         float* __restrict__ X0, NsBufs b, int par, int write_lo) {
  __shared__ float T[32][65];
  const PowerItem it = items[blockIdx.x];
  const float inv = 1.f / sigma[it.mat];
  const int n = it.n, ldx = (n + 7) & ~7, ldxt = (it.m + 7) & ~7;
  __nv_bfloat16* xh = b.xh[par] + it.bx_off;
  __nv_bfloat16* xl = b.xl[par] + it.bx_off;
  __nv_bfloat16* th = b.th[par] + it.bx_off;
  __nv_bfloat16* tl = b.tl[par] + it.bx_off;
  for (int rt = it.r0; rt < it.r1; rt += 32)
    for (int ct = 0; ct < n; ct += 64) {   // 32 x 64 tile: row-major pass, then transposed pass via smem
      for (int e = threadIdx.x; e < 32 * 64; e += 256) {
        const int rr = e >> 6, cc = e & 63, r = rt + rr, c = ct + cc;
        float x = 0.f;
        if (r < it.r1 && c < n) {
          x = W[it.off + (int64_t)r * n + c] * inv;
          X0[it.off + (int64_t)r * n + c] = x;
          __nv_bfloat16 h, l;
          split(x, h, l);
          xh[(int64_t)r * ldx + c] = h;
          if (write_lo) xl[(int64_t)r * ldx + c] = l;
        }
        T[rr][cc] = x;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 64; e += 256) {
        const int cc = e >> 5, rr = e & 31, r = rt + rr, c = ct + cc;
        if (r < it.r1 && c < n) {
          __nv_bfloat16 h, l;
          split(T[rr][cc], h, l);
          th[(int64_t)c * ldxt + r] = h;
          if (write_lo) tl[(int64_t)c * ldxt + r] = l;
        }
      }
      __syncthreads();
    }
}

NsBufs make_bufs(Plan& p, float* const bufs[BUF_COUNT]) {
  NsBufs b;
  b.X[0] = bufs[BUF_X];
  b.X[1] = bufs[BUF_Y];
  b.R = bufs[BUF_G];
  auto bx = reinterpret_cast<__nv_bfloat16*>(p.d_bx);
  const int64_t nx = p.bx_numel > 64 ? p.bx_numel : 64;
  for (int k = 0; k < 2; ++k) {
    b.xh[k] = bx + (0 + k) * nx;
    b.xl[k] = bx + (2 + k) * nx;
    b.th[k] = bx + (4 + k) * nx;
    b.tl[k] = bx + (6 + k) * nx;
  }
  auto br = reinterpret_cast<__nv_bfloat16*>(p.d_br);
  b.rh = br;
  b.rl = br + (p.br_numel > 64 ? p.br_numel : 64);
  return b;
}

template <int NPASS, int S>
int launch_impl(const NsDesc* d, int nd, int tiles, NsBufs b, int par, int write_lo, cudaStream_t s) {
  constexpr int STAGE = (NPASS == 3 ? 4 : 2) * 128 * 128;
  const size_t smem = 1024 + (size_t)S * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ns_tc_kernel<NPASS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ns_tc_kernel<NPASS, S><<<tiles, 256, smem, s>>>(d, nd, b, par, write_lo);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_ns_tc(Plan& p, float* const bufs[BUF_COUNT], int par, bool gram, int npass, bool write_lo, void* stream) {
  const int tiles = gram ? p.ns_gram_tiles : p.ns_upd_tiles;
  if (tiles == 0) return 0;
  const NsDesc* d = gram ? p.d_ns_gram : p.d_ns_upd;
  const int nd = (int)(gram ? p.ns_gram.size() : p.ns_upd.size());
  NsBufs b = make_bufs(p, bufs);
  p.launches++;
  if (npass == 3) return launch_impl<3, 3>(d, nd, tiles, b, par, write_lo, (cudaStream_t)stream);
  return launch_impl<1, 3>(d, nd, tiles, b, par, write_lo, (cudaStream_t)stream);
}

int launch_scale_bf16(Plan& p, const float* W, float* X0, int par, bool write_lo, void* stream) {
  if (p.power_items.empty()) return 0;
  float* bufs[BUF_COUNT] = {X0, X0, nullptr, nullptr};
  NsBufs b = make_bufs(p, bufs);
  scale_bf16_kernel<<<(int)p.power_items.size(), 256, 0, (cudaStream_t)stream>>>(p.d_power_items, W, p.d_sigma, X0,
                                                                               b, par, write_lo);
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
