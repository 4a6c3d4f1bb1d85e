// a6 for layers with a tiny reduction (ci_g * k^2 <= 64, e.g. the RGB stem of
// cfg2 / the 4x4 s4 RKO stem of cfg3) on the tensor cores.
//
// The whole reduction fits one 64-wide K block, so a tile is a single
// 128-pixel im2col block: each of 128 threads writes its pixel's K values
// (taps in (a, b) order, channels innermost, zero-padded to a multiple of 16)
// as one SWIZZLE_128B K-major row; one thread issues ceil(K/16)
// tcgen05.mma M=128 N=co K=16 against the resident weight tile (co rows x K,
// loaded once per CTA); each thread then drains its own TMEM row (bias, RNE
// to BF16) into its pixel's NHWC output row.  Several CTAs per SM overlap the
// gather of one tile with the MMA / epilogue of another.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "orth_internal.h"
#include "pdl.h"
#include "tma_host.h"
#include "umma.cuh"

namespace orth {
namespace {

struct StemArgs {
  int N, H, W, Ci, Co, k, s, d, pt, pl, Ho, Wo, circ;
  int KT, nq;   // reduction length, K=16 steps
  int tiles;
};

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

template <int CO, int CI, int KS>
__global__ void __launch_bounds__(128) conv_stem_tc(const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ wt,
                                                    const float* __restrict__ bias, __nv_bfloat16* __restrict__ y,
                                                    const __grid_constant__ StemArgs a,
                                                    const __grid_constant__ CUtensorMap tmY) {
  constexpr int TM = CO < 32 ? 32 : CO;   // TMEM columns (power of two >= 32)
  __shared__ __align__(1024) uint8_t As[128 * 128];
  __shared__ __align__(1024) uint8_t Bs[CO * 128];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  umma::griddep_launch_dependents();
  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, TM);
  if (tid == 0) {
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::griddep_wait();   // PDL: weights and x of the previous kernels are complete
  // resident weights: row o = W[o][0..KT) (GEMM layout), zero-padded to 64
  for (int e = tid; e < CO * 8; e += 128) {
    const int o = e >> 3, c = e & 7;
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k0 = c * 8 + 2 * j;
      const float lo = k0 < a.KT ? __bfloat162float(wt[(int64_t)o * a.KT + k0]) : 0.f;
      const float hi = k0 + 1 < a.KT ? __bfloat162float(wt[(int64_t)o * a.KT + k0 + 1]) : 0.f;
      __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
      v[j] = *reinterpret_cast<uint32_t*>(&b2);
    }
    *reinterpret_cast<uint4*>(Bs + umma::sw128_off(o, c)) = make_uint4(v[0], v[1], v[2], v[3]);
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t sa = umma::smem_u32(As), sb = umma::smem_u32(Bs);
  constexpr uint32_t IDESC = umma::idesc_bf16(128, CO);
  const int M = a.N * a.Ho * a.Wo;
  int phase = 0;
  for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, phase ^= 1) {
    // ---- im2col row of this thread's pixel (As is free: tid 0 waited for the last store's reads
    // before the trailing __syncthreads of the previous tile)
    const int m = tile * 128 + tid;
    {
      constexpr int KT = CI * KS * KS;
      static_assert(KT <= 64, "one 64-wide K block");
      float vals[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) vals[k] = 0.f;
      if (m < M) {
        const int hw = a.Ho * a.Wo, n = m / hw, r = m - n * hw, u = r / a.Wo, v = r - u * a.Wo;
        const __nv_bfloat16* xn = x + (int64_t)n * a.H * a.W * a.Ci;
#pragma unroll
        for (int ta = 0; ta < KS; ++ta) {
          int h = u * a.s - a.pt + a.d * ta;
          bool hok = true;
          if (a.circ) h = wrapi(h, a.H); else hok = h >= 0 && h < a.H;
#pragma unroll
          for (int tb = 0; tb < KS; ++tb) {
            int w = v * a.s - a.pl + a.d * tb;
            bool ok = hok;
            if (a.circ) w = wrapi(w, a.W); else ok = ok && w >= 0 && w < a.W;
            const __nv_bfloat16* px = xn + ((int64_t)h * a.W + w) * a.Ci;
#pragma unroll
            for (int c = 0; c < CI; ++c) vals[(ta * KS + tb) * CI + c] = ok ? __bfloat162float(px[c]) : 0.f;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(vals[c * 8 + 2 * j], vals[c * 8 + 2 * j + 1]);
          v[j] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(As + umma::sw128_off(tid, c)) = make_uint4(v[0], v[1], v[2], v[3]);
      }
    }
    umma::fence_proxy_async_smem();   // generic-proxy smem writes -> tcgen05.mma reads
    umma::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      umma::tc_fence_after();
      for (int q = 0; q < a.nq; ++q)
        umma::mma_bf16(tmem, umma::sdesc_sw128(sa + 32 * q), umma::sdesc_sw128(sb + 32 * q), IDESC, q > 0);
      umma::mma_commit(&done_bar);
    }
    umma::mbar_wait(&done_bar, phase);
    umma::tc_fence_after();
    // ---- epilogue: this thread's TMEM row -> bias -> BF16 into a SWIZZLE_128B staging tile (the
    // A tile, consumed by now) -> one TMA tensor store per 64 channels (the tile's 128 pixels are
    // consecutive NHWC rows: a dense box)
    umma::bulk_wait_read0();   // the previous tile's store has finished reading the staging tile
#pragma unroll
    for (int c0 = 0; c0 < CO; c0 += 64) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c0 + 32 * h), v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float v0 = v[8 * i + 2 * j], v1 = v[8 * i + 2 * j + 1];
            if (bias) { v0 += bias[c0 + 32 * h + 8 * i + 2 * j]; v1 += bias[c0 + 32 * h + 8 * i + 2 * j + 1]; }
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
            pk[j] = *reinterpret_cast<uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(As + umma::sw128_off(tid, h * 4 + i)) =
              make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      umma::fence_proxy_async_smem();   // staging writes -> TMA (async proxy) reads
      __syncthreads();
      if (tid == 0) {
        umma::tma_store_2d(&tmY, umma::smem_u32(As), c0, tile * 128);   // rows past M are clipped by TMA
        umma::bulk_commit();
        if (c0 + 64 < CO) umma::bulk_wait_read0();   // staging reused by the next 64 channels
      }
      if (c0 + 64 < CO) __syncthreads();
    }
    if (tid == 0) umma::bulk_wait_read0();
    umma::tc_fence_before();
    __syncthreads();   // A tile (staging) and TMEM free for the next tile
  }
  if (tid == 0) umma::bulk_wait0();   // all stores complete before exit
  umma::tc_fence_after();
  if (warp == 0) umma::tmem_dealloc(tmem, TM);
}

template <int CO, int CI, int KS>
int launch_stem(const __nv_bfloat16* x, const __nv_bfloat16* w, const float* bias, __nv_bfloat16* y,
                const StemArgs& a, cudaStream_t s) {
  g_conv_variant = ORTH_CV_STEM;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // CTAs per SM: each tile is a serial gather -> MMA -> store chain, so residency hides the latency
  // (TMEM: CO <= 128 columns per CTA, up to 4 per SM at CO = 128; smem 16 + CO/8 KB)
  static const int per_sm = std::getenv("ORTH_STEM_CTAS_PER_SM") ? std::atoi(std::getenv("ORTH_STEM_CTAS_PER_SM"))
                                                                  : (CO <= 64 ? 6 : 4);
  const int grid = std::min(a.tiles, sms * per_sm);
  // output viewed as (Co channels, N*Ho*Wo pixels), box 64 x 128, SWIZZLE_128B
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  auto enc = tensor_map_encoder();
  const cuuint64_t dims[2] = {(cuuint64_t)a.Co, (cuuint64_t)a.N * a.Ho * a.Wo};
  const cuuint64_t strides[1] = {(cuuint64_t)a.Co * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  if (!enc || enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return (int)cudaErrorInvalidValue;
  launch_pdl(conv_stem_tc<CO, CI, KS>, dim3(grid), dim3(128), 0, s, x, w, bias, y, a, tm);
  return (int)cudaGetLastError();
}

}  // namespace

// -1: not applicable (caller falls back)
int launch_conv_fwd_stem(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                         int H, int W, int Ho, int Wo, void* stream) {
  const int KT = L.ci * L.k * L.k;
  // instantiated for the RGB stems of the paper-shaped workloads: 3 channels, 3x3 or 4x4 taps
  if (L.g != 1 || KT > 64 || L.ci != 3 || (L.k != 3 && L.k != 4) || (L.co != 64 && L.co != 128) ||
      ((uintptr_t)y & 15))
    return -1;
  StemArgs a{};
  a.N = N; a.H = H; a.W = W; a.Ci = L.ci_f; a.Co = L.co_f; a.k = L.k; a.s = L.s; a.d = L.d;
  a.pt = L.pt; a.pl = L.pl; a.Ho = Ho; a.Wo = Wo;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  a.KT = KT;
  a.nq = (KT + 15) / 16;
  a.tiles = (int)(((int64_t)N * Ho * Wo + 127) / 128);
  if (a.tiles == 0) return 0;
  const auto* xi = static_cast<const __nv_bfloat16*>(x);
  const auto* wi = static_cast<const __nv_bfloat16*>(kernel);
  auto* yo = static_cast<__nv_bfloat16*>(y);
  cudaStream_t s = (cudaStream_t)stream;
  if (L.k == 3) {
    switch (L.co) {
      case 64: return launch_stem<64, 3, 3>(xi, wi, bias, yo, a, s);
      default: return launch_stem<128, 3, 3>(xi, wi, bias, yo, a, s);
    }
  }
  switch (L.co) {
    case 64: return launch_stem<64, 3, 4>(xi, wi, bias, yo, a, s);
    default: return launch_stem<128, 3, 4>(xi, wi, bias, yo, a, s);
  }
}

}  // namespace orth
