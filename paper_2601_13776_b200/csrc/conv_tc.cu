// a6 on the 5th-generation tensor cores: implicit-GEMM conv forward, BF16 in,
// FP32 accumulation in TMEM, BF16 out (P:122 forward "single call", P:332-338
// stride / dilation / groups; circular or zero padding, reading R11).
//
// GEMM view per group g: D[M = N*Ho*Wo pixels, N = co_g] = A[M, K] B[N, K]^T with
// K = (tap, channel), A[m, (a,b,c)] = x~[n, s*u + d*a - p_t, s*v + d*b - p_l, g*ci_g + c]
// and B = the BF16 GEMM-layout kernel (C_o, k, k, C_i/g), already K-major.
//
// CTA = 256 threads, tile 128 pixels x BN channels, K block = one tap x 64
// channels (one 128-byte swizzled row per pixel / output channel).  All
// threads gather A and B with 16-byte cp.async (zero-fill for padding / tails,
// index wrap for circular padding) into an S-stage ring; one thread issues 4
// tcgen05.mma (M=128, N=BN, K=16) per block and commits to the stage's
// mbarrier, which gates the reuse of that stage.  The accumulator lives in
// TMEM; the epilogue (8 warps: lane quarter x column half) adds the bias,
// rounds to BF16 (RNE) and stores NHWC rows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"
#include "umma.cuh"

namespace orth {
namespace {

struct TcConvArgs {
  int N, H, W, Ci, Co, ci_g, co_g, k, s, d, pt, pl, Ho, Wo, circ;
  int tiles_m;
};

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

template <int BN, int S>
__global__ void __launch_bounds__(256, 1)
    conv_fwd_tc(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                const float* __restrict__ bias, __nv_bfloat16* __restrict__ y, TcConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * A_BYTES;
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int rn[128], rh[128], rw[128];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.z;
  const int n0 = blockIdx.y * BN;
  const int64_t M = (int64_t)a.N * a.Ho * a.Wo;
  const int64_t m0 = (int64_t)blockIdx.x * 128;

  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, BN);
  if (tid == 32) {
    for (int i = 0; i < S; ++i) umma::mbar_init(&empty_bar[i], 1);
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  if (tid < 128) {
    const int64_t m = m0 + tid;
    if (m < M) {
      const int64_t hw = (int64_t)a.Ho * a.Wo;
      const int n = (int)(m / hw), r = (int)(m % hw);
      rn[tid] = n;
      rh[tid] = (r / a.Wo) * a.s - a.pt;
      rw[tid] = (r % a.Wo) * a.s - a.pl;
    } else {
      rn[tid] = -1; rh[tid] = 0; rw[tid] = 0;
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  const int kc = (a.ci_g + 63) / 64;
  const int kk2 = a.k * a.k;
  const int nk = kk2 * kc;
  constexpr uint32_t IDESC = umma::idesc_bf16(128, BN);
  const uint32_t sA0 = umma::smem_u32(sA), sB0 = umma::smem_u32(sB);

  for (int kb = 0; kb < nk + S - 1; ++kb) {
    if (kb < nk) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const int tap = kb / kc, c0 = (kb % kc) * 64;
      const int ta = tap / a.k, tb = tap % a.k;
      const int c = tid & 7;
      const bool cok = c0 + c * 8 < a.ci_g;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i;
        const int n = rn[r];
        int h = rh[r] + a.d * ta, ww = rw[r] + a.d * tb;
        bool ok = cok && n >= 0;
        if (a.circ) {
          h = wrapi(h, a.H);
          ww = wrapi(ww, a.W);
        } else {
          ok = ok && h >= 0 && h < a.H && ww >= 0 && ww < a.W;
        }
        const __nv_bfloat16* src =
            ok ? x + (((int64_t)n * a.H + h) * a.W + ww) * a.Ci + (int64_t)g * a.ci_g + c0 + c * 8 : x;
        umma::cp_async16(sA0 + st * A_BYTES + umma::sw128_off(r, c), src, ok);
      }
#pragma unroll
      for (int i = 0; i < BN / 32; ++i) {
        const int r = (tid >> 3) + 32 * i;
        const int o = n0 + r;
        const bool ok = cok && o < a.co_g;
        const __nv_bfloat16* src = ok ? w + (((int64_t)g * a.co_g + o) * kk2 + tap) * a.ci_g + c0 + c * 8 : w;
        umma::cp_async16(sB0 + st * B_BYTES + umma::sw128_off(r, c), src, ok);
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
        const uint32_t a_addr = sA0 + st * A_BYTES, b_addr = sB0 + st * B_BYTES;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          umma::mma_bf16(tmem, umma::sdesc_sw128(a_addr + 32 * q), umma::sdesc_sw128(b_addr + 32 * q), IDESC,
                         (j | q) != 0);
        umma::mma_commit(&empty_bar[st]);
      }
    }
  }
  if (tid == 0) umma::mma_commit(&done_bar);
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();

  // epilogue: warp -> (lane quarter q, column half)
  const int q = warp & 3, half = warp >> 2;
  const int r = q * 32 + lane;
  const int64_t m = m0 + r;
#pragma unroll
  for (int cc = 0; cc < BN / 2; cc += 32) {
    const int col = half * (BN / 2) + cc;
    float v[32];
    umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
    if (m < M) {
      const int o = g * a.co_g + n0 + col;
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float v0 = v[2 * i], v1 = v[2 * i + 1];
        if (bias) { v0 += bias[o + 2 * i]; v1 += bias[o + 2 * i + 1]; }
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
        pk[i] = *reinterpret_cast<uint32_t*>(&b2);
      }
      uint4* dst = reinterpret_cast<uint4*>(y + m * a.Co + o);
#pragma unroll
      for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, BN);
}

template <int BN, int S>
int launch_tc(const LayerInfo& L, const __nv_bfloat16* x, const __nv_bfloat16* w, const float* bias,
              __nv_bfloat16* y, TcConvArgs a, cudaStream_t stream) {
  const size_t smem = 1024 + (size_t)S * (128 * 128 + BN * 128);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_fwd_tc<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)a.tiles_m, (unsigned)(L.co / BN), (unsigned)L.g);
  conv_fwd_tc<BN, S><<<grid, 256, smem, stream>>>(x, w, bias, y, a);
  return (int)cudaGetLastError();
}

}  // namespace

bool conv_fwd_tc_eligible(const LayerInfo& L) {
  return L.co % 64 == 0 && L.ci % 8 == 0 && L.ci_f % 8 == 0 && L.co_f % 8 == 0;
}

int launch_conv_fwd_tc(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                       int H, int W, int Ho, int Wo, void* stream) {
  TcConvArgs a;
  a.N = N; a.H = H; a.W = W; a.Ci = L.ci_f; a.Co = L.co_f; a.ci_g = L.ci; a.co_g = L.co;
  a.k = L.k; a.s = L.s; a.d = L.d; a.pt = L.pt; a.pl = L.pl; a.Ho = Ho; a.Wo = Wo;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  const int64_t M = (int64_t)N * Ho * Wo;
  a.tiles_m = (int)((M + 127) / 128);
  auto xs = (const __nv_bfloat16*)x;
  auto ws = (const __nv_bfloat16*)kernel;
  auto ys = (__nv_bfloat16*)y;
  cudaStream_t s = (cudaStream_t)stream;
  if (L.co % 256 == 0) return launch_tc<256, 4>(L, xs, ws, bias, ys, a, s);
  if (L.co % 128 == 0) return launch_tc<128, 6>(L, xs, ws, bias, ys, a, s);
  return launch_tc<64, 8>(L, xs, ws, bias, ys, a, s);
}

}  // namespace orth
