// a6/a7 SIMT implicit-GEMM convolution (first CUDA path; FP32 accumulation).
//
// Forward:
//   y[n,u,v,o] = sum_{a,b,c} K[o,c,a,b] x~[n, s u + d a - p_t, s v + d b - p_l, g*ci_g + c]
// Adjoint / transposed (R13/R14), gather form:
//   x[n,h,w,i] = sum_{a,b,o} K[o,i,a,b] y[n,u,v,o] over the (u,v) with
//   s u + d a - p_t == h (mod H for circular, exactly for zero padding).
// Activations are NHWC; bf16 I/O reads the BF16 GEMM-layout kernel
// (C_o, k, k, C_i/g), f32 I/O the FP32 PyTorch-layout kernel (C_o, C_i/g, k, k).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "orth_internal.h"

namespace orth {
namespace {

struct ConvArgs {
  int N, H, W, Ci, Co, ci_g, co_g, k, s, d, pt, pl, Ho, Wo, circ;
};

template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T> __device__ __forceinline__ void st(T* p, float v);
template <> __device__ __forceinline__ void st<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ int wrap(int x, int n) { x %= n; return x < 0 ? x + n : x; }

constexpr int BM = 64, BN = 64, BK = 16;

// T: activation type; W: kernel element type (bf16 -> GEMM layout, float -> canonical)
template <typename T, typename Wt>
__global__ void __launch_bounds__(256) conv_fwd_simt(const T* __restrict__ x, const Wt* __restrict__ wt,
                                                     const float* __restrict__ bias, T* __restrict__ y, ConvArgs a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ int pn[BM], ph[BM], pw[BM];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int g = blockIdx.z;
  const int64_t M = (int64_t)a.N * a.Ho * a.Wo;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  if (tid < BM) {
    const int64_t m = m0 + tid;
    if (m < M) {
      const int64_t hw = (int64_t)a.Ho * a.Wo;
      const int n = (int)(m / hw), r = (int)(m % hw);
      pn[tid] = n; ph[tid] = (r / a.Wo) * a.s - a.pt; pw[tid] = (r % a.Wo) * a.s - a.pl;
    } else {
      pn[tid] = -1; ph[tid] = 0; pw[tid] = 0;
    }
  }
  __syncthreads();
  float acc[4][4] = {};
  const int kk2 = a.k * a.k;
  for (int tap = 0; tap < kk2; ++tap) {
    const int ta = tap / a.k, tb = tap % a.k;
    for (int c0 = 0; c0 < a.ci_g; c0 += BK) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256, kk = e % BK, i = e / BK;
        float v = 0.f;
        const int n = pn[i];
        if (n >= 0 && c0 + kk < a.ci_g) {
          int h = ph[i] + a.d * ta, w = pw[i] + a.d * tb;
          bool ok = true;
          if (a.circ) { h = wrap(h, a.H); w = wrap(w, a.W); }
          else ok = h >= 0 && h < a.H && w >= 0 && w < a.W;
          if (ok) v = ld(x + (((int64_t)n * a.H + h) * a.W + w) * a.Ci + g * a.ci_g + c0 + kk);
        }
        As[kk][i] = v;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256, kk = e % BK, j = e / BK;
        float v = 0.f;
        const int oc = n0 + j, c = c0 + kk;
        if (oc < a.co_g && c < a.ci_g) {
          const int64_t o = (int64_t)g * a.co_g + oc;
          if (sizeof(Wt) == 2) v = ld(wt + (o * kk2 + tap) * a.ci_g + c);
          else v = ld(wt + (o * a.ci_g + c) * kk2 + tap);
        }
        Bs[kk][j] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float aa[4] = {av.x, av.y, av.z, av.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], bb[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int oc = n0 + tx * 4 + j;
      if (oc >= a.co_g) continue;
      const int o = g * a.co_g + oc;
      float v = acc[i][j];
      if (bias) v += bias[o];
      st(y + m * a.Co + o, v);
    }
  }
}

// adjoint: output pixels over the big grid, reduction over (tap, o)
template <typename T, typename Wt>
__global__ void __launch_bounds__(256) conv_bwd_simt(const T* __restrict__ yv, const Wt* __restrict__ wt,
                                                     const float* __restrict__ bias, T* __restrict__ x, ConvArgs a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ int pn[BM], ph[BM], pw[BM];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int g = blockIdx.z;
  const int64_t M = (int64_t)a.N * a.H * a.W;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  if (tid < BM) {
    const int64_t m = m0 + tid;
    if (m < M) {
      const int64_t hw = (int64_t)a.H * a.W;
      const int n = (int)(m / hw), r = (int)(m % hw);
      pn[tid] = n; ph[tid] = r / a.W + a.pt; pw[tid] = r % a.W + a.pl;
    } else {
      pn[tid] = -1; ph[tid] = 0; pw[tid] = 0;
    }
  }
  __syncthreads();
  float acc[4][4] = {};
  const int kk2 = a.k * a.k;
  for (int tap = 0; tap < kk2; ++tap) {
    const int ta = tap / a.k, tb = tap % a.k;
    for (int c0 = 0; c0 < a.co_g; c0 += BK) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256, kk = e % BK, i = e / BK;
        float v = 0.f;
        const int n = pn[i];
        if (n >= 0 && c0 + kk < a.co_g) {
          int th = ph[i] - a.d * ta, tw = pw[i] - a.d * tb;
          if (a.circ) { th = wrap(th, a.H); tw = wrap(tw, a.W); }
          bool ok = th >= 0 && tw >= 0 && (th % a.s) == 0 && (tw % a.s) == 0;
          const int u = th / a.s, vv = tw / a.s;
          ok = ok && u < a.Ho && vv < a.Wo;
          if (ok) v = ld(yv + (((int64_t)n * a.Ho + u) * a.Wo + vv) * a.Co + g * a.co_g + c0 + kk);
        }
        As[kk][i] = v;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256, j = e % BN, kk = e / BN;
        float v = 0.f;
        const int ic = n0 + j, oc = c0 + kk;
        if (ic < a.ci_g && oc < a.co_g) {
          const int64_t o = (int64_t)g * a.co_g + oc;
          if (sizeof(Wt) == 2) v = ld(wt + (o * kk2 + tap) * a.ci_g + ic);
          else v = ld(wt + (o * a.ci_g + ic) * kk2 + tap);
        }
        Bs[kk][j] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float aa[4] = {av.x, av.y, av.z, av.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], bb[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ic = n0 + tx * 4 + j;
      if (ic >= a.ci_g) continue;
      const int c = g * a.ci_g + ic;
      float v = acc[i][j];
      if (bias) v += bias[c];
      st(x + m * a.Ci + c, v);
    }
  }
}

// Small reduction (ci_g * k^2 <= 64, e.g. the RGB stem): im2col of 128 pixels
// into shared memory, the whole kernel slab in shared memory, FP32 FFMA; each
// thread owns one pixel and writes 16-byte runs of 8 output channels.
__global__ void __launch_bounds__(256) conv_fwd_smallk(const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ wt,
                                                       const float* __restrict__ bias, __nv_bfloat16* __restrict__ y,
                                                       ConvArgs a) {
  extern __shared__ float sm[];
  const int KT = a.ci_g * a.k * a.k, ld = KT | 1;   // odd row stride: conflict-free per-thread rows
  float* patch = sm;                   // [256][KT | 1]: one im2col row per thread
  float* ws = sm + 256 * ld;           // [KT][co_g] (16-byte aligned: 256 * ld * 4 is)
  const int g = blockIdx.z, tid = threadIdx.x;
  const int M = a.N * a.Ho * a.Wo;
  for (int e = tid; e < KT * a.co_g; e += 256) {     // GEMM layout (co, k, k, ci_g): row o is K-contiguous
    const int o = e / KT, kk = e - o * KT;
    ws[kk * a.co_g + o] = __bfloat162float(wt[((int64_t)g * a.co_g + o) * KT + kk]);
  }
  const int m = blockIdx.x * 256 + tid;
  float* prow = patch + tid * ld;
  if (m < M) {   // this thread's im2col row, taps in (a, b) order, channels innermost
    const int hw = a.Ho * a.Wo, n = m / hw, r = m - n * hw, u = r / a.Wo, v = r - u * a.Wo;
    const __nv_bfloat16* xn = x + (int64_t)n * a.H * a.W * a.Ci + g * a.ci_g;
    int kk = 0;
    for (int ta = 0; ta < a.k; ++ta) {
      int h = u * a.s - a.pt + a.d * ta;
      bool hok = true;
      if (a.circ) h = wrap(h, a.H); else hok = h >= 0 && h < a.H;
      for (int tb = 0; tb < a.k; ++tb) {
        int w = v * a.s - a.pl + a.d * tb;
        bool ok = hok;
        if (a.circ) w = wrap(w, a.W); else ok = ok && w >= 0 && w < a.W;
        const __nv_bfloat16* px = xn + ((int64_t)h * a.W + w) * a.Ci;
        for (int c = 0; c < a.ci_g; ++c, ++kk) prow[kk] = ok ? __bfloat162float(px[c]) : 0.f;
      }
    }
  }
  __syncthreads();
  if (m >= M) return;
  const float4* ws4 = reinterpret_cast<const float4*>(ws);
  const int co4 = a.co_g / 4;
  for (int c0 = 0; c0 < a.co_g; c0 += 32) {          // 32 output channels per pass (co_g % 16 == 0)
    const int nc = a.co_g - c0 < 32 ? a.co_g - c0 : 32;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    for (int kk = 0; kk < KT; ++kk) {
      const float av = prow[kk];
      const float4* wr = ws4 + kk * co4 + c0 / 4;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (4 * j < nc) {
          const float4 w4 = wr[j];                      // warp-uniform address: broadcast
          acc[4 * j] = fmaf(av, w4.x, acc[4 * j]);
          acc[4 * j + 1] = fmaf(av, w4.y, acc[4 * j + 1]);
          acc[4 * j + 2] = fmaf(av, w4.z, acc[4 * j + 2]);
          acc[4 * j + 3] = fmaf(av, w4.w, acc[4 * j + 3]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (8 * q >= nc) break;
      uint32_t pk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v0 = acc[8 * q + 2 * j], v1 = acc[8 * q + 2 * j + 1];
        if (bias) {
          v0 += bias[g * a.co_g + c0 + 8 * q + 2 * j];
          v1 += bias[g * a.co_g + c0 + 8 * q + 2 * j + 1];
        }
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
        pk[j] = *reinterpret_cast<uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(y + (int64_t)m * a.Co + g * a.co_g + c0 + 8 * q) =
          make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
}

ConvArgs make_args(const LayerInfo& L, int N, int H, int W, int Ho, int Wo) {
  ConvArgs a;
  a.N = N; a.H = H; a.W = W; a.Ci = L.ci_f; a.Co = L.co_f; a.ci_g = L.ci; a.co_g = L.co;
  a.k = L.k; a.s = L.s; a.d = L.d; a.pt = L.pt; a.pl = L.pl; a.Ho = Ho; a.Wo = Wo;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  return a;
}

}  // namespace

int launch_conv_fwd(const LayerInfo& L, const void* kernel, void* scratch, const float* bias, const void* x, void* y,
                    int N, int H, int W, int Ho, int Wo, int io, void* stream) {
  if (io == ORTH_BF16 && scratch && conv_fwd_tc_eligible(L) && !getenv("ORTH_FORCE_SIMT"))
    return launch_conv_fwd_tc(L, kernel, scratch, bias, x, y, N, H, W, Ho, Wo, stream);
  const ConvArgs a = make_args(L, N, H, W, Ho, Wo);
  const int64_t M = (int64_t)N * Ho * Wo;
  const int KT = L.ci * L.k * L.k;
  if (io == ORTH_BF16 && !getenv("ORTH_FORCE_SIMT") && !getenv("ORTH_NO_STEM_TC")) {   // tensor-core stem
    const int e = launch_conv_fwd_stem(L, kernel, bias, x, y, N, H, W, Ho, Wo, stream);
    if (e >= 0) return e;
  }
  if (io == ORTH_BF16 && KT <= 64 && L.co % 16 == 0 && L.co_f % 8 == 0 && !getenv("ORTH_FORCE_SIMT")) {
    const size_t smem = (size_t)(256 * (KT | 1) + KT * L.co) * sizeof(float);
    if (smem <= 200 * 1024) {
      static size_t attr = 0;
      if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(conv_fwd_smallk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
      }
      dim3 g2((unsigned)((M + 255) / 256), 1, (unsigned)L.g);
      g_conv_variant = ORTH_CV_SMALLK;
      conv_fwd_smallk<<<g2, 256, smem, (cudaStream_t)stream>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)kernel,
                                                               bias, (__nv_bfloat16*)y, a);
      return (int)cudaGetLastError();
    }
  }
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((L.co + BN - 1) / BN), (unsigned)L.g);
  cudaStream_t s = (cudaStream_t)stream;
  g_conv_variant = ORTH_CV_SIMT;
  if (io == ORTH_BF16)
    conv_fwd_simt<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)kernel, bias, (__nv_bfloat16*)y, a);
  else
    conv_fwd_simt<float, float><<<grid, 256, 0, s>>>((const float*)x, (const float*)kernel, bias, (float*)y, a);
  return (int)cudaGetLastError();
}

// Adjoint of a patch conv (k = s, d = 1, H = s Ho, W = s Wo, circular or unpadded: the RKO stem): every x
// pixel (s i - p_t + a, s j - p_l + b) (mod H, W) receives exactly tap (a, b) of y[i, j] -- x[n, ., ., c] =
// sum_o K[o, c, a, b] y[n, i, j, o] (+ bias[c]).  One warp per (y pixel, group): y's co_g channels staged in
// shared memory with the group's weights, lanes over the k^2 ci_g outputs of the patch.  (The general SIMT adjoint tiles 64 output
// channels and visits all k^2 taps per pixel: for the 3-channel stem that was 111 ms at batch 256.)
template <typename T, typename Wt>
__global__ void __launch_bounds__(256) conv_bwd_patch(const T* __restrict__ yv, const Wt* __restrict__ wt,
                                                      const float* __restrict__ bias, T* __restrict__ x, ConvArgs a) {
  // shared: the group's weights as [o][tap ci_g + ic] FP32, then [8 warps][co_g] staged y channels;
  // a block covers 8 x PPW y pixels (each warp PPW of them), so the weights are read once per 64 pixels
  extern __shared__ float sm[];
  constexpr int PPW = 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = blockIdx.y;
  const int kk2 = a.k * a.k, nout = kk2 * a.ci_g;
  float* ws = sm;
  float* yw = sm + (size_t)a.co_g * nout + warp * a.co_g;
  for (int idx = threadIdx.x; idx < a.co_g * nout; idx += blockDim.x) {
    const int o = idx / nout, e = idx - o * nout, tap = e / a.ci_g, ic = e - tap * a.ci_g;
    const int64_t oo = (int64_t)g * a.co_g + o;
    ws[idx] = sizeof(Wt) == 2 ? ld(wt + (oo * kk2 + tap) * a.ci_g + ic) : ld(wt + (oo * a.ci_g + ic) * kk2 + tap);
  }
  __syncthreads();
  const int64_t M = (int64_t)a.N * a.Ho * a.Wo;
  for (int p = 0; p < PPW; ++p) {
    const int64_t m = ((int64_t)blockIdx.x * 8 + warp) * PPW + p;
    if (m >= M) break;
    __syncwarp();
    for (int o = lane; o < a.co_g; o += 32) yw[o] = ld(yv + m * a.Co + (int64_t)g * a.co_g + o);
    __syncwarp();
    const int n = (int)(m / ((int64_t)a.Ho * a.Wo)), r = (int)(m - (int64_t)n * a.Ho * a.Wo);
    const int i = r / a.Wo, j = r - i * a.Wo;
    for (int e = lane; e < nout; e += 32) {
      const int tap = e / a.ci_g, ic = e - tap * a.ci_g;
      const int ta = tap / a.k, tb = tap - ta * a.k;
      float acc = 0.f;
      for (int o = 0; o < a.co_g; ++o) acc = fmaf(yw[o], ws[o * nout + e], acc);
      const int c = g * a.ci_g + ic;
      if (bias) acc += bias[c];
      int h = a.s * i - a.pt + ta, w = a.s * j - a.pl + tb;   // circular: (i, a) -> h is a bijection
      if (a.circ) { h = wrap(h, a.H); w = wrap(w, a.W); }
      st(x + (((int64_t)n * a.H + h) * a.W + w) * a.Ci + c, acc);
    }
  }
}

int launch_conv_bwd(const LayerInfo& L, const void* kernel, void* wt_scratch, const float* bias, const void* y,
                    void* x, int N, int H, int W, int Ho, int Wo, int io, void* stream) {
  if (io == ORTH_BF16 && wt_scratch && conv_bwd_tc_eligible(L) && !getenv("ORTH_FORCE_SIMT"))
    return launch_conv_bwd_tc(L, kernel, wt_scratch, bias, y, x, N, H, W, Ho, Wo, stream);
  const ConvArgs a = make_args(L, N, H, W, Ho, Wo);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t patch_sm = ((size_t)L.co * L.k * L.k * L.ci + 8 * (size_t)L.co) * sizeof(float);
  if (L.k == L.s && L.d == 1 && (a.circ || (a.pt == 0 && a.pl == 0)) && H == L.s * Ho && W == L.s * Wo &&
      patch_sm <= 48 * 1024 && !getenv("ORTH_CONV_NO_PATCH_BWD")) {
    g_conv_variant = ORTH_CV_SIMT;
    const int64_t My = (int64_t)N * Ho * Wo;
    if (My == 0) return 0;
    dim3 pg((unsigned)((My + 63) / 64), (unsigned)L.g);
    const size_t sm = patch_sm;
    if (io == ORTH_BF16)
      conv_bwd_patch<__nv_bfloat16, __nv_bfloat16><<<pg, 256, sm, s>>>(
          (const __nv_bfloat16*)y, (const __nv_bfloat16*)kernel, bias, (__nv_bfloat16*)x, a);
    else
      conv_bwd_patch<float, float><<<pg, 256, sm, s>>>((const float*)y, (const float*)kernel, bias, (float*)x, a);
    return (int)cudaGetLastError();
  }
  const int64_t M = (int64_t)N * H * W;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((L.ci + BN - 1) / BN), (unsigned)L.g);
  g_conv_variant = ORTH_CV_SIMT;
  if (io == ORTH_BF16)
    conv_bwd_simt<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(
        (const __nv_bfloat16*)y, (const __nv_bfloat16*)kernel, bias, (__nv_bfloat16*)x, a);
  else
    conv_bwd_simt<float, float><<<grid, 256, 0, s>>>((const float*)y, (const float*)kernel, bias, (float*)x, a);
  return (int)cudaGetLastError();
}

}  // namespace orth
