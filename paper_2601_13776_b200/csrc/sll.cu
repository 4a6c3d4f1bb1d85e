// f4: SLL x AOC fused down-sampling block (P:381-399,
// App. B.3; readings R28-R30).
//
// Construction (orth_compose_kernel):
//   SLL unit  W (c_out x c_in x k x k, role K):   V[Delta] = sum_t W_t^T W_{t+Delta}  (GemmPhase sll_v,
//             reading W in place), then sll_scale_kernel: d_i = sum_j sum_Delta |V[Delta][i][j]|,
//             s_i = d_i^{-1/2} (1 if d_i = 0), K_t[o][i] = W[o, i, t] s_i (tap-major; AOL, R28).
//   block     C = K (*) K_pre, A = K_post (*) K_pre, B = K_post (*) K^T   (GemmPhase blk_mm on the emitted
//             FP32 kernels), then blk_merge_kernel: M = [A | -2 B] with A, B embedded at their pad offsets
//             in a common window (R29).  A second emit writes C and M into the block's kernel region.
// Forward (orth_conv_forward on the block): h = C * x + bias (conv kernels), z = [x | relu(h)]
// (relu_concat_kernel, one pass), y = M *_s z (conv kernels) -- P:394-396 with the merged kernels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

__global__ void __launch_bounds__(256) sll_scale_kernel(const SllItem* __restrict__ items, const float* __restrict__ ortho,
                                                        float* __restrict__ Wk) {
  const SllItem it = items[blockIdx.x];
  const int ci = it.ci, co = it.co, kk = it.k * it.k;
  const int k2 = 2 * it.k - 1;
  const int64_t taps = (int64_t)k2 * k2, c2 = (int64_t)ci * ci;
  const float* V = Wk + it.v_off;
  float* sc = Wk + it.s_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < ci; i += 8) {   // a warp per row of V: d_i
    float di = 0.f;
    for (int64_t p = 0; p < taps; ++p) {
      const float* row = V + p * c2 + (int64_t)i * ci;
      for (int j = lane; j < ci; j += 32) di += fabsf(row[j]);
    }
    for (int o = 16; o > 0; o >>= 1) di += __shfl_xor_sync(0xffffffffu, di, o);
    if (lane == 0) sc[i] = di > 0.f ? rsqrtf(di) : 1.f;
  }
  __syncthreads();
  const float* W = ortho + it.src_off;
  float* K = Wk + it.kt_off;
  const int64_t total = (int64_t)kk * co * ci;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {   // tap-major K_t[o][i] = W[o, i, t] s_i
    const int64_t t = e / ((int64_t)co * ci), r = e - t * co * ci;
    const int64_t o = r / ci, i = r - o * ci;
    K[e] = W[(o * ci + i) * kk + t] * sc[i];
  }
}

__global__ void __launch_bounds__(256) blk_merge_kernel(const BlkItem* __restrict__ items, float* __restrict__ Wk) {
  const BlkItem it = items[blockIdx.y];
  const int cz = it.c + it.cs;
  const int64_t plane = (int64_t)it.co * cz;
  const int64_t total = (int64_t)it.kM * it.kM * plane;
  float* M = Wk + it.m_off;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / plane, r = e - p * plane;
    const int p1 = (int)(p / it.kM), p2 = (int)(p - (int64_t)p1 * it.kM);
    const int o = (int)(r / cz), j = (int)(r - (int64_t)o * cz);
    float v = 0.f;
    if (j < it.c) {
      const int q1 = p1 - it.oa, q2 = p2 - it.oa;
      if (q1 >= 0 && q2 >= 0 && q1 < it.kA && q2 < it.kA)
        v = Wk[it.a_off + ((int64_t)(q1 * it.kA + q2) * it.co + o) * it.c + j];
    } else {
      const int q1 = p1 - it.ob, q2 = p2 - it.ob;
      if (q1 >= 0 && q2 >= 0 && q1 < it.kB && q2 < it.kB)
        v = -2.f * Wk[it.b_off + ((int64_t)(q1 * it.kB + q2) * it.co + o) * it.cs + (j - it.c)];
    }
    M[e] = v;
  }
}

// z[pixel] = [x[pixel] | relu(h[pixel])]  (NHWC rows of c and cs channels -> c + cs), 16-byte vectors
// when every row is (8 bf16 / 4 f32)-aligned, else elements
template <typename T, int V>
__global__ void __launch_bounds__(256) relu_concat_kernel(const T* __restrict__ x, const T* __restrict__ h,
                                                          T* __restrict__ z, int64_t pixels, int c, int cs) {
  const int cz = c + cs;
  const bool vec = (c % V == 0) && (cs % V == 0);
  const int64_t per = vec ? cz / V : cz;
  const int64_t total = pixels * per;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t px = e / per;
    const int q = (int)(e - px * per);
    if (vec) {
      const int ch = q * V;
      uint4 v;
      if (ch < c) {
        v = *reinterpret_cast<const uint4*>(x + px * c + ch);
      } else {
        v = *reinterpret_cast<const uint4*>(h + px * cs + (ch - c));
        T* t = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = (float)t[i] > 0.f ? t[i] : T(0.f);
      }
      *reinterpret_cast<uint4*>(z + px * cz + ch) = v;
    } else {
      const int ch = q;
      T v = ch < c ? x[px * c + ch] : h[px * cs + (ch - c)];
      if (ch >= c && !((float)v > 0.f)) v = T(0.f);
      z[px * cz + ch] = v;
    }
  }
}

}  // namespace

int launch_sll_scale(Plan& p, const float* ortho, void* stream) {
  if (p.sll.empty()) return 0;
  sll_scale_kernel<<<(unsigned)p.sll.size(), 256, 0, (cudaStream_t)stream>>>(p.d_sll, ortho, p.d_comp);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_blk_merge(Plan& p, void* stream) {
  if (p.blk.empty()) return 0;
  int64_t mx = 1;
  for (auto& b : p.blk) mx = std::max<int64_t>(mx, (int64_t)b.kM * b.kM * b.co * (b.c + b.cs));
  const int bx = (int)std::min<int64_t>((mx + 255) / 256, 1024);
  blk_merge_kernel<<<dim3((unsigned)bx, (unsigned)p.blk.size()), 256, 0, (cudaStream_t)stream>>>(p.d_blk, p.d_comp);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_relu_concat(const void* x, const void* h, void* z, int64_t pixels, int c, int cs, int io, void* stream) {
  const int64_t total = pixels * (c + cs);
  const int blocks = (int)std::min<int64_t>((total / 4 + 255) / 256 + 1, 148 * 16);
  if (io == ORTH_BF16)
    relu_concat_kernel<__nv_bfloat16, 8><<<blocks, 256, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)h, (__nv_bfloat16*)z, pixels, c, cs);
  else
    relu_concat_kernel<float, 4><<<blocks, 256, 0, (cudaStream_t)stream>>>((const float*)x, (const float*)h,
                                                                           (float*)z, pixels, c, cs);
  return (int)cudaGetLastError();
}

}  // namespace orth
