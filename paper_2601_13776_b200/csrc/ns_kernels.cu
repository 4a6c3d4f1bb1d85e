// Pre-scaling (a2) and the FP32-accurate batched GEMM used by Bjorck/NS (a3)
// and the composition chain (a4/a5).
//
//  * power iteration (reading R2): per iteration one pass
//    over W: t = W v (warp per row), partial w = sum_r t_r W[r,:] and
//    partial |Wv|^2 per row chunk; a finalize CTA per matrix reduces the
//    partials in chunk order (deterministic), u = Wv/|Wv|, w = W^T u,
//    sigma = |w|, v = w/sigma.
//  * gemm_f32: ragged batch of D = alpha * sum_seg A_seg B_seg + beta * C
//    problems (descriptors built once by plan.cpp), 64x64 tiles, FP32 FFMA
//    (the FP32-accurate path: 1e-5 parity needs FP32 products, R16).
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"

namespace orth {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ int find_problem(const GemmDesc* __restrict__ d, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) gemm_f32_kernel(const GemmDesc* __restrict__ descs, int ndesc,
                                                       const GemmSeg* __restrict__ segs, float* b0, float* b1,
                                                       float* b2, float* b3) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int pidx = find_problem(descs, ndesc, blockIdx.x);
  const GemmDesc d = descs[pidx];
  float* bufs[4] = {b0, b1, b2, b3};
  const int local = blockIdx.x - d.tile_begin;
  const int m0 = (local / d.tiles_n) * BM, n0 = (local % d.tiles_n) * BN;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const bool a_k_contig = d.sa_k == 1;
  const bool b_n_contig = d.sb_n == 1;
  for (int sg = 0; sg < d.seg_count; ++sg) {
    const GemmSeg s = segs[d.seg_begin + sg];
    const float* __restrict__ A = bufs[d.a_buf] + s.a_off;
    const float* __restrict__ A2 = s.a2_off >= 0 ? bufs[d.a_buf] + s.a2_off : nullptr;
    const float* __restrict__ B = bufs[d.b_buf] + s.b_off;
    for (int k0 = 0; k0 < d.K; k0 += BK) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256;
        int i, kk;
        if (a_k_contig) { i = e / BK; kk = e % BK; } else { kk = e / BM; i = e % BM; }
        const int gi = m0 + i, gk = k0 + kk;
        float v = 0.f;
        if (gi < d.M && gk < d.K) {
          const int64_t o = (int64_t)gi * d.sa_m + (int64_t)gk * d.sa_k;
          v = A[o];
          if (A2) v -= A2[o];
        }
        As[kk][i] = v;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * 256;
        int j, kk;
        if (b_n_contig) { kk = e / BN; j = e % BN; } else { j = e / BK; kk = e % BK; }
        const int gj = n0 + j, gk = k0 + kk;
        Bs[kk][j] = (gj < d.N && gk < d.K) ? B[(int64_t)gk * d.sb_k + (int64_t)gj * d.sb_n] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  const float* __restrict__ C = d.c_off >= 0 ? bufs[d.c_buf] + d.c_off : nullptr;
  float* __restrict__ D = bufs[d.d_buf] + d.d_off;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = m0 + ty * 4 + i;
    if (gi >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = n0 + tx * 4 + j;
      if (gj >= d.N) continue;
      float v = d.alpha * acc[i][j];
      if (C) v = fmaf(d.beta, C[(int64_t)gi * d.ldc + gj], v);
      if (gi == gj) v += d.diag;
      D[(int64_t)gi * d.ldd + gj] = v;
    }
  }
}

// ---------------------------------------------------------------- pre-scaling
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed tree), blockDim.x == 256
__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = (threadIdx.x < 8) ? red[threadIdx.x] : 0.f;
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) red[8] = r;
  __syncthreads();
  return red[8];
}

// One CTA per PowerItem.  Power: partial[chunk] = (sum_r t_r W[r,:], sum_r t_r^2)
// with t = W v.  Frobenius: partial[chunk][0] = sum of squares.
__global__ void __launch_bounds__(256) power_partial_kernel(const PowerItem* __restrict__ items,
                                                            const float* __restrict__ W, const float* __restrict__ vin,
                                                            int use_const, int frob, float* __restrict__ partial,
                                                            int64_t stride) {
  extern __shared__ float sm[];
  __shared__ float red[9];
  const PowerItem it = items[blockIdx.x];
  const int n = it.n;
  const float* __restrict__ Wm = W + it.off;
  float* __restrict__ out = partial + (int64_t)it.chunk * stride;
  const int rows = it.r1 - it.r0;
  if (frob) {
    float acc = 0.f;
    const int64_t beg = (int64_t)it.r0 * n, end = (int64_t)it.r1 * n;
    for (int64_t e = beg + threadIdx.x; e < end; e += 256) { const float x = Wm[e]; acc = fmaf(x, x, acc); }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) out[0] = acc;
    return;
  }
  float* v = sm;          // n
  float* t = sm + n;      // rows
  const float inv = rsqrtf((float)n);
  const float* vsrc = use_const ? nullptr : vin + it.cache_off;
  for (int j = threadIdx.x; j < n; j += 256) v[j] = use_const ? inv : vsrc[j];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float tt = 0.f;
  for (int r = warp; r < rows; r += 8) {
    const float* row = Wm + (int64_t)(it.r0 + r) * n;
    float a = 0.f;
    for (int j = lane; j < n; j += 32) a = fmaf(row[j], v[j], a);
    a = warp_sum(a);
    if (lane == 0) t[r] = a;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < rows; r += 256) tt = fmaf(t[r], t[r], tt);
  tt = block_sum(tt, red);
  for (int j = threadIdx.x; j < n; j += 256) {
    float a = 0.f;
    for (int r = 0; r < rows; ++r) a = fmaf(t[r], Wm[(int64_t)(it.r0 + r) * n + j], a);
    out[j] = a;
  }
  if (threadIdx.x == 0) out[n] = tt;
}

// One CTA per owned matrix: reduce partials in chunk order.
__global__ void __launch_bounds__(256) power_finalize_kernel(const MatItem* __restrict__ mats,
                                                             const float* __restrict__ partial, int64_t stride,
                                                             int frob, float* __restrict__ vbuf,
                                                             float* __restrict__ cache_out, float* __restrict__ sigma,
                                                             int32_t* __restrict__ status) {
  __shared__ float red[9];
  const MatItem M = mats[blockIdx.x];
  const int n = M.n;
  if (frob) {
    float s = 0.f;
    if (threadIdx.x == 0)
      for (int c = 0; c < M.nchunks; ++c) s += partial[(int64_t)(M.chunk0 + c) * stride];
    if (threadIdx.x == 0) {
      float sg = sqrtf(s);
      if (!(sg > 0.f) || !isfinite(sg)) { atomicCAS(status, 0, (int)ORTH_ERR_ZERO_NORM); sg = 1.f; }
      sigma[M.mat] = sg;
    }
    return;
  }
  // |Wv|^2: one chunk per thread (nchunks <= 64), fixed-tree block sum
  float ss = threadIdx.x < M.nchunks ? partial[(int64_t)(M.chunk0 + threadIdx.x) * stride + n] : 0.f;
  ss = block_sum(ss, red);
  const bool bad = !(ss > 0.f) || !isfinite(ss);
  const float inv_wv = bad ? 0.f : rsqrtf(ss);
  float nw = 0.f;
  for (int j = threadIdx.x; j < n; j += 256) {
    float w = 0.f;
#pragma unroll 8
    for (int c = 0; c < M.nchunks; ++c) w += partial[(int64_t)(M.chunk0 + c) * stride + j];
    w *= inv_wv;
    vbuf[M.cache_off + j] = w;
    nw = fmaf(w, w, nw);
  }
  nw = block_sum(nw, red);
  float sg = sqrtf(nw);
  const bool bad2 = bad || !(sg > 0.f) || !isfinite(sg);
  if (bad2) sg = 1.f;
  const float inv = 1.f / sg;
  for (int j = threadIdx.x; j < n; j += 256) {
    const float v = vbuf[M.cache_off + j] * inv;
    vbuf[M.cache_off + j] = v;
    if (cache_out) cache_out[M.cache_off + j] = v;
  }
  if (threadIdx.x == 0) {
    sigma[M.mat] = sg;
    if (bad2) atomicCAS(status, 0, (int)ORTH_ERR_ZERO_NORM);
  }
}

__global__ void __launch_bounds__(256) scale_kernel(const PowerItem* __restrict__ items, const float* __restrict__ W,
                                                    const float* __restrict__ sigma, float* __restrict__ X0) {
  const PowerItem it = items[blockIdx.x];
  const float inv = 1.f / sigma[it.mat];
  const int64_t beg = it.off + (int64_t)it.r0 * it.n, end = it.off + (int64_t)it.r1 * it.n;
  for (int64_t e = beg + threadIdx.x; e < end; e += 256) X0[e] = W[e] * inv;
}

// |I - G|_F per owned matrix from its Gram; non-finite -> NOT_CONVERGED
__global__ void __launch_bounds__(256) residual_kernel(const MatItem* __restrict__ mats, const float* __restrict__ G,
                                                       float* __restrict__ res, int32_t* __restrict__ status,
                                                       int is_r) {
  __shared__ float red[9];
  const MatItem M = mats[blockIdx.x];
  const int s = M.m < M.n ? M.m : M.n;
  const float* g = G + M.gram_off;
  float a = 0.f;
  for (int64_t e = threadIdx.x; e < (int64_t)s * s; e += 256) {
    const int i = (int)(e / s), j = (int)(e % s);
    const float r = is_r ? g[e] : (i == j ? 1.f : 0.f) - g[e];
    a = fmaf(r, r, a);
  }
  a = block_sum(a, red);
  if (threadIdx.x == 0) {
    const float r = sqrtf(a);
    if (res) res[M.mat] = r;
    if (!isfinite(r)) atomicCAS(status, 0, (int)ORTH_ERR_NOT_CONVERGED);
  }
}

}  // namespace

int launch_gemm_f32(const GemmPhase& ph, float* const bufs[BUF_COUNT], void* stream) {
  if (ph.total_tiles == 0) return 0;
  gemm_f32_kernel<<<ph.total_tiles, 256, 0, (cudaStream_t)stream>>>(ph.d_descs, (int)ph.descs.size(), ph.d_segs,
                                                                    bufs[0], bufs[1], bufs[2], bufs[3]);
  return (int)cudaGetLastError();
}

int launch_power_partial(Plan& p, const float* W, const float* v_in, int use_const_v, int frob, void* stream) {
  if (p.power_items.empty()) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(power_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  int64_t maxn = 0, maxr = 0;
  for (auto& it : p.power_items) { maxn = it.n > maxn ? it.n : maxn; maxr = (it.r1 - it.r0) > maxr ? (it.r1 - it.r0) : maxr; }
  const size_t smem = frob ? 0 : (size_t)(maxn + maxr) * sizeof(float);
  power_partial_kernel<<<(int)p.power_items.size(), 256, smem, (cudaStream_t)stream>>>(
      p.d_power_items, W, v_in, use_const_v, frob, p.d_partial, p.partial_stride);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_power_finalize(Plan& p, float* cache_out, int frob, int, void* stream) {
  if (p.mat_items.empty()) return 0;
  power_finalize_kernel<<<(int)p.mat_items.size(), 256, 0, (cudaStream_t)stream>>>(
      p.d_mat_items, p.d_partial, p.partial_stride, frob, p.d_vbuf, cache_out, p.d_sigma, p.d_status);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_scale(Plan& p, const float* W, float* X0, void* stream) {
  if (p.power_items.empty()) return 0;
  scale_kernel<<<(int)p.power_items.size(), 256, 0, (cudaStream_t)stream>>>(p.d_power_items, W, p.d_sigma, X0);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_residual(Plan& p, float* residual_out, void* stream) {
  if (p.mat_items.empty()) return 0;
  residual_kernel<<<(int)p.mat_items.size(), 256, 0, (cudaStream_t)stream>>>(p.d_mat_items, p.d_gram, residual_out,
                                                                             p.d_status, 0);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_residual_r(Plan& p, float* residual_out, void* stream) {
  if (p.mat_items.empty()) return 0;
  residual_kernel<<<(int)p.mat_items.size(), 256, 0, (cudaStream_t)stream>>>(p.d_mat_items, p.d_gram, residual_out,
                                                                             p.d_status, 1);
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
