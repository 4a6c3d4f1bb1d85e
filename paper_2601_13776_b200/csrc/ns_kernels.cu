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

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include <cstdint>

#include "orth_internal.h"
#include "pdl.h"
#include "umma.cuh"

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

// ---------------------------------------------------------------- power iteration (O2)
// One power step of the oracle (prescale_power): wv = W v; u = wv / |wv|;
// w = W^T u; sig = |w|; v = w / sig.  Split over row items (t = W v, |t|^2
// partials) and column items (w = W^T u, |w|^2 partials) with a grid barrier
// between; every norm is a fixed-order sum over the matrix's items.
#ifdef ORTH_POWER_TRACE
__device__ unsigned long long power_trace[1024 * 8];
#endif
__device__ __forceinline__ void power_grid_sync(unsigned* bar, unsigned target) {
#ifdef ORTH_POWER_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024 && target / gridDim.x <= 7) {   // arrival time at barrier k
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    power_trace[blockIdx.x * 8 + target / gridDim.x] = t;
  }
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;   // relaxed polls + one acquire fence (an ld.acquire per poll invalidates L1 each time)
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

// fixed-order sum of cnt partials (thread 0), broadcast through smem
// (the partials are fetched by all threads at once -- one L2 round trip -- and
// summed by thread 0 in index order from shared memory: deterministic)
__device__ __forceinline__ float ordered_sum(const float* p, int cnt, float* slot) {
  __shared__ float vals[256];
  __syncthreads();
  for (int c = threadIdx.x; c < cnt && c < 256; c += blockDim.x) vals[c] = __ldcg(p + c);
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int c = 0; c < cnt; ++c) s += c < 256 ? vals[c] : __ldcg(p + c);
    *slot = s;
  }
  __syncthreads();
  return *slot;
}

constexpr int kPowerStage = 10240;   // floats of a W block staged in smem by one power item

struct PowerBufs {
  float* t;       // t = W v, per matrix at t_off
  float* tpart;   // |t|^2 per row item
  float* wpart;   // |w|^2 per column item
};

__global__ void __launch_bounds__(256) power_fused_kernel(const PowerItem* __restrict__ items, int n_items,
                                                          const ColItem* __restrict__ cols, int n_cols,
                                                          const MatItem* __restrict__ mats, int n_mats,
                                                          const float* __restrict__ W, const float* vin0, int use_const,
                                                          int frob, int iters, PowerBufs pb, float* vbuf,
                                                          float* __restrict__ cache_out, float* __restrict__ sigma,
                                                          int32_t* __restrict__ status, unsigned* bar) {
  extern __shared__ float sm[];
  __shared__ float red[9];
  __shared__ float slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned k = 0;
#ifdef ORTH_POWER_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    power_trace[blockIdx.x * 8 + 0] = t;
  }
#endif
  if (frob) {   // |W|_F: sums of squares per row item, then per matrix in item order
    for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
      const PowerItem it = items[i];
      const float* Wm = W + it.off;
      float acc = 0.f;
      for (int64_t e = (int64_t)it.r0 * it.n + threadIdx.x; e < (int64_t)it.r1 * it.n; e += 256) {
        const float x = Wm[e];
        acc = fmaf(x, x, acc);
      }
      acc = block_sum(acc, red);
      if (threadIdx.x == 0) pb.tpart[it.chunk] = acc;
    }
    power_grid_sync(bar, ++k * gridDim.x);
    for (int m = blockIdx.x; m < n_mats; m += gridDim.x) {
      const MatItem M = mats[m];
      float sg = sqrtf(ordered_sum(pb.tpart + M.chunk0, M.nchunks, &slot));
      if (threadIdx.x == 0) {
        if (!(sg > 0.f) || !isfinite(sg)) { atomicCAS(status, 0, (int)ORTH_ERR_ZERO_NORM); sg = 1.f; }
        sigma[M.mat] = sg;
      }
    }
    return;
  }
  for (int itr = 0; itr < iters; ++itr) {
    // ---- A: t = W v over row items (T threads per row, shuffle-reduced)
    for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
      const PowerItem it = items[i];
      const int n = it.n, rows = it.r1 - it.r0;
      float scale;
      const float* vsrc;
      if (itr == 0) {
        scale = use_const ? rsqrtf((float)n) : 1.f;
        vsrc = use_const ? nullptr : vin0 + it.cache_off;
      } else {   // v = w / |w| of the previous step
        const MatItem M = mats[it.midx];
        const float ww = ordered_sum(pb.wpart + M.col0, M.ncols, &slot);
        scale = ww > 0.f ? rsqrtf(ww) : 0.f;
        vsrc = vbuf + it.cache_off;
      }
      float* v = sm;
      for (int j = threadIdx.x; j < n; j += 256) v[j] = vsrc ? vsrc[j] * scale : scale;
      int T = 1;
      while (T < 32 && rows * T * 2 <= 256) T *= 2;
      float tt = 0.f;
      const float* Wm = W + it.off;
      // stage the block in smem with all loads in flight (rows padded to n + 4)
      const int ldw = n + 4;
      float* Ws = sm + ((n + 3) & ~3);
      const bool staged = (n & 3) == 0 && rows * ldw <= kPowerStage;
      if (staged) {
        const float4* src = reinterpret_cast<const float4*>(Wm + (int64_t)it.r0 * n);
        const int n4 = n >> 2;
        for (int e = threadIdx.x; e < rows * n4; e += 256) {
          const int r = e / n4, c = e - r * n4;
          *reinterpret_cast<float4*>(Ws + r * ldw + 4 * c) = __ldg(src + e);
        }
      }
      __syncthreads();
      for (int r0 = 0; r0 < rows; r0 += 256 / T) {
        const int r = r0 + threadIdx.x / T, sub = threadIdx.x % T;
        float a = 0.f;
        if (r < rows) {
          if (staged) {   // four independent accumulators (the chain was LDS-latency bound), summed in order
            const float* row = Ws + r * ldw;
            float a1 = 0.f, a2 = 0.f, a3 = 0.f;
            int j = sub;
            for (; j + 3 * T < n; j += 4 * T) {
              a = fmaf(row[j], v[j], a);
              a1 = fmaf(row[j + T], v[j + T], a1);
              a2 = fmaf(row[j + 2 * T], v[j + 2 * T], a2);
              a3 = fmaf(row[j + 3 * T], v[j + 3 * T], a3);
            }
            for (; j < n; j += T) a = fmaf(row[j], v[j], a);
            a = (a + a1) + (a2 + a3);
          } else {
            const float* row = Wm + (int64_t)(it.r0 + r) * n;
            float a2 = 0.f;
            int j = sub;
#pragma unroll 4
            for (; j + T < n; j += 2 * T) {
              a = fmaf(__ldg(row + j), v[j], a);
              a2 = fmaf(__ldg(row + j + T), v[j + T], a2);
            }
            if (j < n) a = fmaf(__ldg(row + j), v[j], a);
            a += a2;
          }
        }
        for (int o = T >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (r < rows && sub == 0) {
          pb.t[it.t_off + it.r0 + r] = a;
          tt = fmaf(a, a, tt);
        }
      }
      tt = block_sum(tt, red);
      if (threadIdx.x == 0) pb.tpart[it.chunk] = tt;
      __syncthreads();
    }
    power_grid_sync(bar, ++k * gridDim.x);
    // ---- B: w = W^T u, u = t / |t|, over column items
    for (int c = blockIdx.x; c < n_cols; c += gridDim.x) {
      const ColItem ci = cols[c];
      const MatItem M = mats[ci.midx];
      const int n = ci.n, m = ci.m, cw = ci.c1 - ci.c0;
      const float tt = ordered_sum(pb.tpart + M.chunk0, M.nchunks, &slot);
      const float inv = tt > 0.f ? rsqrtf(tt) : 0.f;
      if (threadIdx.x == 0 && !(tt > 0.f && isfinite(tt))) atomicCAS(status, 0, (int)ORTH_ERR_ZERO_NORM);
      float* u = sm;
      for (int r = threadIdx.x; r < m; r += 256) u[r] = pb.t[ci.t_off + r] * inv;
      const int lanes = cw <= 16 ? 16 : cw < 256 ? ((cw + 31) / 32) * 32 : 256;   // column threads
      const int ng = 256 / lanes, g = threadIdx.x / lanes, jj = threadIdx.x % lanes;
      float* part = sm + ((m + 3) & ~3);   // ng x lanes
      const float* Wm = W + ci.off;
      // stage the column block in smem (rows of cw padded to cw + 4) when it fits
      const int ldc = cw + 4;
      float* Ws = part + 256;
      const bool staged = ((n | ci.c0 | cw) & 3) == 0 && m * ldc <= kPowerStage;
      if (staged) {
        const int c4n = cw >> 2;
        for (int e = threadIdx.x; e < m * c4n; e += 256) {
          const int r = e / c4n, c = e - r * c4n;
          *reinterpret_cast<float4*>(Ws + r * ldc + 4 * c) =
              __ldg(reinterpret_cast<const float4*>(Wm + (int64_t)r * n + ci.c0) + c);
        }
      }
      __syncthreads();
      float ww = 0.f;
      for (int j0 = 0; j0 < cw; j0 += lanes) {
        const int j = ci.c0 + j0 + jj;
        float a = 0.f;
        if (g < ng && j0 + jj < cw) {
          if (staged) {
            float a1 = 0.f, a2 = 0.f, a3 = 0.f;
            int r = g;
            for (; r + 3 * ng < m; r += 4 * ng) {
              a = fmaf(Ws[r * ldc + j0 + jj], u[r], a);
              a1 = fmaf(Ws[(r + ng) * ldc + j0 + jj], u[r + ng], a1);
              a2 = fmaf(Ws[(r + 2 * ng) * ldc + j0 + jj], u[r + 2 * ng], a2);
              a3 = fmaf(Ws[(r + 3 * ng) * ldc + j0 + jj], u[r + 3 * ng], a3);
            }
            for (; r < m; r += ng) a = fmaf(Ws[r * ldc + j0 + jj], u[r], a);
            a = (a + a1) + (a2 + a3);
          } else {
#pragma unroll 8
            for (int r = g; r < m; r += ng) a = fmaf(__ldg(Wm + (int64_t)r * n + j), u[r], a);
          }
        }
        if (g < ng) part[g * lanes + jj] = a;
        __syncthreads();
        if (threadIdx.x < lanes && j0 + threadIdx.x < cw) {
          float w = 0.f;
          for (int q = 0; q < ng; ++q) w += part[q * lanes + threadIdx.x];
          vbuf[ci.cache_off + ci.c0 + j0 + threadIdx.x] = w;
          ww = fmaf(w, w, ww);
        }
        __syncthreads();
      }
      ww = block_sum(ww, red);
      if (threadIdx.x == 0) pb.wpart[ci.chunk] = ww;
      __syncthreads();
    }
    power_grid_sync(bar, ++k * gridDim.x);
  }
  // ---- finalize: sig = |w|, v = w / sig (cache), per matrix
  for (int mi = blockIdx.x; mi < n_mats; mi += gridDim.x) {
    const MatItem M = mats[mi];
    const float ww = ordered_sum(pb.wpart + M.col0, M.ncols, &slot);
    float sg = sqrtf(ww);
    const bool bad = !(sg > 0.f) || !isfinite(sg);
    if (bad) sg = 1.f;
    const float inv = 1.f / sg;
    for (int j = threadIdx.x; j < M.n; j += 256) {
      const float v = vbuf[M.cache_off + j] * inv;
      vbuf[M.cache_off + j] = v;
      if (cache_out) cache_out[M.cache_off + j] = v;
    }
    if (threadIdx.x == 0) {
      sigma[M.mat] = sg;
      if (bad) atomicCAS(status, 0, (int)ORTH_ERR_ZERO_NORM);
    }
    __syncthreads();
  }
  (void)warp;
  (void)lane;
}

__global__ void __launch_bounds__(256) scale_kernel(const PowerItem* __restrict__ items, const float* __restrict__ W,
                                                    const float* __restrict__ sigma, float* __restrict__ X0,
                                                    unsigned* __restrict__ power_bar) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *power_bar = 0u;   // re-arm the fused power kernel's barrier
  const PowerItem it = items[blockIdx.x];
  const float inv = 1.f / sigma[it.mat];
  const int64_t beg = it.off + (int64_t)it.r0 * it.n, end = it.off + (int64_t)it.r1 * it.n;
  for (int64_t e = beg + threadIdx.x; e < end; e += 256) X0[e] = W[e] * inv;
}

// Residual reduction in two deterministic stages (R20).  Stage 1: one CTA per residual item
// (a ~16K-element slice of a matrix's s x s Gram G, or of R = I - X^T X when is_r) writes its sum of
// squares of (I - G) to part[item].  Stage 2: one warp per matrix sums its items in item order:
// r = |I - G|_F.  NOT_CONVERGED when r is non-finite or the checked value exceeds tol > 0: r itself for
// the final residual, or -- bound = 1, r of the LAST iteration's input X_{T-1} -- the bound on the
// result's residual: with R symmetric and X' = X (I + R/2), I - X'^T X' = 3/4 R^2 + 1/4 R^3 exactly,
// so |I - X_T^T X_T|_F <= 3/4 r^2 + 1/4 r^3.
__global__ void __launch_bounds__(256) residual_part_kernel(const ResItem* __restrict__ items,
                                                            const MatItem* __restrict__ mats,
                                                            const float* __restrict__ G, float* __restrict__ part,
                                                            int is_r) {
  __shared__ float red[9];
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const ResItem it = items[blockIdx.x];
  const MatItem M = mats[it.midx];
  const int64_t s = M.m < M.n ? M.m : M.n;
  const float* g = G + M.gram_off;
  float a = 0.f;
  for (int64_t e = it.e0 + threadIdx.x; e < it.e1; e += 256) {
    const int64_t i = e / s, j = e - i * s;
    const float r = is_r ? g[e] : (i == j ? 1.f : 0.f) - g[e];
    a = fmaf(r, r, a);
  }
  a = block_sum(a, red);
  if (threadIdx.x == 0) part[blockIdx.x] = a;
}

__global__ void __launch_bounds__(256) residual_final_kernel(const MatItem* __restrict__ mats, int nmats,
                                                             const float* __restrict__ part, float* __restrict__ res,
                                                             int32_t* __restrict__ status, float tol, int bound) {
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const int w = (int)(blockIdx.x * 8 + (threadIdx.x >> 5)), lane = threadIdx.x & 31;
  if (w >= nmats) return;
  const MatItem M = mats[w];
  float a = 0.f;
  for (int i = lane; i < M.nres; i += 32) a += part[M.res0 + i];   // fixed per-lane order
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) {
    const float r = sqrtf(a);
    if (res) res[M.mat] = r;
    const float chk = bound ? r * r * (0.75f + 0.25f * r) : r;
    if (!isfinite(r) || (tol > 0.f && !(chk <= tol))) atomicCAS(status, 0, (int)ORTH_ERR_NOT_CONVERGED);
  }
}

}  // namespace

int launch_gemm_f32(const GemmPhase& ph, float* const bufs[BUF_COUNT], void* stream) {
  if (ph.total_tiles == 0) return 0;
  gemm_f32_kernel<<<ph.total_tiles, 256, 0, (cudaStream_t)stream>>>(ph.d_descs, (int)ph.descs.size(), ph.d_segs,
                                                                    bufs[0], bufs[1], bufs[2], bufs[3]);
  return (int)cudaGetLastError();
}

int launch_power_fused(Plan& p, const float* W, const float* v_in, int use_const_v, int frob, int iters,
                       float* cache_out, void* stream) {
  if (p.power_items.empty()) return 0;
  int64_t maxn = 0, maxm = 0;
  for (auto& m : p.mat_items) { maxn = std::max<int64_t>(maxn, m.n); maxm = std::max<int64_t>(maxm, m.m); }
  // smem: v (n) + staged block for row items; u (m) + 256 partial sums + staged block for column items
  const size_t smem = (size_t)(std::max<int64_t>(((maxn + 3) & ~3), ((maxm + 3) & ~3) + 256) + kPowerStage) *
                      sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(power_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, power_fused_kernel, 256, smem);
  if (occ < 1) return (int)cudaErrorInvalidConfiguration;
  const int n_items = (int)p.power_items.size(), n_cols = (int)p.col_items.size(), n_mats = (int)p.mat_items.size();
  static const int mult = std::getenv("ORTH_POWER_CTAS_PER_SM") ? std::atoi(std::getenv("ORTH_POWER_CTAS_PER_SM")) : 4;
  const int grid = std::max(1, std::min(std::max(n_items, n_cols), std::max(1, std::min(occ, mult)) * sms));
  PowerBufs pb;
  pb.t = p.d_partial;
  pb.tpart = p.d_partial + pad_up(p.t_numel, kPadF32);
  pb.wpart = pb.tpart + pad_up(p.n_chunks, kPadF32);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr_c[1];
  attr_c[0].id = cudaLaunchAttributeCooperative;
  attr_c[0].val.cooperative = 1;
  cfg.attrs = attr_c;
  cfg.numAttrs = 1;
  p.launches++;
  const int e = (int)cudaLaunchKernelEx(&cfg, power_fused_kernel, (const PowerItem*)p.d_power_items, n_items,
                                        (const ColItem*)p.d_col_items, n_cols, (const MatItem*)p.d_mat_items, n_mats,
                                        W, v_in, use_const_v, frob, iters, pb, p.d_vbuf, cache_out, p.d_sigma,
                                        p.d_status, power_bar(p));
#ifdef ORTH_POWER_TRACE
  {   // per barrier k: mean / max arrival after the kernel start (all CTAs)
    cudaStreamSynchronize((cudaStream_t)stream);
    static unsigned long long h[1024 * 8];
    cudaMemcpyFromSymbol(h, power_trace, sizeof(h));
    const int nb = std::min(grid, 1024);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < nb; ++c) t0 = std::min(t0, h[c * 8]);
    std::printf("power_fused grid=%d items=%d cols=%d:", grid, n_items, n_cols);
    for (int q = 1; q <= 2 * iters && q < 8; ++q) {
      double mean = 0, mx = 0;
      for (int c = 0; c < nb; ++c) { const double d = (double)(h[c * 8 + q] - t0) * 1e-3; mean += d; mx = std::max(mx, d); }
      std::printf(" b%d %.1f/%.1f", q, mean / nb, mx);
    }
    std::printf(" us (mean/max arrival)\n");
  }
#endif
  return e;
}

int launch_scale(Plan& p, const float* W, float* X0, void* stream) {
  if (p.power_items.empty()) return 0;
  scale_kernel<<<(int)p.power_items.size(), 256, 0, (cudaStream_t)stream>>>(p.d_power_items, W, p.d_sigma, X0,
                                                                            power_bar(p));
  p.launches++;
  return (int)cudaGetLastError();
}

static int residual_two_stage(Plan& p, int is_r, float* res, float tol, int bound, void* stream) {
  if (p.mat_items.empty()) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_pdl(residual_part_kernel, dim3((unsigned)p.res_items.size()), dim3(256), 0, st,
             (const ResItem*)p.d_res_items, (const MatItem*)p.d_mat_items, (const float*)p.d_gram, p.d_res_part, is_r);
  const int nm = (int)p.mat_items.size();
  launch_pdl(residual_final_kernel, dim3((unsigned)((nm + 7) / 8)), dim3(256), 0, st, (const MatItem*)p.d_mat_items,
             nm, (const float*)p.d_res_part, res, p.d_status, tol, bound);
  p.launches += 2;
  return (int)cudaGetLastError();
}

int launch_residual(Plan& p, float* residual_out, void* stream) {
  return residual_two_stage(p, 0, residual_out, p.opts.ns_tol, 0, stream);
}

int launch_converged_check(Plan& p, int is_r, float tol, void* stream) {
  return residual_two_stage(p, is_r, p.d_ns_res, tol, 1, stream);
}

int launch_residual_r(Plan& p, float* residual_out, void* stream) {
  return residual_two_stage(p, 1, residual_out, p.opts.ns_tol, 0, stream);
}

}  // namespace orth
