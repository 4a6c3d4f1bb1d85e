// f1: weight gradient of the conv apply (a6), the
// contraction behind P:122's training wall time: for every group g and tap
// t = (a, b)
//   dK[g co + o, i, a, b] = sum_{pixels p} dy[p, g co + o] x~[pix(p, t), g ci + i]
// a GEMM with M = c_out/g, N = c_in/g and K = the N Ho Wo output pixels.
//
// wgrad_tc<BN>: one CTA per (pixel split, group, tap, 128-row M tile, BN-wide
// N tile).  4 producer warps gather 64 pixels per stage with 16-byte
// cp.async: the dy rows (128 channels) and the tap-shifted x rows (BN
// channels; zero fill outside the image or circular wrap) land as MN-MAJOR
// SWIZZLE_128B tiles -- a pixel's channels are contiguous in NHWC, exactly the
// MN-major atom (64 MN elements x 8 K rows) -- so no transpose is needed.  One
// thread issues tcgen05.mma M=128 N=BN K=16 (MN-major A and B) into TMEM; the
// epilogue writes the FP32 tile as this split's partial.  wgrad_reduce sums the
// splits in a fixed order into the PyTorch-layout FP32 dK (deterministic, no
// atomics).  wgrad_simt: FP32 I/O (and BF16 shapes the 16-byte gather cannot
// take), one thread per dK element, fixed pixel order.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"
#include "umma.cuh"

namespace orth {
namespace {

struct WgArgs {
  int N, H, W, Ho, Wo;
  int Ci, Co;              // channels of an x row / a dy row (forward view)
  int ci, co, g, k, s, d, pt, pl, circ;
  int64_t pixels;          // N Ho Wo
  int splits, tiles_m, tiles_n, kk;
  int64_t per_split;       // pixels per split (multiple of 64)
  int tpc, tgroups;        // taps per CTA (consecutive in row-major tap order), tap groups
};

constexpr int kProd = 256;   // 8 producer / epilogue warps

// input pixel (flattened n, h, w) read by output pixel p at tap (ta, tb); -1 = zero padding.  32-bit:
// N Ho Wo and N H W stay below 2^31 for every workload here (checked on the host)
__device__ __forceinline__ int in_pixel32(const WgArgs& a, int p, int ta, int tb) {
  const int hw = a.Ho * a.Wo;
  const int n = p / hw;
  const int r = p - n * hw;
  const int u = r / a.Wo, v = r - u * a.Wo;
  int h = a.s * u + a.d * ta - a.pt, w = a.s * v + a.d * tb - a.pl;
  if (a.circ) {
    h %= a.H; if (h < 0) h += a.H;
    w %= a.W; if (w < 0) w += a.W;
  } else if (h < 0 || h >= a.H || w < 0 || w >= a.W) {
    return -1;
  }
  return (n * a.H + h) * a.W + w;
}

__device__ __forceinline__ int64_t in_pixel(const WgArgs& a, int64_t p, int ta, int tb) {
  return in_pixel32(a, (int)p, ta, tb);
}

// One CTA = (pixel split, group, tap group of TPC consecutive taps, 128-row co tile, BN-wide ci tile).
// Per stage (64 pixels): the dy tile (A, MN-major, 16 KB) is gathered ONCE and multiplied with TPC
// tap-shifted x tiles (B_j, MN-major) into TPC accumulators (TPC * BN <= 512 TMEM columns).  Each of
// the 256 producer threads owns one quarter of one pixel row: it resolves its pixel's input offsets
// itself (no per-stage barrier) and issues its 16-byte cp.async chunks.
template <int BN, int TPC, int S>
__global__ void __launch_bounds__(kProd + 32, 1)
    wgrad_tc(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy, WgArgs a,
             float* __restrict__ part) {
  constexpr int A_BYTES = 2 * 8192, B_BYTES = (BN / 64) * 8192, STAGE = A_BYTES + TPC * B_BYTES;
  constexpr int TCOLS = TPC * BN <= 32 ? 32 : TPC * BN <= 64 ? 64 : TPC * BN <= 128 ? 128 : TPC * BN <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t full_bar[S], empty_bar[S], done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5;
  int64_t idx = blockIdx.x;
  const int nb = (int)(idx % a.tiles_n); idx /= a.tiles_n;
  const int mb = (int)(idx % a.tiles_m); idx /= a.tiles_m;
  const int tg = (int)(idx % a.tgroups); idx /= a.tgroups;
  const int grp = (int)(idx % a.g); idx /= a.g;
  const int split = (int)idx;
  const int t0 = tg * TPC;
  const int ntap = min(TPC, a.kk - t0);
  const int m0 = mb * 128, n0 = nb * BN;
  const int p_begin = (int)((int64_t)split * a.per_split);
  const int p_end = (int)(a.pixels < (int64_t)p_begin + a.per_split ? a.pixels : (int64_t)p_begin + a.per_split);
  const int nk = (p_end - p_begin + 63) / 64;

  if (warp == 8) umma::tmem_alloc(&tmem_base_sh, TCOLS);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], kProd);
      umma::mbar_init(&empty_bar[i], 1);
    }
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);

  if (warp < 8) {
    // ---------------- producers: thread = (pixel row r, quarter q)
    const int r = tid >> 2, q = tid & 3;
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const int p = p_begin + kb * 64 + r;
      const bool pin = p < p_end;
      const uint32_t sa = s0 + st * STAGE;
      // A: the dy row of pixel p, channels m0 .. m0 + 127 (16 chunks, 4 per thread)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = q * 4 + jj;
        const int o = m0 + 8 * j;
        const bool ok = pin && o < a.co;
        const __nv_bfloat16* src = dy + (ok ? ((int64_t)p * a.Co + (int64_t)grp * a.co + o) : 0);
        umma::cp_async16(sa + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4), src, ok);
      }
      // B_j: x rows of the tap-shifted input pixel, BN / 8 chunks (BN / 32 per thread)
      for (int jt = 0; jt < ntap; ++jt) {
        const int t = t0 + jt;
        const int ta = t / a.k, tb = t - ta * a.k;
        const int ip = pin ? in_pixel32(a, p, ta, tb) : -1;
        const uint32_t sb = sa + A_BYTES + jt * B_BYTES;
#pragma unroll
        for (int jj = 0; jj < BN / 32; ++jj) {
          const int j = q * (BN / 32) + jj;
          const int i = n0 + 8 * j;
          const bool ok = ip >= 0 && i < a.ci;
          const __nv_bfloat16* src = x + (ok ? ((int64_t)ip * a.Ci + (int64_t)grp * a.ci + i) : 0);
          umma::cp_async16(sb + (j >> 3) * 8192 + r * 128 + (((j & 7) ^ (r & 7)) << 4), src, ok);
        }
      }
      umma::cp_async_mbar_arrive(&full_bar[st]);
    }
    // ---------------- epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31, column half (w / 4)
    umma::mbar_wait(&done_bar, 0);
    umma::tc_fence_after();
    const int lq = warp & 3, half = warp >> 2;
    const int o = m0 + lq * 32 + (tid & 31);
    for (int jt = 0; jt < ntap; ++jt) {
      float* dst = part + (((int64_t)split * a.g + grp) * a.kk + t0 + jt) * ((int64_t)a.co * a.ci);
#pragma unroll 1
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(jt * BN + c0), v);
        if (o < a.co) {
          float* row = dst + (int64_t)o * a.ci + n0 + c0;
          if (n0 + c0 + 32 <= a.ci && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(row + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + c0 + j < a.ci) row[j] = v[j];
          }
        }
      }
    }
  } else if (tid == kProd) {
    // ---------------- MMA issuer: per stage, 4 K=16 steps x TPC taps sharing the A tile
    constexpr uint32_t IDESC = umma::idesc_bf16(128, BN) | (1u << 15) | (1u << 16);   // A, B MN-major
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      umma::mbar_wait(&full_bar[st], (kb / S) & 1);
      umma::fence_proxy_async_smem();   // cp.async (generic proxy) rows -> tcgen05.mma (async proxy)
      umma::tc_fence_after();
      const uint32_t sa = s0 + st * STAGE;
      for (int jt = 0; jt < ntap; ++jt) {
        const uint32_t sb = sa + A_BYTES + jt * B_BYTES;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          umma::mma_bf16(tmem + (uint32_t)(jt * BN), umma::sdesc_sw128_mn(sa + 2048 * q, 8192),
                         umma::sdesc_sw128_mn(sb + 2048 * q, 8192), IDESC, (kb | q) != 0);
      }
      umma::mma_commit(&empty_bar[st]);
    }
    umma::mma_commit(&done_bar);
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 8) umma::tmem_dealloc(tmem, TCOLS);
}

// dK[(g co + o) ci k^2 + i k^2 + t] = sum over splits (in order) of part[split][g][t][o][i]
__global__ void __launch_bounds__(256) wgrad_reduce(const float* __restrict__ part, WgArgs a, float* __restrict__ dK) {
  const int64_t total = (int64_t)a.g * a.co * a.ci * a.kk;
  const int64_t slab = (int64_t)a.g * a.kk * a.co * a.ci;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e % a.kk);
    int64_t r = e / a.kk;
    const int i = (int)(r % a.ci); r /= a.ci;
    const int o = (int)(r % a.co);
    const int grp = (int)(r / a.co);
    const int64_t src = (((int64_t)grp * a.kk + t) * a.co + o) * a.ci + i;
    float acc = 0.f;
    for (int sp = 0; sp < a.splits; ++sp) acc += part[sp * slab + src];
    dK[e] = acc;
  }
}

// SIMT weight gradient over pixel splits: thread = one dK element, walking its split's pixels in order
// (fixed order, deterministic); the splits are then reduced by wgrad_reduce_simt in split order.
template <typename T>
__global__ void __launch_bounds__(256) wgrad_simt(const T* __restrict__ x, const T* __restrict__ dy, WgArgs a,
                                                  float* __restrict__ part) {
  const int64_t total = (int64_t)a.g * a.co * a.ci * a.kk;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int split = blockIdx.y;
  if (e >= total) return;
  // element order e = ((grp kk + t) ci + i) co + o: a warp shares (grp, t, i) -- one broadcast x value per
  // pixel -- and reads 32 consecutive dy channels (coalesced)
  const int o = (int)(e % a.co);
  int64_t r = e / a.co;
  const int i = (int)(r % a.ci); r /= a.ci;
  const int t = (int)(r % a.kk);
  const int grp = (int)(r / a.kk);
  const int ta = t / a.k, tb = t - ta * a.k;
  const int64_t p0 = (int64_t)split * a.per_split, p1 = min(a.pixels, p0 + a.per_split);
  float acc = 0.f;
  for (int64_t p = p0; p < p1; ++p) {
    const int64_t ip = in_pixel(a, p, ta, tb);
    if (ip < 0) continue;
    acc = fmaf((float)dy[p * a.Co + (int64_t)grp * a.co + o], (float)x[ip * a.Ci + (int64_t)grp * a.ci + i], acc);
  }
  if (a.splits > 1) part[(int64_t)split * total + e] = acc;
  else part[(((int64_t)grp * a.co + o) * a.ci + i) * a.kk + t] = acc;   // straight into dK
}

// Small-kernel SIMT weight gradient (the RGB stem: c_in = 3 is not tensor-core aligned): the per-group
// element count E = co ci k^2 <= 4096 fits 256 threads x 16 registers.  A persistent CTA walks 64-pixel
// chunks (chunk = blockIdx.x + j gridDim.x, in order), staging each chunk's dy rows and tap-shifted x
// values in shared memory; thread tid owns elements e = tid + 256 j (order ((t ci + i) co + o): a warp
// reads one broadcast x value and consecutive dy channels).  One partial per CTA, reduced in CTA order.
constexpr int kSmallP = 64, kSmallJ = 16;
template <typename T>
__global__ void __launch_bounds__(256) wgrad_simt_small(const T* __restrict__ x, const T* __restrict__ dy, WgArgs a,
                                                        float* __restrict__ part) {
  extern __shared__ float sm[];
  const int grp = blockIdx.y;
  const int tci = a.kk * a.ci, E = a.co * tci;
  float* dys = sm;                       // [kSmallP][co]
  float* xs = sm + kSmallP * a.co;       // [kSmallP][kk ci]
  float acc[kSmallJ];
  int od[kSmallJ], ox[kSmallJ];   // per owned element: its dy channel and x column (hoisted divisions)
#pragma unroll
  for (int j = 0; j < kSmallJ; ++j) {
    acc[j] = 0.f;
    const int e = threadIdx.x + 256 * j, ti = e / a.co;
    od[j] = e - ti * a.co;
    ox[j] = ti;
  }
  const int64_t chunks = (a.pixels + kSmallP - 1) / kSmallP;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int64_t p0 = c * kSmallP;
    const int np = (int)(a.pixels - p0 < kSmallP ? a.pixels - p0 : kSmallP);
    for (int q = threadIdx.x; q < kSmallP * a.co; q += blockDim.x) {
      const int pp = q / a.co, o = q - pp * a.co;
      dys[q] = pp < np ? (float)dy[(p0 + pp) * a.Co + (int64_t)grp * a.co + o] : 0.f;
    }
    for (int q = threadIdx.x; q < kSmallP * tci; q += blockDim.x) {
      const int pp = q / tci, r = q - pp * tci, t = r / a.ci, i = r - t * a.ci;
      const int64_t ip = pp < np ? in_pixel(a, p0 + pp, t / a.k, t % a.k) : -1;
      xs[q] = ip >= 0 ? (float)x[ip * a.Ci + (int64_t)grp * a.ci + i] : 0.f;
    }
    __syncthreads();
    for (int pp = 0; pp < np; ++pp) {
      const float* dr = dys + pp * a.co;
      const float* xr = xs + pp * tci;
#pragma unroll
      for (int j = 0; j < kSmallJ; ++j)
        if (threadIdx.x + 256 * j < E) acc[j] = fmaf(dr[od[j]], xr[ox[j]], acc[j]);
    }
    __syncthreads();
  }
  float* out = part + ((int64_t)blockIdx.x * a.g + grp) * E;
#pragma unroll
  for (int j = 0; j < kSmallJ; ++j) {
    const int e = threadIdx.x + 256 * j;
    if (e < E) out[e] = acc[j];
  }
}

__global__ void __launch_bounds__(256) wgrad_reduce_simt(const float* __restrict__ part, WgArgs a,
                                                         float* __restrict__ dK) {
  const int64_t total = (int64_t)a.g * a.co * a.ci * a.kk;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int sp = 0; sp < a.splits; ++sp) acc += part[sp * total + e];
    const int o = (int)(e % a.co);
    int64_t r = e / a.co;
    const int i = (int)(r % a.ci); r /= a.ci;
    const int t = (int)(r % a.kk);
    const int grp = (int)(r / a.kk);
    dK[(((int64_t)grp * a.co + o) * a.ci + i) * a.kk + t] = acc;
  }
}

WgArgs make_args(const LayerInfo& L, int N, int H, int W, int Ho, int Wo) {
  WgArgs a{};
  a.N = N; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
  a.Ci = L.ci_f; a.Co = L.co_f; a.ci = L.ci; a.co = L.co; a.g = L.g;
  a.k = L.k; a.s = L.s; a.d = L.d; a.pt = L.pt; a.pl = L.pl;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  a.pixels = (int64_t)N * Ho * Wo;
  a.kk = L.k * L.k;
  return a;
}

bool tc_ok(const LayerInfo& L) { return L.ci % 8 == 0 && L.co % 8 == 0 && L.ci_f % 8 == 0 && L.co_f % 8 == 0; }

int pick_bn(const LayerInfo& L) { return L.ci > 128 ? 256 : L.ci > 64 ? 128 : 64; }
// taps per CTA (sharing the dy tile): 1 for 256-wide ci tiles (4 stages of 48 KB), else up to 3
// (BN = 128: 3 stages of 64 KB; BN = 64: 4 stages of 40 KB) -- one row of a 3 x 3 kernel
int pick_tpc(const LayerInfo& L) {
  const int bn = pick_bn(L);
  return bn == 256 ? 1 : std::min(3, L.k * L.k);
}

int wgrad_splits(const LayerInfo& L, int64_t pixels) {
  const int tpc = pick_tpc(L);
  const int64_t base = (int64_t)L.g * ((L.k * L.k + tpc - 1) / tpc) * ((L.co + 127) / 128) *
                       ((L.ci + pick_bn(L) - 1) / pick_bn(L));
  int64_t sp = std::max<int64_t>(1, (2 * 148 + base - 1) / base);        // ~2 waves of CTAs
  sp = std::min<int64_t>(sp, std::max<int64_t>(1, pixels / 512));       // >= 512 pixels per split
  return (int)std::min<int64_t>(sp, 64);
}

template <int BN, int TPC, int S>
int launch_tc(const __nv_bfloat16* x, const __nv_bfloat16* dy, const WgArgs& a, float* part, cudaStream_t s) {
  constexpr size_t STAGE = 2 * 8192 + (size_t)TPC * (BN / 64) * 8192;
  const size_t smem = 1024 + S * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(wgrad_tc<BN, TPC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t tiles = (int64_t)a.splits * a.g * a.tgroups * a.tiles_m * a.tiles_n;
  wgrad_tc<BN, TPC, S><<<(unsigned)tiles, kProd + 32, smem, s>>>(x, dy, a, part);
  return (int)cudaGetLastError();
}

int launch_tc_any(int bn, int tpc, const __nv_bfloat16* x, const __nv_bfloat16* dy, const WgArgs& a, float* part,
                  cudaStream_t s) {
  if (bn == 256) return launch_tc<256, 1, 4>(x, dy, a, part, s);
  if (bn == 128) {
    if (tpc >= 3) return launch_tc<128, 3, 3>(x, dy, a, part, s);
    if (tpc == 2) return launch_tc<128, 2, 3>(x, dy, a, part, s);
    return launch_tc<128, 1, 4>(x, dy, a, part, s);
  }
  if (tpc >= 3) return launch_tc<64, 3, 4>(x, dy, a, part, s);
  if (tpc == 2) return launch_tc<64, 2, 4>(x, dy, a, part, s);
  return launch_tc<64, 1, 4>(x, dy, a, part, s);
}

}  // namespace

// the small-kernel SIMT path: E <= 4096 elements per group, staging <= 96 KB
static bool small_ok(const LayerInfo& L) {
  return (int64_t)L.co * L.ci * L.k * L.k <= 256 * kSmallJ && (int64_t)kSmallP * (L.co + L.k * L.k * L.ci) * 4 <= 96 * 1024;
}
static int small_ctas(const LayerInfo& L, int64_t pixels) {
  const int64_t chunks = (pixels + kSmallP - 1) / kSmallP;
  return (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (8 * 148 + L.g - 1) / L.g));
}

// SIMT pixel splits: enough CTAs for ~4 waves, >= 64 pixels per split
static int simt_splits(const LayerInfo& L, int64_t pixels) {
  if (small_ok(L)) return small_ctas(L, pixels);
  const int64_t blocks = ((int64_t)L.g * L.co * L.ci * L.k * L.k + 255) / 256;
  int64_t sp = std::max<int64_t>(1, (4 * 148 + blocks - 1) / blocks);
  sp = std::min<int64_t>(sp, std::max<int64_t>(1, pixels / 64));
  return (int)std::min<int64_t>(sp, 4096);
}

int64_t wgrad_workspace_bytes(const LayerInfo& L, int N, int Ho, int Wo, int io) {
  const int64_t pixels = (int64_t)N * Ho * Wo;
  if (io != ORTH_BF16 || !tc_ok(L)) return simt_splits(L, pixels) > 1 ? (int64_t)simt_splits(L, pixels) * L.kernel_numel * 4 : 0;
  return (int64_t)wgrad_splits(L, pixels) * L.kernel_numel * 4;
}

int launch_wgrad(const LayerInfo& L, const void* x, const void* dy, float* dK, int N, int H, int W, int Ho, int Wo,
                 int io, void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  WgArgs a = make_args(L, N, H, W, Ho, Wo);
  const int64_t total = (int64_t)L.g * L.co * L.ci * a.kk;
  const int rb = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (io == ORTH_BF16 && tc_ok(L) && ws && ws_bytes >= wgrad_workspace_bytes(L, N, Ho, Wo, io)) {
    a.splits = wgrad_splits(L, a.pixels);
    a.per_split = ((a.pixels + a.splits - 1) / a.splits + 63) / 64 * 64;
    a.splits = (int)((a.pixels + a.per_split - 1) / a.per_split);
    const int bn = pick_bn(L);
    const int tpc = pick_tpc(L);
    a.tpc = tpc;
    a.tgroups = (a.kk + tpc - 1) / tpc;
    a.tiles_m = (L.co + 127) / 128;
    a.tiles_n = (L.ci + bn - 1) / bn;
    g_conv_variant = 0;
    float* part = static_cast<float*>(ws);
    int e = launch_tc_any(bn, tpc, (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, a, part, s);
    if (e) return e;
    wgrad_reduce<<<rb, 256, 0, s>>>(part, a, dK);
    return (int)cudaGetLastError();
  }
  g_conv_variant = ORTH_CV_SIMT;
  if (small_ok(L) && ws && ws_bytes >= wgrad_workspace_bytes(L, N, Ho, Wo, io)) {
    a.splits = small_ctas(L, a.pixels);
    const size_t smem = (size_t)kSmallP * (L.co + a.kk * L.ci) * 4;
    const dim3 grid((unsigned)a.splits, (unsigned)L.g);
    float* part = static_cast<float*>(ws);
    if (io == ORTH_BF16) {
      cudaFuncSetAttribute(wgrad_simt_small<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      wgrad_simt_small<__nv_bfloat16><<<grid, 256, smem, s>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, a, part);
    } else {
      cudaFuncSetAttribute(wgrad_simt_small<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      wgrad_simt_small<float><<<grid, 256, smem, s>>>((const float*)x, (const float*)dy, a, part);
    }
    wgrad_reduce_simt<<<rb, 256, 0, s>>>(part, a, dK);
    return (int)cudaGetLastError();
  }
  a.splits = simt_splits(L, a.pixels);
  if (a.splits > 1 && (!ws || ws_bytes < (int64_t)a.splits * L.kernel_numel * 4)) a.splits = 1;
  a.per_split = (a.pixels + a.splits - 1) / a.splits;
  a.splits = (int)((a.pixels + a.per_split - 1) / a.per_split);
  float* out = a.splits > 1 ? static_cast<float*>(ws) : dK;
  const dim3 grid((unsigned)((total + 255) / 256), (unsigned)a.splits);
  if (io == ORTH_BF16)
    wgrad_simt<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, a, out);
  else
    wgrad_simt<float><<<grid, 256, 0, s>>>((const float*)x, (const float*)dy, a, out);
  if (a.splits > 1) wgrad_reduce_simt<<<rb, 256, 0, s>>>(out, a, dK);
  return (int)cudaGetLastError();
}

}  // namespace orth
