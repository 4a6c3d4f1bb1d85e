// Bjorck / Newton-Schulz on the 5th-generation tensor cores (a3),
// residual form (reading R16):
//     R  = I - X^T X          (Gram on the short side, R4)
//     X' = X + beta * X R      (tall; wide: X + beta * R X)
// X is the FP32 master.  Every phase's epilogue also writes the BF16 (hi, and
// for the 3-pass split lo = bf16(x - hi)) copies the NEXT phase consumes:
// the Gram writes R (symmetric, so its rows are both operands' rows), the
// update writes X' row-major.  Operands that are columns of X (tall Gram
// A = B = X^T, wide update B = X) are loaded MN-major straight from the
// row-major copy, so no transposed copy exists.  Mainloop: TMA (SWIZZLE_128B)
// into a 3-stage ring, one thread issuing tcgen05.mma M=128 N=128 K=16 (x4 per
// 64-wide K block, x3 for the hi/lo split), FP32 accumulation in TMEM.
// Ragged batch: one flat tile list over all matrices of all layers
// (descriptors from plan.cpp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "orth_internal.h"
#include "pdl.h"
#include "umma.cuh"
#include "tma_host.h"

namespace orth {
namespace {

struct NsBufs {
  float* X[2];
  float* R;
  __nv_bfloat16 *xh[2], *xl[2], *rh, *rl;
  unsigned long long* trace;   // diagnostics (ORTH_NS_TRACE): 4 globaltimer stamps per CTA, else null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// select a[i] without dynamic indexing (which would move the parameter struct to local memory)
template <class T>
__device__ __forceinline__ T pick(T const (&a)[2], int i) { return i ? a[1] : a[0]; }

__device__ __forceinline__ int find_ns(const NsDesc* __restrict__ d, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {   // low half = a
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
// hi = bf16(x), lo = bf16(x - hi) for 4 values, packed into registers
__device__ __forceinline__ void split4(float a, float b, float c, float d, uint2& hi, uint2& lo) {
  hi.x = pack_bf16(a, b);
  hi.y = pack_bf16(c, d);
  const float ha = __uint_as_float(hi.x << 16), hb = __uint_as_float(hi.x & 0xFFFF0000u);
  const float hc = __uint_as_float(hi.y << 16), hd = __uint_as_float(hi.y & 0xFFFF0000u);
  lo.x = pack_bf16(a - ha, b - hb);
  lo.y = pack_bf16(c - hc, d - hd);
}

__device__ __forceinline__ void split(float x, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  l = __float2bfloat16_rn(x - __bfloat162float(h));
}

// One 128 (MN) x 64 (K) BF16 operand tile.  K-major: one 64 x 128 box.
// MN-major (columns of row-major X): two 64 (MN) x 64 (K) boxes, 8 KB apart.
__device__ __forceinline__ void load_operand(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int k0, int mn0,
                                             int kind) {
  if (kind == 3) {          // columns of row-major X, 3-D map (64 MN, K, MN / 64): both 64-wide blocks in one box
    umma::tma_load_3d(dst, map, bar, 0, k0, mn0 >> 6);
  } else if (kind == 1) {   // columns of row-major X: two 64 (MN) x 64 (K) boxes
    umma::tma_load_2d(dst, map, bar, mn0, k0);
    umma::tma_load_2d(dst + 8192, map, bar, mn0 + 64, k0);
  } else {                  // rows: one 64 (K) x 128 box
    umma::tma_load_2d(dst, map, bar, k0, mn0);
  }
}
// descriptor of the q-th K=16 slice of an operand tile
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int q, int mn_major) {
  return mn_major ? umma::sdesc_sw128_mn(base + 2048 * q, 8192) : umma::sdesc_sw128(base + 32 * q);
}

template <int NPASS, int S>
__global__ void __launch_bounds__(256, (NPASS == 1 ? 2 : 1))
    ns_tc_kernel(const NsDesc* __restrict__ descs, const int* __restrict__ tile_desc, NsBufs bufs, int par,
                 int write_lo, int write_f, const CUtensorMap* __restrict__ maps) {
  constexpr bool SPLIT = NPASS == 3;
  constexpr int TILE = 128 * 128;
  constexpr int STAGE = (SPLIT ? 4 : 2) * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t full_bar[S];
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (bufs.trace && tid == 0) bufs.trace[8 * blockIdx.x] = gtimer();
  const NsDesc d = descs[tile_desc[blockIdx.x]];   // host-built tile -> problem table (one load)
  const int local = blockIdx.x - d.tile_begin;
  const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;

  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, 128);
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&empty_bar[i], 1);
      umma::mbar_init(&full_bar[i], 1);
    }
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int a_mn = d.a_kind & 1, b_mn = d.b_kind & 1;   // operand = columns of row-major X: MN-major (kinds 1, 3)
  const uint32_t IDESC = umma::idesc_bf16(128, 128) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
  if (bufs.trace && tid == 0) bufs.trace[8 * blockIdx.x + 1] = gtimer();

  const int nk = (d.K + 63) / 64;
  if (tid == 0) {
    // ---- TMA producer: 128 x 64 BF16 boxes (SWIZZLE_128B, OOB -> 0) of A and B (hi, lo)
    const CUtensorMap* ma = maps + d.map_a + 2 * par;
    const CUtensorMap* mb = maps + d.map_b + 2 * par;
    constexpr uint32_t BYTES = (SPLIT ? 4 : 2) * TILE;
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const uint32_t sa = s0 + st * STAGE;
      umma::mbar_arrive_expect_tx(&full_bar[st], BYTES);
      load_operand(sa, ma, &full_bar[st], kb * 64, m0, d.a_kind);
      load_operand(sa + TILE, mb, &full_bar[st], kb * 64, n0, d.b_kind);
      if (SPLIT) {
        load_operand(sa + 2 * TILE, ma + 1, &full_bar[st], kb * 64, m0, d.a_kind);
        load_operand(sa + 3 * TILE, mb + 1, &full_bar[st], kb * 64, n0, d.b_kind);
      }
    }
  } else if (tid == 32) {
    // ---- MMA issuer
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      umma::mbar_wait(&full_bar[st], (kb / S) & 1);
      umma::tc_fence_after();
      const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t dah = op_desc(ah, q, a_mn), dbh = op_desc(bh, q, b_mn);
        umma::mma_bf16(tmem, dah, dbh, IDESC, (kb | q) != 0);
        if (SPLIT) {
          umma::mma_bf16(tmem, dah, op_desc(bl, q, b_mn), IDESC, 1);
          umma::mma_bf16(tmem, op_desc(al, q, a_mn), dbh, IDESC, 1);
        }
      }
      umma::mma_commit(&empty_bar[st]);
    }
    umma::mma_commit(&done_bar);
  }
  // Prefetch this thread's C fragments (previous X, update phase) into registers
  // while the MMAs run: 2 halves x 8 row-pass groups of 4 floats.
  float4 cpre[16];
  {
    const bool fv = (d.ldf & 3) == 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int h = u >> 3, e = tid + 256 * (u & 7), r = e >> 4, c4 = (e & 15) * 4;
      const int i = m0 + r, j0 = n0 + h * 64 + c4;
      cpre[u] = (d.epi == 1 && fv && i < d.M && j0 + 4 <= d.N)
                    ? __ldg(reinterpret_cast<const float4*>(bufs.X[0] + d.f_off + (int64_t)i * d.ldf + j0))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();
  if (bufs.trace && tid == 64) bufs.trace[8 * blockIdx.x + 2] = gtimer();

  // ---------------------------------------------------------------- epilogue
  // Two 64-column halves.  TMEM -> fp32 smem tile (row stride 68 floats: the
  // row-per-thread float4 writes and the row-wise float4 reads are both
  // conflict-free) -> one coalesced row pass (C in, D out as FP32, BF16 hi/lo
  // row copies).  The Gram's FP32 R is only written when asked (residual).
  // The operand ring is free once done_bar completed.
  const bool upd = d.epi == 1;
  const int ldb16 = upd ? d.ldx : d.ldr;   // padded row length of the row-major bf16 outputs
  __nv_bfloat16* oh = upd ? pick(bufs.xh, par ^ 1) + d.bx_off : bufs.rh + d.br_off;
  __nv_bfloat16* ol = upd ? pick(bufs.xl, par ^ 1) + d.bx_off : bufs.rl + d.br_off;
  float* F = upd ? bufs.X[0] + d.f_off : bufs.R + d.f_off;
  const float* Cm = bufs.X[0] + d.f_off;
  const bool wf = upd || write_f;
  constexpr int LDF = 68;
  float* Sf = reinterpret_cast<float*>(smem);                              // [128][68] fp32
  const bool fvec = (d.ldf & 3) == 0;      // 16-byte aligned fp32 rows
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    {
      const int q = warp & 3, sub = warp >> 2, r = q * 32 + lane;
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 64 + sub * 32), v);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        *reinterpret_cast<float4*>(Sf + r * LDF + sub * 32 + 4 * t) =
            make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
    }
    umma::tc_fence_before();
    __syncthreads();
    if (bufs.trace && tid == 0) bufs.trace[8 * blockIdx.x + 4 + 2 * h] = gtimer();
    // row pass: element group e -> (row r, 4 columns c4*4 .. +3)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + 256 * u;
      const int r = e >> 4, c4 = (e & 15) * 4;
      const int i = m0 + r, j0 = n0 + h * 64 + c4;
      float4 a = *reinterpret_cast<const float4*>(Sf + r * LDF + c4);
      float o[4] = {a.x, a.y, a.z, a.w};
      const bool row_ok = i < d.M;
      const int64_t fo = (int64_t)i * d.ldf + j0;
      if (row_ok && fvec && j0 + 4 <= d.N) {
        const float4 c = cpre[h * 8 + u];
        o[0] = fmaf(d.alpha, o[0], d.beta * c.x);
        o[1] = fmaf(d.alpha, o[1], d.beta * c.y);
        o[2] = fmaf(d.alpha, o[2], d.beta * c.z);
        o[3] = fmaf(d.alpha, o[3], d.beta * c.w);
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] += (i == j0 + k) ? d.diag : 0.f;
        if (wf) *reinterpret_cast<float4*>(F + fo) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (row_ok && j0 + k < d.N) {
            o[k] = fmaf(d.alpha, o[k], upd ? d.beta * __ldg(Cm + fo + k) : 0.f) + ((i == j0 + k) ? d.diag : 0.f);
            if (wf) F[fo + k] = o[k];
          } else {
            o[k] = 0.f;   // keeps every bf16 padding element zero
          }
        }
      }
      uint2 hv, lv;   // register-packed bf16 quads (no local arrays)
      split4(o[0], o[1], o[2], o[3], hv, lv);
      if (row_ok && j0 < ldb16) {   // ldb16 % 8 == 0 and j0 % 4 == 0: the 4-group is inside the padded row
        const int64_t bo = (int64_t)i * ldb16 + j0;
        *reinterpret_cast<uint2*>(oh + bo) = hv;
        if (write_lo) *reinterpret_cast<uint2*>(ol + bo) = lv;
      }
    }
    __syncthreads();
    if (bufs.trace && tid == 0) bufs.trace[8 * blockIdx.x + 5 + 2 * h] = gtimer();
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 128);
  if (bufs.trace && tid == 0) bufs.trace[8 * blockIdx.x + 3] = gtimer();
}

// X0 = W / sigma and its BF16 row copies (hi, and lo when the first Gram is
// 3-pass); padding columns [n, pad8(n)) of the BF16 rows are written as zero.
__global__ void __launch_bounds__(256) scale_bf16_kernel(const PowerItem* __restrict__ items,
                                                         const float* __restrict__ W, const float* __restrict__ sigma,
                                                         float* __restrict__ X0, NsBufs b, int par, int write_lo,
                                                         unsigned* __restrict__ bars, int nbars,
                                                         unsigned* __restrict__ power_bar_p) {
  umma::griddep_launch_dependents();
  umma::griddep_wait();   // PDL: the power kernel (sigma, and its barrier word re-armed below) is complete
  if (blockIdx.x == 0) {   // re-arm the persistent NS group barriers and the fused power kernel's barrier
    for (int i = threadIdx.x; i < nbars; i += 256) bars[i] = 0u;
    if (threadIdx.x == 0) *power_bar_p = 0u;
  }
  const PowerItem it = items[blockIdx.x];
  const float inv = 1.f / sigma[it.mat];
  const int n = it.n, ldx = (n + 7) & ~7, g4 = ldx >> 2;
  __nv_bfloat16* xh = pick(b.xh, par) + it.bx_off;
  __nv_bfloat16* xl = pick(b.xl, par) + it.bx_off;
  const bool vec = (n & 3) == 0;
  const int64_t total = (int64_t)(it.r1 - it.r0) * g4;
  for (int64_t e = threadIdx.x; e < total; e += 256) {
    const int r = it.r0 + (int)(e / g4), c = (int)(e % g4) * 4;
    const int64_t fo = it.off + (int64_t)r * n + c;
    float x[4];
    if (vec && c < n) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(W + fo));
      x[0] = w.x * inv; x[1] = w.y * inv; x[2] = w.z * inv; x[3] = w.w * inv;
      *reinterpret_cast<float4*>(X0 + fo) = make_float4(x[0], x[1], x[2], x[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x[k] = c + k < n ? __ldg(W + fo + k) * inv : 0.f;
        if (c + k < n) X0[fo + k] = x[k];
      }
    }
    uint2 hv, lv;
    split4(x[0], x[1], x[2], x[3], hv, lv);
    const int64_t bo = (int64_t)r * ldx + c;
    *reinterpret_cast<uint2*>(xh + bo) = hv;
    if (write_lo) *reinterpret_cast<uint2*>(xl + bo) = lv;
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
  }
  auto br = reinterpret_cast<__nv_bfloat16*>(p.d_br);
  b.rh = br;
  b.rl = br + (p.br_numel > 64 ? p.br_numel : 64);
  b.trace = nullptr;
  return b;
}

template <int NPASS, int S>
int launch_impl(const NsDesc* d, const int* td, int tiles, NsBufs b, int par, int write_lo, int write_f,
                const CUtensorMap* maps, cudaStream_t s) {
  constexpr int STAGE = (NPASS == 3 ? 4 : 2) * 128 * 128;
  const size_t smem = 1024 + (size_t)(S * STAGE > 128 * 129 * 4 ? S * STAGE : 128 * 129 * 4);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ns_tc_kernel<NPASS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ns_tc_kernel<NPASS, S><<<tiles, 256, smem, s>>>(d, td, b, par, write_lo, write_f, maps);
  return (int)cudaGetLastError();
}

}  // namespace

// One 2-D map per (matrix operand, parity, hi/lo) over the row-major BF16
// copy, row stride = padded row length, SWIZZLE_128B.  K-major operands (rows
// of X or R): dims (K, rows), box 64 x 128.  MN-major operands (columns of X):
// dims (n, m) of X itself, box 64 x 64.
orth_status_t build_ns_tma(Plan& p) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ORTH_ERR_CUDA;
  }
  float* fake[BUF_COUNT] = {nullptr, nullptr, nullptr, nullptr};
  NsBufs b = make_bufs(p, fake);
  std::vector<CUtensorMap> maps;
  auto add4 = [&](int kind, int64_t off, int64_t K, int64_t rows, int64_t ld) {
    const int base = (int)maps.size();
    for (int par = 0; par < 2; ++par)
      for (int lo = 0; lo < 2; ++lo) {
        const __nv_bfloat16* ptr = (kind == 2 ? (lo ? b.rl : b.rh) : (lo ? b.xl[par] : b.xh[par])) + off;
        CUtensorMap m;
        std::memset(&m, 0, sizeof(m));
        if (kind == 3) {   // MN-major, 3-D (64 columns, K rows, column blocks): a 128-wide operand in one box
          const cuuint64_t dims3[3] = {64, (cuuint64_t)K, (cuuint64_t)(rows / 64)};
          const cuuint64_t strides3[2] = {(cuuint64_t)ld * 2, 128};
          const cuuint32_t box3[3] = {64, 64, 2};
          const cuuint32_t es3[3] = {1, 1, 1};
          if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(ptr), dims3, strides3, box3,
                  es3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return -1;
          maps.push_back(m);
          continue;
        }
        // MN-major: inner dim = the operand's MN extent (columns of X), outer = K (rows of X)
        const cuuint64_t dims[2] = {(cuuint64_t)(kind == 1 ? rows : K), (cuuint64_t)(kind == 1 ? K : rows)};
        const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
        const cuuint32_t box[2] = {64, kind == 1 ? 64u : 128u};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(ptr), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return -1;
        maps.push_back(m);
      }
    return base;
  };
  // Gram operands that are columns of X (kind 1) with a 64-multiple extent load through a 3-D map (kind 3:
  // one TMA per operand and K block instead of two; the issuing thread pays ~90 cycles per TMA, measured
  // by tools/micro/tma_ld_bw.cu).  Update operands keep 2-D maps (their 64-wide tiles load one block).
  static const bool no3d = std::getenv("ORTH_NS_NO_TMA3D") != nullptr;   // A/B switch
  for (auto& d : p.ns_gram) {
    if (no3d) break;
    if (d.a_kind == 1 && d.M % 64 == 0) d.a_kind = 3;
    if (d.b_kind == 1 && d.N % 64 == 0) d.b_kind = 3;
  }
  auto operand_map = [&](const NsDesc& d, bool a) {
    const int kind = a ? d.a_kind : d.b_kind;
    const int64_t off = a ? d.a_off : d.b_off, ld = a ? d.lda : d.ldb;
    const int64_t rows = a ? d.M : d.N;
    return add4(kind, off, d.K, rows, ld);
  };
  for (auto* v : {&p.ns_gram, &p.ns_upd})
    for (auto& d : *v) {
      d.map_a = operand_map(d, true);
      d.map_b = operand_map(d, false);
      if (d.map_a < 0 || d.map_b < 0) {
        set_error("tensor map encoding failed for an NS operand");
        return ORTH_ERR_CUDA;
      }
    }
  if (maps.empty()) return ORTH_OK;
  std::vector<int> tg, tu;   // tile -> problem tables
  for (int i = 0; i < (int)p.ns_gram.size(); ++i) {
    const NsDesc& d = p.ns_gram[i];
    for (int t = 0; t < ((d.M + 127) / 128) * d.tiles_n; ++t) tg.push_back(i);
  }
  for (int i = 0; i < (int)p.ns_upd.size(); ++i) {
    const NsDesc& d = p.ns_upd[i];
    for (int t = 0; t < ((d.M + 127) / 128) * d.tiles_n; ++t) tu.push_back(i);
  }
  const size_t mbytes = maps.size() * sizeof(CUtensorMap);
  cudaError_t e = cudaMalloc(&p.d_ns_maps, mbytes + (tg.size() + tu.size()) * sizeof(int));
  if (e == cudaSuccess)
    e = cudaMemcpy(p.d_ns_maps, maps.data(), mbytes, cudaMemcpyHostToDevice);
  p.d_ns_tile_gram = reinterpret_cast<int*>(static_cast<char*>(p.d_ns_maps) + mbytes);
  p.d_ns_tile_upd = p.d_ns_tile_gram + tg.size();
  if (e == cudaSuccess && !tg.empty())
    e = cudaMemcpy(p.d_ns_tile_gram, tg.data(), tg.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !tu.empty())
    e = cudaMemcpy(p.d_ns_tile_upd, tu.data(), tu.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.ns_gram.empty())
    e = cudaMemcpy(p.d_ns_gram, p.ns_gram.data(), p.ns_gram.size() * sizeof(NsDesc), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.ns_upd.empty())
    e = cudaMemcpy(p.d_ns_upd, p.ns_upd.data(), p.ns_upd.size() * sizeof(NsDesc), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error("NS tensor map upload failed: %s", cudaGetErrorString(e));
    return ORTH_ERR_CUDA;
  }
  return ORTH_OK;
}

int launch_ns_tc(Plan& p, float* const bufs[BUF_COUNT], int par, bool gram, int npass, bool write_lo, bool write_f,
                 void* stream) {
  const int tiles = gram ? p.ns_gram_tiles : p.ns_upd_tiles;
  if (tiles == 0) return 0;
  const NsDesc* d = gram ? p.d_ns_gram : p.d_ns_upd;
  const int nd = (int)(gram ? p.ns_gram.size() : p.ns_upd.size());
  NsBufs b = make_bufs(p, bufs);
  p.launches++;
  auto maps = reinterpret_cast<const CUtensorMap*>(p.d_ns_maps);
  const int* td = gram ? p.d_ns_tile_gram : p.d_ns_tile_upd;
  (void)nd;
  static unsigned long long* trace = nullptr;
  static const bool tracing = std::getenv("ORTH_NS_TRACE") != nullptr;
  if (tracing) {   // diagnostics only: serialises the stream and prints a per-launch summary
    if (!trace) cudaMalloc(&trace, 4096 * 8 * sizeof(unsigned long long));
    b.trace = trace;
  }
  const int e = npass == 3 ? launch_impl<3, 3>(d, td, tiles, b, par, write_lo, write_f, maps, (cudaStream_t)stream)
                           : launch_impl<1, 3>(d, td, tiles, b, par, write_lo, write_f, maps, (cudaStream_t)stream);
  if (tracing && !e) {
    std::vector<unsigned long long> h((size_t)tiles * 8);
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t3 = 0;
    double setup = 0, mainl = 0, epi = 0, mx_main = 0, last_start = 0;
    double ep[4] = {0, 0, 0, 0};
    for (int i = 0; i < tiles; ++i) t0 = std::min(t0, h[8 * i]);
    for (int i = 0; i < tiles; ++i) {
      const unsigned long long* q = &h[8 * i];
      ep[0] += q[4] - q[2]; ep[1] += q[5] - q[4]; ep[2] += q[6] - q[5]; ep[3] += q[7] - q[6];
      t3 = std::max(t3, q[3]);
      setup += q[1] - q[0]; mainl += q[2] - q[1]; epi += q[3] - q[2];
      mx_main = std::max(mx_main, (double)(q[2] - q[1]));
      last_start = std::max(last_start, (double)(q[0] - t0));
    }
    std::printf("ns_tc %s npass=%d tiles=%d span=%.2fus setup=%.2f main=%.2f (max %.2f) epi=%.2f [ld0 %.2f row0 %.2f tr0+ld1 %.2f row1 %.2f] last_start=%.2f\n",
                gram ? "gram" : "upd ", npass, tiles, (t3 - t0) * 1e-3, setup / tiles * 1e-3, mainl / tiles * 1e-3,
                mx_main * 1e-3, epi / tiles * 1e-3, ep[0] / tiles * 1e-3, ep[1] / tiles * 1e-3, ep[2] / tiles * 1e-3,
                ep[3] / tiles * 1e-3, last_start * 1e-3);
  }
  return e;
}

int launch_scale_bf16(Plan& p, const float* W, float* X0, int par, bool write_lo, void* stream) {
  if (p.power_items.empty()) return 0;
  float* bufs[BUF_COUNT] = {X0, X0, nullptr, nullptr};
  NsBufs b = make_bufs(p, bufs);
  launch_pdl(scale_bf16_kernel, dim3((unsigned)p.power_items.size()), dim3(256), 0, (cudaStream_t)stream,
             (const PowerItem*)p.d_power_items, W, (const float*)p.d_sigma, X0, b, par, (int)write_lo, p.nsp_bars,
             p.nsp_bars ? p.nsp_zero_n : 0, power_bar(p));
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
