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
#include <cstring>
#include <vector>

#include "orth_internal.h"
#include "umma.cuh"
#include "tma_host.h"

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
    ns_tc_kernel(const NsDesc* __restrict__ descs, const int* __restrict__ tile_desc, NsBufs bufs, int par,
                 int write_lo, const CUtensorMap* __restrict__ maps) {
  constexpr bool SPLIT = NPASS == 3;
  constexpr int TILE = 128 * 128;
  constexpr int STAGE = (SPLIT ? 4 : 2) * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[S];
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
  constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);

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
      umma::tma_load_2d(sa, ma, &full_bar[st], kb * 64, m0);
      umma::tma_load_2d(sa + TILE, mb, &full_bar[st], kb * 64, n0);
      if (SPLIT) {
        umma::tma_load_2d(sa + 2 * TILE, ma + 1, &full_bar[st], kb * 64, m0);
        umma::tma_load_2d(sa + 3 * TILE, mb + 1, &full_bar[st], kb * 64, n0);
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
        umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, (kb | q) != 0);
        if (SPLIT) {
          umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
          umma::mma_bf16(tmem, umma::sdesc_sw128(al + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, 1);
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
                    ? __ldg(reinterpret_cast<const float4*>(bufs.X[par] + d.f_off + (int64_t)i * d.ldf + j0))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();

  // ---------------------------------------------------------------- epilogue
  // Two 64-column halves.  TMEM -> fp32 smem tile (row stride 68 floats: the
  // row-per-thread float4 writes and the row-wise float4 reads are both
  // conflict-free) -> one coalesced row pass (C in, D out as FP32, BF16 hi/lo
  // row copies) that also stages the BF16 transpose -> one coalesced pass of
  // X'^T rows (update phase only).  The operand ring is free once done_bar completed.
  const bool upd = d.epi == 1;
  const int ldb16 = upd ? d.ldx : d.ldr;   // padded row length of the row-major bf16 outputs
  __nv_bfloat16* oh = upd ? bufs.xh[par ^ 1] + d.bx_off : bufs.rh + d.br_off;
  __nv_bfloat16* ol = upd ? bufs.xl[par ^ 1] + d.bx_off : bufs.rl + d.br_off;
  float* F = upd ? bufs.X[par ^ 1] + d.f_off : bufs.R + d.f_off;
  const float* Cm = bufs.X[par] + d.f_off;
  __nv_bfloat16* th = bufs.th[par ^ 1] + d.bx_off;
  __nv_bfloat16* tl = bufs.tl[par ^ 1] + d.bx_off;
  constexpr int LDF = 68, LDT = 136;
  float* Sf = reinterpret_cast<float*>(smem);                              // [128][68] fp32
  __nv_bfloat16* sTh = reinterpret_cast<__nv_bfloat16*>(smem + 128 * LDF * 4);   // [64][136] bf16
  __nv_bfloat16* sTl = sTh + 64 * LDT;
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
        *reinterpret_cast<float4*>(F + fo) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (row_ok && j0 + k < d.N) {
            o[k] = fmaf(d.alpha, o[k], upd ? d.beta * __ldg(Cm + fo + k) : 0.f) + ((i == j0 + k) ? d.diag : 0.f);
            F[fo + k] = o[k];
          } else {
            o[k] = 0.f;   // keeps every bf16 padding element zero
          }
        }
      }
      __nv_bfloat16 hb[4], lb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) split(o[k], hb[k], lb[k]);
      if (row_ok && j0 < ldb16) {   // ldb16 % 8 == 0 and j0 % 4 == 0: the 4-group is inside the padded row
        const int64_t bo = (int64_t)i * ldb16 + j0;
        *reinterpret_cast<uint2*>(oh + bo) = *reinterpret_cast<const uint2*>(hb);
        if (write_lo) *reinterpret_cast<uint2*>(ol + bo) = *reinterpret_cast<const uint2*>(lb);
      }
      if (upd) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sTh[(c4 + k) * LDT + r] = hb[k];
          if (write_lo) sTl[(c4 + k) * LDT + r] = lb[k];
        }
      }
    }
    __syncthreads();
    if (upd) {   // rows of X'^T: 16-byte chunks along i
      for (int e = tid; e < 64 * 16; e += 256) {
        const int cl = e >> 4, i8 = (e & 15) * 8;
        const int j = n0 + h * 64 + cl, i0 = m0 + i8;
        if (j < d.N && i0 < d.ldxt) {
          const int64_t o = (int64_t)j * d.ldxt + i0;
          *reinterpret_cast<uint4*>(th + o) = *reinterpret_cast<const uint4*>(sTh + cl * LDT + i8);
          if (write_lo) *reinterpret_cast<uint4*>(tl + o) = *reinterpret_cast<const uint4*>(sTl + cl * LDT + i8);
        }
      }
      __syncthreads();
    }
  }
  umma::tc_fence_before();
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
int launch_impl(const NsDesc* d, const int* td, int tiles, NsBufs b, int par, int write_lo, const CUtensorMap* maps,
                cudaStream_t s) {
  constexpr int STAGE = (NPASS == 3 ? 4 : 2) * 128 * 128;
  const size_t smem = 1024 + (size_t)(S * STAGE > 128 * 129 * 4 ? S * STAGE : 128 * 129 * 4);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ns_tc_kernel<NPASS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  ns_tc_kernel<NPASS, S><<<tiles, 256, smem, s>>>(d, td, b, par, write_lo, maps);
  return (int)cudaGetLastError();
}

}  // namespace

// One 2-D map per (matrix, operand kind, parity, hi/lo): dims (K, rows), row
// stride = padded row length; box 64 x 128, SWIZZLE_128B.
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
        const __nv_bfloat16* ptr = (kind == 0 ? (lo ? b.xl[par] : b.xh[par])
                                    : kind == 1 ? (lo ? b.tl[par] : b.th[par])
                                                : (lo ? b.rl : b.rh)) + off;
        CUtensorMap m;
        std::memset(&m, 0, sizeof(m));
        const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
        const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
        const cuuint32_t box[2] = {64, 128};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(ptr), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return -1;
        maps.push_back(m);
      }
    return base;
  };
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

int launch_ns_tc(Plan& p, float* const bufs[BUF_COUNT], int par, bool gram, int npass, bool write_lo, void* stream) {
  const int tiles = gram ? p.ns_gram_tiles : p.ns_upd_tiles;
  if (tiles == 0) return 0;
  const NsDesc* d = gram ? p.d_ns_gram : p.d_ns_upd;
  const int nd = (int)(gram ? p.ns_gram.size() : p.ns_upd.size());
  NsBufs b = make_bufs(p, bufs);
  p.launches++;
  auto maps = reinterpret_cast<const CUtensorMap*>(p.d_ns_maps);
  const int* td = gram ? p.d_ns_tile_gram : p.d_ns_tile_upd;
  (void)nd;
  if (npass == 3) return launch_impl<3, 3>(d, td, tiles, b, par, write_lo, maps, (cudaStream_t)stream);
  return launch_impl<1, 3>(d, td, tiles, b, par, write_lo, maps, (cudaStream_t)stream);
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
