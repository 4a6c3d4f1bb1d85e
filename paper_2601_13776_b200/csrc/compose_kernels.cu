// a5 emit: copy each (layer, group) kernel from its construction buffer into
// (1) the FP32 PyTorch weight layout (C_o, C_i/g, k, k) and (2) the BF16
// GEMM layout (C_o, k, k, C_i/g) used by the conv kernels (RNE rounding, R16).
// Sources: tap-major chain/AOC results (slice [:co, :ci] of width ld, P:321
// BCOP slicing, R5) or the RKO reshape R.reshape(co, ci, s, s) (R7).
//
// CTA = output rows o = blockIdx.x + k gridDim.x of item blockIdx.y; thread =
// input channel i: reads the k^2 taps of (o, i) (coalesced across i), writes
// the BF16 GEMM row [o][t][i] (coalesced) and the FP32 PyTorch row [o][i][t]
// (k^2 consecutive floats per thread, contiguous across the warp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"
#include "pdl.h"
#include "umma.cuh"

namespace orth {
namespace {

__global__ void __launch_bounds__(128) emit_kernel(const EmitItem* __restrict__ items, const float* b0,
                                                   const float* b1, const float* b2, const float* b3,
                                                   float* __restrict__ kf32, __nv_bfloat16* __restrict__ kbf16) {
  extern __shared__ float row_sm[];   // one FP32 output row [i][t] (k^2 ci floats)
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const EmitItem e = items[blockIdx.y];
  const float* base = e.src_buf == 0 ? b0 : e.src_buf == 1 ? b1 : e.src_buf == 2 ? b2 : b3;
  const float* src = base + e.src_off;
  const int kk = e.k * e.k, ci = e.ci;
  const int slab = kk * ci;
  for (int o = blockIdx.x; o < e.co; o += gridDim.x) {
    float* f = kf32 + e.f32_off + (int64_t)o * slab;
    __nv_bfloat16* bq = kbf16 ? kbf16 + e.bf16_off + (int64_t)o * slab : nullptr;
    if (e.mode == 2) {   // tap-major without the shared-memory row stage (large k^2 ci rows: SOC E)
      for (int i = threadIdx.x; i < ci; i += 128) {
        const float* col = src + (int64_t)o * e.ld + i;
        for (int t = 0; t < kk; ++t) {
          const float v = __ldg(col + (int64_t)t * e.tap_stride);
          f[(int64_t)i * kk + t] = v;
          if (bq) bq[(int64_t)t * ci + i] = __float2bfloat16_rn(v);
        }
      }
      continue;
    }
    if (e.mode == 1) {   // RKO: K[o, i, t] = R[o, i*s^2 + t] (k = s): the FP32 row is a straight copy
      const float* row = src + (int64_t)o * slab;
      for (int x = threadIdx.x; x < slab; x += 128) f[x] = __ldg(row + x);
      if (bq)
        for (int i = threadIdx.x; i < ci; i += 128)
          for (int t = 0; t < kk; ++t) bq[(int64_t)t * ci + i] = __float2bfloat16_rn(__ldg(row + i * kk + t));
      continue;
    }
    // tap-major: K[o, i, t] = src[t*tap_stride + o*ld + i]; stage [i][t] (stride k^2, odd -> conflict-free)
    __syncthreads();
    if ((ci & 1) == 0 && kk <= 16) {   // channel pairs, all taps' loads in flight before use
      for (int i = 2 * threadIdx.x; i < ci; i += 256) {
        const float* col = src + (int64_t)o * e.ld + i;
        float2 v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < kk) v[t] = make_float2(__ldg(col + (int64_t)t * e.tap_stride), __ldg(col + (int64_t)t * e.tap_stride + 1));
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < kk) {
            row_sm[i * kk + t] = v[t].x;
            row_sm[(i + 1) * kk + t] = v[t].y;
            if (bq) *reinterpret_cast<__nv_bfloat162*>(bq + (int64_t)t * ci + i) = __floats2bfloat162_rn(v[t].x, v[t].y);
          }
      }
    } else if ((ci & 1) == 0) {   // channel pairs: one 4-byte BF16x2 store per (tap, pair)
      for (int i = 2 * threadIdx.x; i < ci; i += 256) {
        const float* col = src + (int64_t)o * e.ld + i;
        for (int t = 0; t < kk; ++t) {
          const float v0 = __ldg(col + (int64_t)t * e.tap_stride), v1 = __ldg(col + (int64_t)t * e.tap_stride + 1);
          row_sm[i * kk + t] = v0;
          row_sm[(i + 1) * kk + t] = v1;
          if (bq) *reinterpret_cast<__nv_bfloat162*>(bq + (int64_t)t * ci + i) = __floats2bfloat162_rn(v0, v1);
        }
      }
    } else {
      for (int i = threadIdx.x; i < ci; i += 128) {
        const float* col = src + (int64_t)o * e.ld + i;
        for (int t = 0; t < kk; ++t) {
          const float v = __ldg(col + (int64_t)t * e.tap_stride);
          row_sm[i * kk + t] = v;
          if (bq) bq[(int64_t)t * ci + i] = __float2bfloat16_rn(v);
        }
      }
    }
    __syncthreads();
    if ((slab & 3) == 0 && ((reinterpret_cast<uintptr_t>(f) & 15) == 0)) {
      for (int x = threadIdx.x; x < slab / 4; x += 128)
        reinterpret_cast<float4*>(f)[x] = reinterpret_cast<const float4*>(row_sm)[x];
    } else {
      for (int x = threadIdx.x; x < slab; x += 128) f[x] = row_sm[x];
    }
  }
}

}  // namespace

int launch_emit_list(Plan& p, const std::vector<EmitItem>& items, const EmitItem* d_items,
                     const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream) {
  if (items.empty()) return 0;
  int maxco = 1;
  size_t smem = 16;
  for (auto& e : items) {
    maxco = e.co > maxco ? e.co : maxco;
    if (e.mode != 2) smem = std::max(smem, (size_t)e.k * e.k * e.ci * sizeof(float));
  }
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  dim3 grid((unsigned)(maxco < 256 ? maxco : 256), (unsigned)items.size());
  launch_pdl(emit_kernel, grid, dim3(128), smem, (cudaStream_t)stream, d_items,
             (const float*)bufs[0], (const float*)bufs[1], (const float*)bufs[2], (const float*)bufs[3], kf32,
             reinterpret_cast<__nv_bfloat16*>(kbf16));
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_emit(Plan& p, const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream) {
  return launch_emit_list(p, p.emit, p.d_emit, bufs, kf32, kbf16, stream);
}


namespace {
// a8: one CTA row per unit (blockIdx.y), CTAs along x stride the unit's elements; 16-byte vectors when
// both the source and destination run are 16-byte aligned (always for the padded gather side; for the
// final side when the unit's numel keeps the alignment), else element copies.
__global__ void __launch_bounds__(256) assemble_kernel(const UnitInfo* __restrict__ units, const float* __restrict__ gf,
                                                       float* __restrict__ kf, const uint16_t* __restrict__ gb,
                                                       uint16_t* __restrict__ kb) {
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const UnitInfo u = units[blockIdx.y];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gf) {
    const float* src = gf + u.gat_f32;
    float* dst = kf + u.fin_f32;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
      const int64_t nv = u.numel / 4;
      for (int64_t e = t0; e < nv; e += stride) reinterpret_cast<float4*>(dst)[e] = reinterpret_cast<const float4*>(src)[e];
      for (int64_t e = nv * 4 + t0; e < u.numel; e += stride) dst[e] = src[e];
    } else {
      for (int64_t e = t0; e < u.numel; e += stride) dst[e] = src[e];
    }
  }
  if (gb) {
    const uint16_t* src = gb + u.gat_bf16;
    uint16_t* dst = kb + u.fin_bf16;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
      const int64_t nv = u.numel / 8;
      for (int64_t e = t0; e < nv; e += stride) reinterpret_cast<uint4*>(dst)[e] = reinterpret_cast<const uint4*>(src)[e];
      for (int64_t e = nv * 8 + t0; e < u.numel; e += stride) dst[e] = src[e];
    } else {
      for (int64_t e = t0; e < u.numel; e += stride) dst[e] = src[e];
    }
  }
}
}  // namespace

int launch_assemble(Plan& p, const float* gf, float* kf, const uint16_t* gb, uint16_t* kb, void* stream) {
  if (p.units.empty() || (!gf && !gb)) return 0;
  int64_t maxn = 1;
  for (auto& u : p.units) maxn = std::max(maxn, u.numel);
  // ~4 x 148 CTAs in total across units, at least one per unit
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>((maxn / 4 + 255) / 256, 592 / (int64_t)p.units.size() + 1));
  launch_pdl(assemble_kernel, dim3((unsigned)per, (unsigned)p.units.size()), dim3(256), 0, (cudaStream_t)stream,
             (const UnitInfo*)p.d_units, gf, kf, gb, kb);
  return (int)cudaGetLastError();
}

}  // namespace orth
