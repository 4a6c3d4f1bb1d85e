// a5 emit: copy each (layer, group) kernel from its construction buffer into
// (1) the FP32 PyTorch weight layout (C_o, C_i/g, k, k) and (2) the BF16
// GEMM layout (C_o, k, k, C_i/g) used by the conv kernels (RNE rounding, R16).
// Sources: tap-major chain/AOC results (slice [:co, :ci] of width ld, P:321
// BCOP slicing, R5) or the RKO reshape R.reshape(co, ci, s, s) (R7).
//
// One output row o per iteration: the row's k^2 x ci slab is staged in shared
// memory (coalesced reads along ci), then written coalesced in both layouts.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

__global__ void __launch_bounds__(256) emit_kernel(const EmitItem* __restrict__ items, const float* b0,
                                                   const float* b1, const float* b2, const float* b3,
                                                   float* __restrict__ kf32, __nv_bfloat16* __restrict__ kbf16) {
  extern __shared__ float buf[];   // [k^2][ci + 1]
  const EmitItem e = items[blockIdx.y];
  const float* bufs[4] = {b0, b1, b2, b3};
  const float* src = bufs[e.src_buf] + e.src_off;
  const int kk = e.k * e.k, ci = e.ci, ld1 = ci + 1;
  const int slab = kk * ci;
  for (int o = blockIdx.x; o < e.co; o += gridDim.x) {
    if (e.mode == 1) {   // RKO: K[o, i, t] = R[o, i*s^2 + t]  (k = s)
      const float* row = src + (int64_t)o * slab;
      for (int x = threadIdx.x; x < slab; x += blockDim.x) buf[(x % kk) * ld1 + x / kk] = row[x];
    } else {             // tap-major: K[o, i, t] = src[t*tap_stride + o*ld + i]
      for (int x = threadIdx.x; x < slab; x += blockDim.x) {
        const int t = x / ci, i = x % ci;
        buf[t * ld1 + i] = src[(int64_t)t * e.tap_stride + (int64_t)o * e.ld + i];
      }
    }
    __syncthreads();
    float* f = kf32 + e.f32_off + (int64_t)o * slab;
    for (int x = threadIdx.x; x < slab; x += blockDim.x) f[x] = buf[(x % kk) * ld1 + x / kk];   // (i, t)
    if (kbf16) {
      __nv_bfloat16* b = kbf16 + e.bf16_off + (int64_t)o * slab;
      for (int x = threadIdx.x; x < slab; x += blockDim.x) b[x] = __float2bfloat16_rn(buf[(x / ci) * ld1 + x % ci]);
    }
    __syncthreads();
  }
}

}  // namespace

int launch_emit(Plan& p, const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream) {
  if (p.emit.empty()) return 0;
  int maxco = 1;
  size_t smem = 0;
  for (auto& e : p.emit) {
    maxco = e.co > maxco ? e.co : maxco;
    const size_t s = (size_t)e.k * e.k * (e.ci + 1) * sizeof(float);
    smem = s > smem ? s : smem;
  }
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  dim3 grid((unsigned)(maxco < 128 ? maxco : 128), (unsigned)p.emit.size());
  emit_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(p.d_emit, bufs[0], bufs[1], bufs[2], bufs[3], kf32,
                                                         reinterpret_cast<__nv_bfloat16*>(kbf16));
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
