// a5 emit: copy each (layer, group) kernel from its construction buffer into
// (1) the FP32 PyTorch weight layout (C_o, C_i/g, k, k) and (2) the BF16
// GEMM layout (C_o, k, k, C_i/g) used by the conv kernels (RNE rounding, R16).
// Sources: tap-major chain/AOC results (slice [:co, :ci] of width ld, P:321
// BCOP slicing, R5) or the RKO reshape R.reshape(co, ci, s, s) (R7).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

__device__ __forceinline__ float emit_src(const EmitItem& e, const float* src, int o, int i, int p, int q) {
  if (e.mode == 1) {
    const int s = e.s;
    return src[(int64_t)o * e.ci * s * s + (int64_t)i * s * s + p * s + q];
  }
  return src[(int64_t)(p * e.k + q) * e.tap_stride + (int64_t)o * e.ld + i];
}

__global__ void __launch_bounds__(256) emit_kernel(const EmitItem* __restrict__ items, const float* b0,
                                                   const float* b1, const float* b2, const float* b3,
                                                   float* __restrict__ kf32, __nv_bfloat16* __restrict__ kbf16) {
  const EmitItem e = items[blockIdx.y];
  const float* bufs[4] = {b0, b1, b2, b3};
  const float* src = bufs[e.src_buf] + e.src_off;
  const int k = e.k, kk = k * k;
  const int64_t total = (int64_t)e.co * e.ci * kk;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += step) {
    // canonical (o, i, p, q)
    {
      const int q = (int)(x % k), p = (int)((x / k) % k);
      const int i = (int)((x / kk) % e.ci), o = (int)(x / ((int64_t)kk * e.ci));
      kf32[e.f32_off + x] = emit_src(e, src, o, i, p, q);
    }
    if (kbf16) {  // GEMM order (o, p, q, i)
      const int i = (int)(x % e.ci);
      const int t = (int)((x / e.ci) % kk);
      const int o = (int)(x / ((int64_t)kk * e.ci));
      kbf16[e.bf16_off + x] = __float2bfloat16_rn(emit_src(e, src, o, i, t / k, t % k));
    }
  }
}

}  // namespace

int launch_emit(Plan& p, const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream) {
  if (p.emit.empty()) return 0;
  int64_t maxn = 1;
  for (auto& e : p.emit) {
    const int64_t t = (int64_t)e.co * e.ci * e.k * e.k;
    maxn = t > maxn ? t : maxn;
  }
  int bx = (int)((maxn + 255) / 256);
  bx = bx > 64 ? 64 : bx;
  dim3 grid(bx, (unsigned)p.emit.size());
  emit_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p.d_emit, bufs[0], bufs[1], bufs[2], bufs[3], kf32,
                                                      reinterpret_cast<__nv_bfloat16*>(kbf16));
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
