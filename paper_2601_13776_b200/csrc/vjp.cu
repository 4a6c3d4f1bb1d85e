// f1: the gradient moves of the composition VJP (the GEMMs
// are GemmPhases built in plan.cpp build_vjp).
//   vjp_deemit_kernel: the final-layout FP32 dK of every owned unit into the VJP
//     layout -- the chain's last-step gradient dS (rows x c taps, zero outside
//     the [:co, :ci] slice: the slice's adjoint is zero padding) or the AOC
//     output gradient dFin (tap-major), or straight into d_ortho for RKO /
//     dense units (the reshape's adjoint is the inverse reshape) and k' = 1 BCOP
//     (dQ[:co, :ci] = dK); dQ of chain units is zeroed first (rows >= r).
//   vjp_scatter_kernel: AOC dR[o][j s^2 + t] = dRab[t][o][j] (the RKO reshape).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

__global__ void __launch_bounds__(256) vjp_deemit_kernel(const VjpItem* __restrict__ items, const float* __restrict__ dK,
                                                         float* __restrict__ arena, float* __restrict__ dortho) {
  const VjpItem it = items[blockIdx.y];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float* src = dK + it.src_off;
  if (it.mode == 2) {   // RKO / dense: identical memory order
    const int64_t n = (int64_t)it.co * it.ci * it.kk;
    for (int64_t e = t0; e < n; e += stride) dortho[it.dst_off + e] = src[e];
    return;
  }
  if (it.mode == 3) {   // BCOP k' = 1: dQ (c x c) = dK on [:co, :ci], 0 elsewhere
    const int64_t n = (int64_t)it.rows * it.c;
    for (int64_t e = t0; e < n; e += stride) {
      const int o = (int)(e / it.c), i = (int)(e - (int64_t)o * it.c);
      dortho[it.dst_off + e] = (o < it.co && i < it.ci) ? src[(int64_t)o * it.ci + i] : 0.f;
    }
    return;
  }
  if (it.zero_off >= 0)
    for (int64_t e = t0; e < it.zero_n; e += stride) dortho[it.zero_off + e] = 0.f;
  if (it.mode == 0) {   // chain unit: dS[t][o][i], o < rows, i < c
    const int64_t n = (int64_t)it.kk * it.rows * it.c;
    for (int64_t e = t0; e < n; e += stride) {
      const int64_t t = e / ((int64_t)it.rows * it.c), r = e - t * it.rows * it.c;
      const int o = (int)(r / it.c), i = (int)(r - (int64_t)o * it.c);
      arena[it.dst_off + e] = (o < it.co && i < it.ci) ? src[((int64_t)o * it.ci + i) * it.kk + t] : 0.f;
    }
  } else {              // AOC: dFin[t][o][i] (co x ci)
    const int64_t n = (int64_t)it.kk * it.co * it.ci;
    for (int64_t e = t0; e < n; e += stride) {
      const int64_t t = e / ((int64_t)it.co * it.ci), r = e - t * it.co * it.ci;
      const int o = (int)(r / it.ci), i = (int)(r - (int64_t)o * it.ci);
      arena[it.dst_off + e] = src[((int64_t)o * it.ci + i) * it.kk + t];
    }
  }
}

__global__ void __launch_bounds__(256) vjp_scatter_kernel(const ScatterItem* __restrict__ items,
                                                          const float* __restrict__ arena, float* __restrict__ dortho) {
  const ScatterItem it = items[blockIdx.y];
  const int64_t n = (int64_t)it.ss * it.co * it.cm;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / ((int64_t)it.co * it.cm), r = e - t * it.co * it.cm;
    const int o = (int)(r / it.cm), j = (int)(r - (int64_t)o * it.cm);
    dortho[it.dst_off + ((int64_t)o * it.cm + j) * it.ss + t] = arena[it.src_off + e];
  }
}

}  // namespace

int launch_vjp_deemit(Plan& p, const float* dK, float* dortho, void* stream) {
  if (p.cv_items.empty()) return 0;
  int64_t mx = 1;
  for (auto& it : p.cv_items) mx = std::max<int64_t>(mx, (int64_t)it.kk * std::max(it.rows, it.co) * std::max(it.c, it.ci));
  const int bx = (int)std::min<int64_t>((mx + 255) / 256, 512);
  vjp_deemit_kernel<<<dim3((unsigned)bx, (unsigned)p.cv_items.size()), 256, 0, (cudaStream_t)stream>>>(
      p.d_cv_items, dK, p.d_vjp, dortho);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_vjp_scatter(Plan& p, float* dortho, void* stream) {
  if (p.cv_scatter.empty()) return 0;
  int64_t mx = 1;
  for (auto& it : p.cv_scatter) mx = std::max<int64_t>(mx, (int64_t)it.ss * it.co * it.cm);
  const int bx = (int)std::min<int64_t>((mx + 255) / 256, 512);
  vjp_scatter_kernel<<<dim3((unsigned)bx, (unsigned)p.cv_scatter.size()), 256, 0, (cudaStream_t)stream>>>(
      p.d_cv_scatter, p.d_vjp, dortho);
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
