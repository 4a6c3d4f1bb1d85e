// f3: Adaptive-SOC explicit exponential kernel (P:124-131
// §3 "Adaptive-SOC ... stores the explicit exponential once per update";
// P:349-361 App. B.2 Theorem "Explicit conv exponential":
//   (Id + K + K(*)K/2! + K(*)K(*)K/3! + ...) * x;   S:259-267).
//
// Per SOC unit (layer, group) of width c with a free k x k kernel K:
//   1. soc_skew_kernel:  S[t][o][i] = (K[o, i, t] - K[i, o, k^2 - 1 - t]) / 2   (tap-major, R25)
//   2. S^(*)j, j = 2..n: GemmPhases of the plan (block convolutions, one c x c GEMM per output tap with a
//      segment per contributing tap pair) on the tensor cores (3-pass hi/lo split, FP32-accurate) or SIMT
//   3. soc_alpha_kernel: the scalar AOL bound (R26).  The AOL matrix of a kernel is
//      V[Delta] = sum_t S_t^T S_{t + Delta}; for a skew kernel S_t^T = -S_{flip(t)}, so
//      V[Delta] = -(S(*)S)[c0 + Delta] and d_i = sum_j sum_p |(S(*)S)[p][i][j]|: the AOL sums come for free
//      from the second power.  alpha = 1 / sqrt(max_i d_i) (1 when S = 0) makes |T(alpha S)| <= 1.
//   4. soc_sum_kernel:   E[p] = delta_{p, centre} I + sum_j alpha^j / j! S^(*)j[p - (n - j)(k - 1)/2]
//      (every power centred in the kn x kn output; odd k).
// The emit kernel then writes E in both kernel layouts; the conv calls apply it
// with "same" padding of k_eff = n (k - 1) + 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

__global__ void __launch_bounds__(256) soc_skew_kernel(const SocItem* __restrict__ items, const float* __restrict__ ortho,
                                                       float* __restrict__ W) {
  const SocItem it = items[blockIdx.y];
  const int64_t c = it.c, kk = (int64_t)it.k * it.k;
  const int64_t total = kk * c * c;
  const float* K = ortho + it.src_off;
  float* S = W + it.u_off[1];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / (c * c), r = e - t * c * c;
    const int64_t o = r / c, i = r - o * c;
    S[e] = 0.5f * (K[(o * c + i) * kk + t] - K[(i * c + o) * kk + (kk - 1 - t)]);
  }
}

__global__ void __launch_bounds__(256) soc_alpha_kernel(const SocItem* __restrict__ items, const float* __restrict__ W,
                                                        float* __restrict__ alpha) {
  __shared__ float red[8];
  const SocItem it = items[blockIdx.x];
  const int c = it.c;
  const int k2 = 2 * (it.k - 1) + 1;
  const int64_t taps = (int64_t)k2 * k2, c2 = (int64_t)c * c;
  const float* U2 = W + it.u_off[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float mx = 0.f;
  for (int i = warp; i < c; i += 8) {   // d_i = sum over taps and columns of |U2[p][i][j]|: a warp per row
    float di = 0.f;
    for (int64_t p = 0; p < taps; ++p) {
      const float* row = U2 + p * c2 + (int64_t)i * c;
      for (int j = lane; j < c; j += 32) di += fabsf(row[j]);
    }
    for (int o = 16; o > 0; o >>= 1) di += __shfl_xor_sync(0xffffffffu, di, o);
    mx = fmaxf(mx, di);
  }
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, red[w]);
    alpha[it.alpha_slot] = m > 0.f ? rsqrtf(m) : 1.f;
  }
}

__global__ void __launch_bounds__(256) soc_sum_kernel(const SocItem* __restrict__ items, const float* __restrict__ alpha,
                                                      float* __restrict__ W) {
  const SocItem it = items[blockIdx.y];
  const int64_t c = it.c, c2 = c * c;
  const int kn = it.kn, ctr = (kn - 1) / 2;
  const int64_t total = (int64_t)kn * kn * c2;
  const float a = alpha[it.alpha_slot];
  float coef[kSocMaxTerms + 1];
  {
    float f = 1.f;
    for (int j = 1; j <= it.terms; ++j) {
      f *= a / (float)j;
      coef[j] = f;
    }
  }
  float* E = W + it.e_off;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / c2, r = e - p * c2;
    const int p1 = (int)(p / kn), p2 = (int)(p - (int64_t)p1 * kn);
    const int64_t o = r / c, i = r - o * c;
    float v = (p1 == ctr && p2 == ctr && o == i) ? 1.f : 0.f;
    for (int j = 1; j <= it.terms; ++j) {
      const int kj = j * (it.k - 1) + 1, off = (it.terms - j) * (it.k - 1) / 2;
      const int q1 = p1 - off, q2 = p2 - off;
      if (q1 < 0 || q2 < 0 || q1 >= kj || q2 >= kj) continue;
      v = fmaf(coef[j], W[it.u_off[j] + (int64_t)(q1 * kj + q2) * c2 + r], v);
    }
    E[e] = v;
  }
}

}  // namespace

int launch_soc_skew(Plan& p, const float* ortho, void* stream) {
  if (p.soc.empty()) return 0;
  int64_t mx = 1;
  for (auto& it : p.soc) mx = std::max<int64_t>(mx, (int64_t)it.k * it.k * it.c * it.c);
  const int bx = (int)std::min<int64_t>((mx + 255) / 256, 1024);
  soc_skew_kernel<<<dim3((unsigned)bx, (unsigned)p.soc.size()), 256, 0, (cudaStream_t)stream>>>(p.d_soc, ortho, p.d_comp);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_soc_alpha(Plan& p, void* stream) {
  if (p.soc.empty()) return 0;
  soc_alpha_kernel<<<(unsigned)p.soc.size(), 256, 0, (cudaStream_t)stream>>>(p.d_soc, p.d_comp, p.d_soc_alpha);
  p.launches++;
  return (int)cudaGetLastError();
}

int launch_soc_sum(Plan& p, void* stream) {
  if (p.soc.empty()) return 0;
  int64_t mx = 1;
  for (auto& it : p.soc) mx = std::max<int64_t>(mx, (int64_t)it.kn * it.kn * it.c * it.c);
  const int bx = (int)std::min<int64_t>((mx + 255) / 256, 2048);
  soc_sum_kernel<<<dim3((unsigned)bx, (unsigned)p.soc.size()), 256, 0, (cudaStream_t)stream>>>(p.d_soc, p.d_soc_alpha,
                                                                                                p.d_comp);
  p.launches++;
  return (int)cudaGetLastError();
}

}  // namespace orth
