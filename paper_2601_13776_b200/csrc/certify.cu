// f2: spectral certificate of a layer's circular conv
// operator on an H x W grid, on the device, for full-size layers (P:455-459,
// App. C: "(ii) scalable spectral norm estimation ... check that the produced
// bounds are valid"; S:444-452 the per-frequency lineage).
//
// The circular stride-s conv with dilation d is a stride-1 conv on the s^2
// polyphase components of x: writing d a - p_t = s q_a + r_a (0 <= r_a < s),
// x[s u + d a - p_t] = x_{r_a}[u + q_a].  Its operator is block-diagonalised by
// the 2-D DFT on the (H/s) x (W/s) grid: at frequency (f1, f2) the symbol is
//   A[o, (i, r_a, r_b)] = sum_{taps with residues (r_a, r_b)} K[o, i, a, b] e^{-2 pi i (f1 q_a / H' + f2 q_b / W')}
// (c_out/g x (c_in/g) s^2 per group).  The operator's singular values are those
// of all A(f1, f2).  On the SHORT side S = min(c_out/g, (c_in/g) s^2):
//   E = A^H A - I (S = columns) or A A^H - I (S = rows), and
//   max |sigma - 1| <= max |sigma^2 - 1| = |E|_2 <= |E|_F.
// Per (group, frequency) the kernels return |E|_F (the certificate) and a
// power-iteration estimate of |E|_2 (a lower bound that converges to it).
//
// Precision: the FP32 kernel values are exact in FP64 and every product and
// sum is FP64 (SIMT DFMA), so the certificate measures the FP32 kernel itself
// (FP64 rounding ~1e-16 relative) -- an FP32 Gram would add ~1e-3 of
// accumulation error at 512 channels, the size of the tolerance.
//
// Kernels: symbol_kernel (one thread per B element, taps looped),
// gram_kernel (64 x 64 complex tile per CTA, k in chunks of 16 staged in
// shared memory, 4 x 4 complex accumulators per thread), stats_kernel (one CTA
// per (group, frequency): |E|_F in a fixed order, then the power iteration).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "orth_internal.h"

namespace orth {
namespace {

struct CertGeo {
  int g, co, ci, k, s, d, pt, pl;
  int Hs, Ws, F;         // polyphase grid, frequencies per group
  int nin;               // ci * s^2
  int S, Kd;             // short side, long side
  int rows_short;        // 1: S = co (E = A A^H), 0: S = nin (E = A^H A)
};

// B[gf][kk][ii] (row-major, ii contiguous): the long side kk, the short side ii, with E = B^H B - I.
// S = nin: B[o][j] = A[o][j];   S = co: B[j][o] = conj(A[o][j]).
__global__ void __launch_bounds__(256) symbol_kernel(const float* __restrict__ K, CertGeo G, double2* __restrict__ B) {
  const int64_t per = (int64_t)G.Kd * G.S;
  const int64_t total = (int64_t)G.g * G.F * per;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gf = e / per;
    const int64_t rem = e - gf * per;
    const int kk = (int)(rem / G.S), ii = (int)(rem - (int64_t)kk * G.S);
    const int grp = (int)(gf / G.F), f = (int)(gf - (int64_t)grp * G.F);
    const int f1 = f / G.Ws, f2 = f - f1 * G.Ws;
    const int o = G.rows_short ? ii : kk;
    const int j = G.rows_short ? kk : ii;
    const int i = j / (G.s * G.s), ra = (j / G.s) % G.s, rb = j % G.s;
    const float* Ko = K + (((int64_t)grp * G.co + o) * G.ci + i) * G.k * G.k;
    double re = 0.0, im = 0.0;
    const int64_t HW = (int64_t)G.Hs * G.Ws;
    for (int a = 0; a < G.k; ++a) {
      const int ta = G.d * a - G.pt;
      const int qa = (ta >= 0) ? ta / G.s : -((-ta + G.s - 1) / G.s);
      if (ta - qa * G.s != ra) continue;
      for (int b = 0; b < G.k; ++b) {
        const int tb = G.d * b - G.pl;
        const int qb = (tb >= 0) ? tb / G.s : -((-tb + G.s - 1) / G.s);
        if (tb - qb * G.s != rb) continue;
        // phase fraction (f1 qa / H' + f2 qb / W') reduced mod 1 exactly in integers
        int64_t num = ((int64_t)f1 * qa * G.Ws + (int64_t)f2 * qb * G.Hs) % HW;
        if (num < 0) num += HW;
        double sn, cs;
        sincospi(-2.0 * (double)num / (double)HW, &sn, &cs);
        const double kv = (double)Ko[a * G.k + b];
        re += kv * cs;
        im += kv * sn;
      }
    }
    B[e] = G.rows_short ? make_double2(re, -im) : make_double2(re, im);
  }
}

constexpr int TS = 64, TK = 16;

// E[gf][i][j] = sum_k conj(B[k][i]) B[k][j] - delta_ij over one 64 x 64 tile; 16 x 16 threads with 4 x 4
// complex accumulators each (16 complex MACs = 64 DFMA per 8 shared-memory 16-byte loads)
__global__ void __launch_bounds__(256) gram_kernel(const double2* __restrict__ B, CertGeo G, double2* __restrict__ E) {
  __shared__ double2 Bi[TK][TS], Bj[TK][TS];
  // E is Hermitian: only tiles ti <= tj are computed (blockIdx.x enumerates the upper triangle row by
  // row); an off-diagonal tile also writes its conjugate mirror
  const int tiles = (G.S + TS - 1) / TS;
  int ti = 0, rem = blockIdx.x;
  while (rem >= tiles - ti) { rem -= tiles - ti; ++ti; }
  const int tj = ti + rem;
  const int64_t gf = blockIdx.y;
  const double2* Bg = B + gf * (int64_t)G.Kd * G.S;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  double2 acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < G.Kd; k0 += TK) {
    for (int x = tid; x < TK * TS; x += 256) {
      const int kr = x / TS, c = x % TS;
      const int kk = k0 + kr, ci = ti * TS + c, cj = tj * TS + c;
      Bi[kr][c] = (kk < G.Kd && ci < G.S) ? Bg[(int64_t)kk * G.S + ci] : make_double2(0.0, 0.0);
      Bj[kr][c] = (kk < G.Kd && cj < G.S) ? Bg[(int64_t)kk * G.S + cj] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 2
    for (int kr = 0; kr < TK; ++kr) {
      double2 av[4], bv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) av[p] = Bi[kr][ty + 16 * p];
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = Bj[kr][tx + 16 * q];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // conj(a) * b
          acc[p][q].x = fma(av[p].x, bv[q].x, fma(av[p].y, bv[q].y, acc[p][q].x));
          acc[p][q].y = fma(av[p].x, bv[q].y, fma(-av[p].y, bv[q].x, acc[p][q].y));
        }
    }
    __syncthreads();
  }
  double2* Eg = E + gf * (int64_t)G.S * G.S;
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = ti * TS + ty + 16 * p, j = tj * TS + tx + 16 * q;
      if (i < G.S && j < G.S) {
        double2 v = acc[p][q];
        if (i == j) v.x -= 1.0;
        Eg[(int64_t)i * G.S + j] = v;
        if (ti != tj) Eg[(int64_t)j * G.S + i] = make_double2(v.x, -v.y);
      }
    }
}

__device__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// one CTA per (group, frequency): |E|_F, then `iters` power iterations z <- E z / |E z| from a fixed start
// (E is Hermitian: the iteration converges to its largest |eigenvalue| = |E|_2); est = |E z| <= |E|_2
__global__ void __launch_bounds__(256) stats_kernel(const double2* __restrict__ E, CertGeo G, int iters,
                                                    double2* __restrict__ zbuf, double* __restrict__ out) {
  __shared__ double red[33];
  const int64_t gf = blockIdx.x;
  const int S = G.S;
  const double2* Eg = E + gf * (int64_t)S * S;
  double2* z = zbuf + gf * (int64_t)2 * S;
  double2* y = z + S;
  double f = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)S * S; e += blockDim.x) {
    const double2 v = Eg[e];
    f += v.x * v.x + v.y * v.y;
  }
  f = block_sum_d(f, red);
  // fixed start vector (not orthogonal to any eigenvector with probability one for real data)
  double nz = 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    const double v = 1.0 + 0.25 * (double)((i * 7919) % 97) / 97.0;
    z[i] = make_double2(v, 0.1 * (double)((i * 104729) % 89) / 89.0);
    nz += z[i].x * z[i].x + z[i].y * z[i].y;
  }
  nz = block_sum_d(nz, red);
  double inv = nz > 0.0 ? rsqrt(nz) : 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) z[i] = make_double2(z[i].x * inv, z[i].y * inv);
  __syncthreads();
  double est = 0.0;
  for (int it = 0; it < iters; ++it) {
    double ny = 0.0;
    for (int r = threadIdx.x; r < S; r += blockDim.x) {   // y = E z (row r: sum_j E[r][j] z[j])
      const double2* row = Eg + (int64_t)r * S;
      double re = 0.0, im = 0.0;
      for (int j = 0; j < S; ++j) {
        const double2 a = row[j], b = z[j];
        re += a.x * b.x - a.y * b.y;
        im += a.x * b.y + a.y * b.x;
      }
      y[r] = make_double2(re, im);
      ny += re * re + im * im;
    }
    ny = block_sum_d(ny, red);
    est = sqrt(ny);
    inv = ny > 0.0 ? rsqrt(ny) : 0.0;
    for (int i = threadIdx.x; i < S; i += blockDim.x) z[i] = make_double2(y[i].x * inv, y[i].y * inv);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[gf * 2] = sqrt(f);
    out[gf * 2 + 1] = est;
  }
}

bool cert_geo(const LayerInfo& L, int H, int W, CertGeo& G) {
  G = CertGeo{};
  if (L.cons == CONS_DENSE) {
    if (H != 1 || W != 1) return false;
    G.g = 1; G.co = L.co; G.ci = L.ci; G.k = 1; G.s = 1; G.d = 1; G.pt = 0; G.pl = 0;
  } else {
    if (H % L.s || W % L.s) return false;
    G.g = L.g; G.co = L.co; G.ci = L.ci; G.k = L.k; G.s = L.s; G.d = L.d; G.pt = L.pt; G.pl = L.pl;
  }
  G.Hs = H / G.s; G.Ws = W / G.s; G.F = G.Hs * G.Ws;
  G.nin = G.ci * G.s * G.s;
  G.rows_short = G.co < G.nin ? 1 : 0;
  G.S = G.rows_short ? G.co : G.nin;
  G.Kd = G.rows_short ? G.nin : G.co;
  return G.F > 0 && G.S > 0;
}

}  // namespace

int64_t certify_workspace_bytes(const LayerInfo& L, int H, int W) {
  CertGeo G;
  if (!cert_geo(L, H, W, G)) return -1;
  const int64_t gf = (int64_t)G.g * G.F;
  return 16 * gf * ((int64_t)G.Kd * G.S + (int64_t)G.S * G.S + 2 * (int64_t)G.S) + 256;
}

int launch_certify(const LayerInfo& L, const float* kernel, int H, int W, int iters, void* ws, double* out,
                   void* stream) {
  CertGeo G;
  if (!cert_geo(L, H, W, G)) return (int)cudaErrorInvalidValue;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t gf = (int64_t)G.g * G.F;
  double2* B = static_cast<double2*>(ws);
  double2* E = B + gf * (int64_t)G.Kd * G.S;
  double2* Z = E + gf * (int64_t)G.S * G.S;
  const int64_t nB = gf * (int64_t)G.Kd * G.S;
  const int blocks = (int)std::min<int64_t>((nB + 255) / 256, 148 * 16);
  symbol_kernel<<<blocks, 256, 0, s>>>(kernel, G, B);
  const int tiles = (G.S + TS - 1) / TS;
  gram_kernel<<<dim3((unsigned)(tiles * (tiles + 1) / 2), (unsigned)gf), 256, 0, s>>>(B, G, E);
  stats_kernel<<<(unsigned)gf, 256, 0, s>>>(E, G, iters, Z, out);
  return (int)cudaGetLastError();
}

}  // namespace orth
