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
// shared memory, 4 x 4 complex accumulators per thread), power_step (one launch
// per power iteration over S/32 x (groups x frequencies) CTAs; the first also
// writes the |E|_F row-block partials), cert_final (fixed-order sums).
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

// Power iteration z <- E z / |E z| from a fixed start (E is Hermitian: it converges to its largest
// |eigenvalue| = |E|_2; est = |E z| <= |E|_2), one launch per iteration so that every (group, frequency)
// matvec is spread over S / 32 CTAs (a CTA per frequency streams E from L2 at a few GB/s).  y_in -> y_out:
// each CTA normalises y_in itself (z = y_in / |y_in|, staged in shared memory), then a warp per row
// (lanes stride the row: coalesced; fixed-order shuffle reduction).  On the first launch (frob = 1) the
// CTA also writes its rows' sum |E_rj|^2 -- the |E|_F partial, summed in row-block order by cert_final.
constexpr int kRowsPerCta = 32;
__global__ void __launch_bounds__(256) power_start(CertGeo G, double2* __restrict__ y0) {
  const int64_t gf = blockIdx.x;
  for (int i = threadIdx.x; i < G.S; i += blockDim.x) {
    const double v = 1.0 + 0.25 * (double)((i * 7919) % 97) / 97.0;
    y0[gf * G.S + i] = make_double2(v, 0.1 * (double)((i * 104729) % 89) / 89.0);
  }
}

__global__ void __launch_bounds__(256) power_step(const double2* __restrict__ E, CertGeo G, const double2* __restrict__ yin,
                                                  double2* __restrict__ yout, double* __restrict__ frob_part, int frob,
                                                  int mv) {
  extern __shared__ double2 zs[];
  __shared__ double red[33];
  const int64_t gf = blockIdx.y;
  const int S = G.S, rb = blockIdx.x, nrb = gridDim.x;
  const double2* Eg = E + gf * (int64_t)S * S;
  const double2* y = yin + gf * S;
  double n = 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) n += y[i].x * y[i].x + y[i].y * y[i].y;
  n = block_sum_d(n, red);
  const double inv = n > 0.0 ? rsqrt(n) : 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) zs[i] = make_double2(y[i].x * inv, y[i].y * inv);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double f = 0.0;
  for (int r = rb * kRowsPerCta + warp; r < min(S, (rb + 1) * kRowsPerCta); r += 8) {
    const double2* row = Eg + (int64_t)r * S;
    double re = 0.0, im = 0.0;
    for (int j = lane; j < S; j += 32) {
      const double2 a = row[j];
      if (frob) f += a.x * a.x + a.y * a.y;
      if (mv) {
        const double2 b = zs[j];
        re += a.x * b.x - a.y * b.y;
        im += a.x * b.y + a.y * b.x;
      }
    }
    if (mv) {
      for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
      }
      if (lane == 0) yout[gf * S + r] = make_double2(re, im);
    }
  }
  if (frob) {
    f = block_sum_d(f, red);
    if (threadIdx.x == 0) frob_part[gf * nrb + rb] = f;
  }
}

__global__ void __launch_bounds__(256) cert_final(CertGeo G, int nrb, const double* __restrict__ frob_part,
                                                  const double2* __restrict__ ylast, double* __restrict__ out) {
  __shared__ double red[33];
  const int64_t gf = blockIdx.x;
  double n = 0.0;
  for (int i = threadIdx.x; i < G.S; i += blockDim.x) {
    const double2 v = ylast[gf * G.S + i];
    n += v.x * v.x + v.y * v.y;
  }
  n = block_sum_d(n, red);
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int b = 0; b < nrb; ++b) f += frob_part[gf * nrb + b];
    out[gf * 2] = sqrt(f);
    out[gf * 2 + 1] = sqrt(n);
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
  const int64_t nrb = (G.S + kRowsPerCta - 1) / kRowsPerCta;
  return 16 * gf * ((int64_t)G.Kd * G.S + (int64_t)G.S * G.S + 2 * (int64_t)G.S) + 8 * gf * nrb + 256;
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
  const int nrb = (G.S + kRowsPerCta - 1) / kRowsPerCta;
  double* fpart = reinterpret_cast<double*>(Z + gf * (int64_t)2 * G.S);
  double2* y[2] = {Z, Z + gf * (int64_t)G.S};
  const size_t zsm = (size_t)G.S * 16;
  if (zsm > 200 * 1024) return (int)cudaErrorInvalidValue;   // S > 12800: z does not fit shared memory
  if (zsm > 48 * 1024) cudaFuncSetAttribute(power_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm);
  power_start<<<(unsigned)gf, 256, 0, s>>>(G, y[0]);
  // iters == 0: one frob-only pass; |E z| is then reported for the start vector's zero image (0)
  if (iters <= 0) {
    power_step<<<dim3((unsigned)nrb, (unsigned)gf), 256, zsm, s>>>(E, G, y[0], y[1], fpart, 1, 0);
    cudaMemsetAsync(y[1], 0, (size_t)gf * G.S * 16, s);
    cert_final<<<(unsigned)gf, 256, 0, s>>>(G, nrb, fpart, y[1], out);
    return (int)cudaGetLastError();
  }
  for (int it = 0; it < iters; ++it)
    power_step<<<dim3((unsigned)nrb, (unsigned)gf), 256, zsm, s>>>(E, G, y[it & 1], y[(it + 1) & 1], fpart,
                                                                    it == 0, 1);
  cert_final<<<(unsigned)gf, 256, 0, s>>>(G, nrb, fpart, y[iters & 1], out);
  return (int)cudaGetLastError();
}

}  // namespace orth
