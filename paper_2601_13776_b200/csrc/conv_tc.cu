// a6 / a7 on the 5th-generation tensor cores: implicit-GEMM convolution and
// its exact adjoint (transposed convolution), BF16 in, FP32 accumulation in
// TMEM, BF16 out (circular or zero padding, reading R11).
//
// Forward, per group g:  D[m, n] = sum_{(a,b), c} x~[pix(m, a, b), g*ci_g + c] * W[g*co_g + n, a, b, c]
//   m = output pixel (N*Ho*Wo), pix = (s u + d a - p_t, s v + d b - p_l) wrapped / zero-padded.
// Adjoint (orth_conv_transpose, R13/R14), gather form with polyphase tiles:
//   output pixels of the large grid are grouped by phase (h mod s, w mod s); in a
//   phase only the taps with (h + p_t - d a) = 0 (mod s) contribute, so the
//   K loop runs over exactly those taps:
//   D[m, n] = sum_{valid (a,b), o} y[(h + p_t - d a)/s, (w + p_l - d b)/s, g*co_g + o] * W[g*co_g + o, a, b, n]
//   (B = W^T per tap, produced by a small transpose kernel into plan workspace).
//
// Persistent, warp-specialised kernel (one CTA per SM, 416 threads):
//   warps 0-7   producers: per tile build a (valid tap, row) -> input pixel
//               table in shared memory (-1 = zero padding; circular padding
//               wraps here), then per stage 16-byte cp.async of the A rows into
//               an S-stage SWIZZLE_128B ring (zero-fill for padding / channel
//               tails); thread 0 also issues the B tile (BN rows x 64 channels
//               of one tap) by TMA.  After cp.async.wait_group + fence.proxy.async
//               they arrive on the stage's `full` mbarrier, LAG stages behind.
//   warp 8      TMEM allocation + one thread issuing tcgen05.mma (M=128, N=BN,
//               K=16, x4 per stage) into one of two TMEM accumulators.
//   warps 9-12  epilogue: tcgen05.ld of their 32-lane quarter, bias, RNE to
//               BF16, NHWC stores; arrive on `tempty`.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "orth_internal.h"
#include "pdl.h"
#include "tma_host.h"
#include "umma.cuh"

#ifdef ORTH_CONV_TRACE
// per CTA: [0] producer tid0 cycles waiting on empty, [1] MMA cycles waiting on full,
// [2] MMA cycles waiting on tempty, [3] total MMA-thread cycles, [4] k-blocks
__device__ unsigned long long ws_trace[160 * 8];
#endif

namespace orth {
namespace {

constexpr int MAX_PHASES = 16;             // s <= 4
struct TcConvArgs {
  int N, H, W, Ho, Wo, k, s, d, pt, pl, circ, transposed;
  int in_C, out_C;        // channel strides of the input / output tensors
  int cr_g, nout_g;       // reduction channels and output channels per group
  int tiles_n, num_tiles;
  int nphase;             // 1 (forward) or s*s (transposed)
  int phase_tile0[MAX_PHASES + 1];   // first tile (over m) of each phase, prefix sums
  int phase_hp[MAX_PHASES], phase_wp[MAX_PHASES], phase_cnt[MAX_PHASES];
  // per phase: contributing taps (count, and as a bit mask when k^2 <= 32), filled by launch_any so that
  // neither the MMA issuer nor the producers evaluate tap_valid's modulo arithmetic per tile
  int phase_nt[MAX_PHASES];
  uint32_t phase_taps[MAX_PHASES];
  int tiles_m;            // = phase_tile0[nphase]
  // thread-block clusters of cs CTAs along M share every B tile (TMA multicast of
  // a BN/cs-row slice per CTA); a cluster tile = cs consecutive M tiles of one phase
  int cs;
  int phase_ctile0[MAX_PHASES + 1];  // first cluster tile of each phase
  int ctiles_m, num_ctiles;
  // split-K (conv_ws only): items ct < base_ctiles are K half 0, the rest half 1 of tile ct - base_ctiles;
  // half 0 leaves its FP32 accumulator in part[tile] ([BN/4][128] float4) and raises flags[tile], half 1
  // waits, adds it, stores the output and clears the flag (fixed order: deterministic)
  int ksplit, base_ctiles;
  float* part;
  unsigned* flags;
  size_t part_bytes;
  // forward only: epilogue through a SWIZZLE_128B staging tile and one TMA tensor store per 64 output
  // channels (the tile's 128 rows are consecutive NHWC pixels); else thread-per-row 16-byte stores
  int tma_out, stage_off;
};

constexpr int NPROD = 256;                 // producer threads (warps 0-7)
constexpr int MMA_WARP = 8;
constexpr int NTHREADS = NPROD + 32 + 128;
constexpr int MAX_TAPS = 169;              // k <= 13 (the SOC explicit exponential: 1 + 6 (3 - 1))

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

struct TileInfo {
  int g, n0, phase, m0, cnt;   // m0: first row inside the phase; cnt: rows of the phase
};

// cluster tile ct, CTA rank r in the cluster -> this CTA's tile (M tiles past the
// phase's end are dummies: all rows >= cnt, loads zero-filled, nothing stored)
__device__ __forceinline__ TileInfo decode_tile(const TcConvArgs& a, int ct, int r, int BN) {
  TileInfo t;
  const int tm = ct % a.ctiles_m, rest = ct / a.ctiles_m;
  const int tn = rest % a.tiles_n;
  t.g = rest / a.tiles_n;
  t.n0 = tn * BN;
  int p = 0;
  while (p + 1 < a.nphase && a.phase_ctile0[p + 1] <= tm) ++p;
  t.phase = p;
  t.m0 = ((tm - a.phase_ctile0[p]) * a.cs + r) * 128;
  t.cnt = a.phase_cnt[p];
  return t;
}

// taps contributing to a phase (all taps for the forward); returns the count
__host__ __device__ __forceinline__ bool tap_valid_calc(const TcConvArgs& a, int phase, int tap) {
  if (!a.transposed) return true;
  const int ph = phase / a.s, pw = phase % a.s;
  const int ta = tap / a.k, tb = tap % a.k;
  return ((ph + a.pt - a.d * ta) % a.s + a.s) % a.s == 0 && ((pw + a.pl - a.d * tb) % a.s + a.s) % a.s == 0;
}
__device__ __forceinline__ bool tap_valid(const TcConvArgs& a, int phase, int tap) {
  if (a.k * a.k <= 32) return (a.phase_taps[phase] >> tap) & 1u;
  return tap_valid_calc(a, phase, tap);
}

// output pixel index (n*Hout + h)*Wout + w of row m of a phase
__device__ __forceinline__ int out_pixel(const TcConvArgs& a, int phase, int m) {
  if (!a.transposed) return m;
  const int hp = a.phase_hp[phase], wp = a.phase_wp[phase];
  const int n = m / (hp * wp), r = m - n * hp * wp;
  const int hh = r / wp, ww = r - hh * wp;
  const int h = phase / a.s + a.s * hh, w = phase % a.s + a.s * ww;
  return (n * a.H + h) * a.W + w;
}

// input pixel of row m for tap (ta, tb); -1 = zero padding
__device__ __forceinline__ int in_pixel(const TcConvArgs& a, int phase, int m, int ta, int tb) {
  if (!a.transposed) {
    const int hw = a.Ho * a.Wo;
    const int n = m / hw, rr = m - n * hw, u = rr / a.Wo, vv = rr - u * a.Wo;
    int h = u * a.s - a.pt + a.d * ta, w = vv * a.s - a.pl + a.d * tb;
    if (a.circ) {
      h = wrapi(h, a.H);
      w = wrapi(w, a.W);
    } else if (h < 0 || h >= a.H || w < 0 || w >= a.W) {
      return -1;
    }
    return (n * a.H + h) * a.W + w;
  }
  const int hp = a.phase_hp[phase], wp = a.phase_wp[phase];
  const int n = m / (hp * wp), r = m - n * hp * wp;
  const int hh = r / wp, ww = r - hh * wp;
  int th = phase / a.s + a.s * hh + a.pt - a.d * ta, tw = phase % a.s + a.s * ww + a.pl - a.d * tb;
  if (a.circ) {
    th = wrapi(th, a.H);
    tw = wrapi(tw, a.W);
  } else if (th < 0 || tw < 0) {
    return -1;
  }
  const int u = th / a.s, v = tw / a.s;   // exact: the phase makes th, tw multiples of s
  if (u >= a.Ho || v >= a.Wo) return -1;
  return (n * a.Ho + u) * a.Wo + v;
}

template <int BN, int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    conv_ws(const __nv_bfloat16* __restrict__ in, const float* __restrict__ bias, __nv_bfloat16* __restrict__ out,
            const __grid_constant__ TcConvArgs a, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmY) {
  extern __shared__ uint8_t smem_raw[];
  umma::griddep_launch_dependents();
  uint8_t* smem = umma::align1024_smem(smem_raw);
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cs = a.cs, crank = cs > 1 ? (int)umma::cluster_ctarank() : 0;
  const int cid = blockIdx.x / cs, ncl = gridDim.x / cs;
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  if (warp == MMA_WARP) umma::tmem_alloc(&tmem_base_sh, 2 * BN);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], NPROD + 1);   // + the TMA issuer's expect_tx arrival
      umma::mbar_init(&empty_bar[i], cs);         // every CTA of the cluster must release a stage
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], 128);
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  if (cs > 1) umma::cluster_sync_all();   // peers' barriers initialised before any multicast
  umma::tc_fence_after();
  umma::griddep_wait();   // PDL: the previous kernel's outputs (x, weights) are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int kk2 = a.k * a.k;

  if (warp < MMA_WARP) {
    // ------------------------------------------------------------ producers
    const int c = tid & 7, rbase = tid >> 3;   // A rows rbase + 32 i
    if (tid == 0) umma::tma_prefetch_desc(&tmB);
    int it = 0, st = 0, ph = 0;                // ring position of k-block `it`
    // No shared pixel table and no producer barriers: a warp's 32 threads gather 16 distinct rows (4 row
    // bases x 4 row groups); lane L < 16 decodes row 4 warp + (L & 3) + 32 (L >> 2) once per tile and
    // resolves its input pixel per tap, the other lanes take theirs by shuffle.  The producers thus start
    // a tile's first stages while the MMAs still consume the previous tile's.
    const int jj = lane >> 3;                                    // this thread's row base = 4 warp + jj
    const int myrow = 4 * warp + (lane & 3) + 32 * ((lane >> 2) & 3);
    const bool wrap_fast = a.H > a.d * (a.k - 1) + a.pt && a.W > a.d * (a.k - 1) + a.pl;   // one add suffices
    for (int ct = cid; ct < a.num_ctiles; ct += ncl) {
      const int khalf = ct / a.base_ctiles;
      const TileInfo t = decode_tile(a, ct - khalf * a.base_ctiles, crank, BN);
      const int c_lo = khalf * (a.cr_g / a.ksplit), c_hi = c_lo + a.cr_g / a.ksplit;
      int nb = -1, hb = 0, wb = 0;   // my decoded row: image (-1: past the phase), base row / column (tap 0)
      {
        const int m = t.m0 + myrow;
        if (m < t.cnt) {
          if (!a.transposed) {
            const int hw = a.Ho * a.Wo, n = m / hw, rr = m - n * hw, u = rr / a.Wo;
            nb = n; hb = u * a.s - a.pt; wb = (rr - u * a.Wo) * a.s - a.pl;
          } else {
            const int hp = a.phase_hp[t.phase], wp = a.phase_wp[t.phase];
            const int n = m / (hp * wp), rr = m - n * hp * wp, hh = rr / wp;
            nb = n; hb = t.phase / a.s + a.s * hh + a.pt; wb = t.phase % a.s + a.s * (rr - hh * wp) + a.pl;
          }
        }
      }
      const __nv_bfloat16* ig = in + (int64_t)t.g * a.cr_g + c * 8;
      const uint32_t off_r[4] = {umma::sw128_off(rbase, c), umma::sw128_off(rbase + 32, c),
                                 umma::sw128_off(rbase + 64, c), umma::sw128_off(rbase + 96, c)};
      for (int tap = 0; tap < kk2; ++tap) {
        if (!tap_valid(a, t.phase, tap)) continue;
        const int ta = tap / a.k, tb = tap - ta * a.k;
        int v = -1;
        if (nb >= 0) {
          if (!a.transposed) {
            int h = hb + a.d * ta, w = wb + a.d * tb;
            bool ok = true;
            if (a.circ) {
              if (wrap_fast) {
                h += h < 0 ? a.H : (h >= a.H ? -a.H : 0);
                w += w < 0 ? a.W : (w >= a.W ? -a.W : 0);
              } else {
                h = wrapi(h, a.H); w = wrapi(w, a.W);
              }
            } else {
              ok = h >= 0 && h < a.H && w >= 0 && w < a.W;
            }
            if (ok) v = (nb * a.H + h) * a.W + w;
          } else {
            int th = hb - a.d * ta, tw = wb - a.d * tb;
            bool ok = true;
            if (a.circ) {
              if (wrap_fast) {   // one add / subtract brings th, tw into range (as for the forward)
                th += th < 0 ? a.H : (th >= a.H ? -a.H : 0);
                tw += tw < 0 ? a.W : (tw >= a.W ? -a.W : 0);
              } else {
                th = wrapi(th, a.H); tw = wrapi(tw, a.W);
              }
            } else {
              ok = th >= 0 && tw >= 0;
            }
            // exact: the phase makes th, tw multiples of s (s = 2: a shift; th, tw >= 0 whenever used)
            const int u = a.s == 2 ? th >> 1 : th / a.s, vv = a.s == 2 ? tw >> 1 : tw / a.s;
            if (ok && u < a.Ho && vv < a.Wo) v = (nb * a.Ho + u) * a.Wo + vv;
          }
        }
        int pix[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pix[i] = __shfl_sync(0xffffffffu, v, jj + 4 * i);
        for (int c0 = c_lo; c0 < c_hi; c0 += 64, ++it) {
#ifdef ORTH_CONV_TRACE
          const long long tw0 = clock64();
#endif
          umma::mbar_wait(&empty_bar[st], ph ^ 1);
#ifdef ORTH_CONV_TRACE
          if (tid == 0) ws_trace[blockIdx.x * 8 + 0] += clock64() - tw0;
#endif
          const uint32_t sa = s0 + st * STAGE;
#ifdef ORTH_CONV_EXP_NOB   // timing experiment only (wrong results): no weight loads ("resident B")
          if (tid == 0) umma::mbar_arrive(&full_bar[st]);
          if (false) {
#else
          if (tid == 0) {   // B tile (BN rows x 64 channels of this tap) by TMA, SWIZZLE_128B, OOB -> 0
#endif
            umma::mbar_arrive_expect_tx(&full_bar[st], B_BYTES);
            if (cs == 1) {
              umma::tma_load_3d(sa + A_BYTES, &tmB, &full_bar[st], c0, tap, t.g * a.nout_g + t.n0);
            } else {   // this CTA's BN/cs-row slice, multicast to the whole cluster
              const int rows = BN / cs;
              umma::tma_load_3d_mc(sa + A_BYTES + crank * rows * 128, &tmB, &full_bar[st], c0, tap,
                                   t.g * a.nout_g + t.n0 + crank * rows, cmask);
            }
          }
          const bool cok = c0 + c * 8 < a.cr_g;
#ifndef ORTH_CONV_EXP_NOA   // timing experiment ORTH_CONV_EXP_NOA: no A gathers (wrong results)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool ok = cok && pix[i] >= 0;
            umma::cp_async16(sa + off_r[i], ok ? ig + (int64_t)pix[i] * a.in_C + c0 : in, ok);
          }
#endif
          // arrive on the stage's barrier when THIS thread's copies have landed (no
          // producer stall: the next stage is issued as soon as its slot is free)
          umma::cp_async_mbar_arrive(&full_bar[st]);
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
    umma::cp_async_wait<0>();
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // Kept warp-uniform for ptxas (see conv_pad.cu, ROW issuers): the cluster / tile indices are derived
      // here rather than taken from the values shared with the other roles, the stage ring is stepped,
      // not divided, and the descriptors are 64-bit values advanced by adds -- with the operands in
      // vector registers every tcgen05.mma sat in an ELECT / R2UR.BROADCAST loop, and on sm_100a the
      // issuing thread's time between MMAs adds to the MMA time.
      constexpr uint32_t IDESC = umma::idesc_bf16(128, BN);
      constexpr uint32_t STAGE16 = STAGE >> 4, A16 = A_BYTES >> 4;
      const int ucs = a.cs, ucr = ucs > 1 ? (int)umma::cluster_ctarank() : 0;
      const int ucid = blockIdx.x / ucs, uncl = gridDim.x / ucs;
      const uint64_t desc0 = umma::sdesc_sw128(umma::smem_base1024_u32(smem_raw));
      int it = 0, tcount = 0, st = 0, ph = 0;
#ifdef ORTH_CONV_TRACE
      const long long t_all = clock64();
      long long w_full = 0, w_te = 0;
#endif
      // the issuer needs only each tile's phase: its M-tile index tm = ct mod ctiles_m (base_ctiles is a
      // multiple of ctiles_m) is stepped, not divided, per tile
      const int kcs = ((a.cr_g + 63) / 64) / a.ksplit;
      int tm = ucid % a.ctiles_m;
      const int tm_step = uncl % a.ctiles_m;
      for (int ct = ucid; ct < a.num_ctiles; ct += uncl, ++tcount) {
        int phase = 0;
        while (phase + 1 < a.nphase && a.phase_ctile0[phase + 1] <= tm) ++phase;
        const int nk = a.phase_nt[phase] * kcs;
        tm += tm_step;
        if (tm >= a.ctiles_m) tm -= a.ctiles_m;
        const int acc = tcount & 1;
#ifdef ORTH_CONV_TRACE
        long long tq = clock64();
#endif
        umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
#ifdef ORTH_CONV_TRACE
        w_te += clock64() - tq;
#endif
        umma::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
#ifdef ORTH_CONV_TRACE
          tq = clock64();
#endif
          umma::mbar_wait(&full_bar[st], ph);
#ifdef ORTH_CONV_TRACE
          w_full += clock64() - tq;
#endif
#ifndef ORTH_DIAG_NOFENCE
          umma::fence_proxy_async_smem();   // cp.async (generic proxy) rows -> tcgen05.mma (async proxy)
#endif
          umma::tc_fence_after();
          const uint64_t ad = desc0 + st * STAGE16, bd = ad + A16;
#pragma unroll
          for (int q = 0; q < 4; ++q) umma::mma_bf16(d_tmem, ad + 2 * q, bd + 2 * q, IDESC, (kb | q) != 0);
          if (ucs == 1) umma::mma_commit(&empty_bar[st]);
          else umma::mma_commit_mc(&empty_bar[st], cmask);   // release the stage in every CTA of the cluster
          if (++st == S) { st = 0; ph ^= 1; }
        }
        umma::mma_commit(&tfull_bar[acc]);
      }
#ifdef ORTH_CONV_TRACE
      ws_trace[blockIdx.x * 8 + 1] = w_full;
      ws_trace[blockIdx.x * 8 + 2] = w_te;
      ws_trace[blockIdx.x * 8 + 3] = clock64() - t_all;
      ws_trace[blockIdx.x * 8 + 4] = it;
#endif
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;               // TMEM lane quarter of this warp (warps 9..12 -> 1,2,3,0)
    const int r = q * 32 + lane;
    int tcount = 0;
    for (int ct = cid; ct < a.num_ctiles; ct += ncl, ++tcount) {
      const int khalf = ct / a.base_ctiles, tb = ct - khalf * a.base_ctiles;
      const TileInfo t = decode_tile(a, tb, crank, BN);
      const int m = t.m0 + r;
      const int opix = m < t.cnt ? out_pixel(a, t.phase, m) : -1;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      const int obase = t.g * a.nout_g + t.n0;
      float4* part = a.ksplit > 1 ? reinterpret_cast<float4*>(a.part) + (int64_t)tb * (BN / 4) * 128 : nullptr;
      if (a.ksplit > 1 && khalf == 0) {   // K half 0: FP32 partial out ([col4][row] float4, coalesced)
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          float v[32];
          umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            __stcg(part + (int64_t)(cc / 4 + i) * 128 + r, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
        }
        umma::tc_fence_before();
        umma::mbar_arrive(&tempty_bar[acc]);
        umma::named_bar_sync(2, 128);
        if (r == 0)   // release, cumulative over the epilogue barrier
          asm volatile("st.release.gpu.global.u32 [%0], 1;" ::"l"(a.flags + tb) : "memory");
        continue;
      }
      if (a.ksplit > 1) {   // K half 1: wait for half 0 of this tile
        if (r == 0) {
          unsigned fv;
          do {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(fv) : "l"(a.flags + tb) : "memory");
          } while (fv == 0u);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        umma::named_bar_sync(2, 128);
      }
      if (a.tma_out) {   // staged, coalesced: per 64 channels one SWIZZLE_128B tile + one TMA store
        uint8_t* Sy = smem + a.stage_off;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 64) {
          if (r == 0) umma::bulk_wait_read0();   // the previous store has read the staging tile
          umma::named_bar_sync(2, 128);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int cc = cb + 32 * hh;
            float v[32];
            umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
            if (part) {
#pragma unroll
              for (int i2 = 0; i2 < 8; ++i2) {
                const float4 pv = __ldcg(part + (int64_t)(cc / 4 + i2) * 128 + r);
                v[4 * i2] += pv.x; v[4 * i2 + 1] += pv.y; v[4 * i2 + 2] += pv.z; v[4 * i2 + 3] += pv.w;
              }
            }
            const int o = obase + cc;
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              uint32_t pk[4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                float v0 = v[8 * i4 + 2 * jj], v1 = v[8 * i4 + 2 * jj + 1];
                if (bias) { v0 += bias[o + 8 * i4 + 2 * jj]; v1 += bias[o + 8 * i4 + 2 * jj + 1]; }
                __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
                pk[jj] = *reinterpret_cast<uint32_t*>(&b2);
              }
              *reinterpret_cast<uint4*>(Sy + umma::sw128_off(r, hh * 4 + i4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          }
          umma::fence_proxy_async_smem();   // staging writes -> TMA (async proxy) reads
          umma::named_bar_sync(2, 128);
          if (r == 0) {   // rows past the last pixel are clipped by TMA
            umma::tma_store_2d(&tmY, umma::smem_u32(Sy), obase + cb, t.m0);
            umma::bulk_commit();
          }
        }
        umma::tc_fence_before();
        umma::mbar_arrive(&tempty_bar[acc]);
        if (part) {
          umma::named_bar_sync(2, 128);
          if (r == 0) a.flags[tb] = 0u;
        }
        continue;
      }
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
        if (part) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 pv = __ldcg(part + (int64_t)(cc / 4 + i) * 128 + r);
            v[4 * i] += pv.x; v[4 * i + 1] += pv.y; v[4 * i + 2] += pv.z; v[4 * i + 3] += pv.w;
          }
        }
        if (opix >= 0) {
          const int o = obase + cc;
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float v0 = v[2 * i], v1 = v[2 * i + 1];
            if (bias) { v0 += bias[o + 2 * i]; v1 += bias[o + 2 * i + 1]; }
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
            pk[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)opix * a.out_C + o);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
      if (part) {   // the partial is consumed: re-arm the flag for the next launch
        umma::named_bar_sync(2, 128);
        if (r == 0) a.flags[tb] = 0u;
      }
    }
  }
  if (a.tma_out && warp > MMA_WARP && ((warp & 3) * 32 + lane) == 0) umma::bulk_wait0();   // stores complete
  umma::tc_fence_before();
  __syncthreads();
  if (cs > 1) umma::cluster_sync_all();   // no peer may still multicast into this CTA
  if (warp == MMA_WARP) umma::tmem_dealloc(tmem, 2 * BN);
}

// 2-SM pair version (cta_group::2): a cluster of two CTAs computes a 256-row
// tile with one tcgen05.mma M=256 N=BN per K=16 step, issued by the leader.
// Each CTA gathers its own 128 A rows (as conv_ws) and TMA-loads its own BN/2
// rows of B; the tensor cores of both SMs read both B halves, so per SM the
// shared-memory traffic per flop drops (the narrow-tile kernels above are
// shared-memory bound).  Synchronisation: the peer's B bytes complete on the
// leader's `full` barrier (cta_group::2 TMA); the peer's cp.async rows are
// relayed by one peer thread (local barrier -> remote arrive on the leader);
// the leader's commits release `empty` / signal `tfull` in both CTAs; both
// CTAs' epilogue warps arrive on the leader's `tempty`.
#ifdef ORTH_EXPERIMENTAL   // 2-SM pair: measured slower on every cfg2 layer
template <int BN, int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    conv_pair(const __nv_bfloat16* __restrict__ in, const float* __restrict__ bias, __nv_bfloat16* __restrict__ out,
              const __grid_constant__ TcConvArgs a, const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  constexpr int HB = BN / 2;   // B rows held by each CTA
  constexpr int A_BYTES = 128 * 128, B_BYTES = HB * 128, STAGE = A_BYTES + B_BYTES;
  int* tab = reinterpret_cast<int*>(smem + S * STAGE);
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int tap_id[MAX_TAPS];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int crank = (int)umma::cluster_ctarank();
  const bool leader = crank == 0;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  if (warp == MMA_WARP) umma::tmem_alloc_pair(&tmem_base_sh, 2 * BN);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      // leader: its producers + its expect_tx arrival + the peer's relay; peer: its producers (relay input)
      umma::mbar_init(&full_bar[i], leader ? NPROD + 2 : NPROD);
      umma::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], 8);   // 4 epilogue warps in each CTA
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::cluster_sync_all();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int kc = (a.cr_g + 63) / 64;
  const int kk2 = a.k * a.k;

  if (warp < MMA_WARP) {
    // ------------------------------------------------------------ producers (as conv_ws)
    const int c = tid & 7, rbase = tid >> 3;
    if (tid == 0) umma::tma_prefetch_desc(&tmB);
    const uint32_t tab_s = umma::smem_u32(tab);
    int st = 0, ph = 0;
    for (int ct = cid; ct < a.num_ctiles; ct += ncl) {
      const TileInfo t = decode_tile(a, ct, crank, BN);
      umma::named_bar_sync(1, NPROD);
      int nt = 0;
      for (int tap = 0; tap < kk2; ++tap)
        if (tap_valid(a, t.phase, tap)) {
          if (tid == 0) tap_id[nt] = tap;
          ++nt;
        }
      umma::named_bar_sync(1, NPROD);
      {
        const int r = tid & 127, m = t.m0 + r;
        int nb = -1, hb = 0, wb = 0;
        if (m < t.cnt) {
          if (!a.transposed) {
            const int hw = a.Ho * a.Wo, n = m / hw, rr = m - n * hw, u = rr / a.Wo;
            nb = n; hb = u * a.s - a.pt; wb = (rr - u * a.Wo) * a.s - a.pl;
          } else {
            const int hp = a.phase_hp[t.phase], wp = a.phase_wp[t.phase];
            const int n = m / (hp * wp), rr = m - n * hp * wp, hh = rr / wp;
            nb = n; hb = t.phase / a.s + a.s * hh + a.pt; wb = t.phase % a.s + a.s * (rr - hh * wp) + a.pl;
          }
        }
        for (int j = tid >> 7; j < nt; j += 2) {
          const int tap = tap_id[j], ta = tap / a.k, tb = tap - ta * a.k;
          int v = -1;
          if (nb >= 0) {
            if (!a.transposed) {
              int h = hb + a.d * ta, w = wb + a.d * tb;
              bool ok = true;
              if (a.circ) { h = wrapi(h, a.H); w = wrapi(w, a.W); }
              else ok = h >= 0 && h < a.H && w >= 0 && w < a.W;
              if (ok) v = (nb * a.H + h) * a.W + w;
            } else {
              int th = hb - a.d * ta, tw = wb - a.d * tb;
              bool ok = true;
              if (a.circ) { th = wrapi(th, a.H); tw = wrapi(tw, a.W); }
              else ok = th >= 0 && tw >= 0;
              const int u = th / a.s, vv = tw / a.s;
              if (ok && u < a.Ho && vv < a.Wo) v = (nb * a.Ho + u) * a.Wo + vv;
            }
          }
          tab[j * 128 + r] = v;
        }
      }
      umma::named_bar_sync(1, NPROD);
      const __nv_bfloat16* ig = in + (int64_t)t.g * a.cr_g + c * 8;
      const uint32_t off_r[4] = {umma::sw128_off(rbase, c), umma::sw128_off(rbase + 32, c),
                                 umma::sw128_off(rbase + 64, c), umma::sw128_off(rbase + 96, c)};
      for (int j = 0; j < nt; ++j) {
        const int tap = tap_id[j];
        const uint32_t trow = tab_s + (uint32_t)(j * 128 + rbase) * 4u;
        int pix[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pix[i] = umma::ld_shared_s32(trow + 128u * i);
        for (int c0 = 0; c0 < a.cr_g; c0 += 64) {
          umma::mbar_wait(&empty_bar[st], ph ^ 1);
          const uint32_t sa = s0 + st * STAGE;
          if (tid == 0) {   // this CTA's BN/2 rows of B; bytes complete on the leader's barrier
            if (leader) umma::mbar_arrive_expect_tx(&full_bar[st], 2 * B_BYTES);
            umma::tma_load_3d_pair(sa + A_BYTES, &tmB, &full_bar[st], c0, tap, t.g * a.nout_g + t.n0 + crank * HB);
          }
          const bool cok = c0 + c * 8 < a.cr_g;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool ok = cok && pix[i] >= 0;
            umma::cp_async16(sa + off_r[i], ok ? ig + (int64_t)pix[i] * a.in_C + c0 : in, ok);
          }
          umma::cp_async_mbar_arrive(&full_bar[st]);
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
    umma::cp_async_wait<0>();
  } else if (warp == MMA_WARP) {
    if (lane == 0) {
      int it = 0, tcount = 0;
      for (int ct = cid; ct < a.num_ctiles; ct += ncl, ++tcount) {
        const TileInfo t = decode_tile(a, ct, crank, BN);
        const int nt = a.phase_nt[t.phase];
        const int nk = nt * kc;
        if (leader) {
          // ---------------------------------------------------- MMA issuer (leader)
          constexpr uint32_t IDESC = umma::idesc_bf16(256, BN);
          const int acc = tcount & 1;
          umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
          umma::tc_fence_after();
          const uint32_t d_tmem = tmem + acc * BN;
          for (int kb = 0; kb < nk; ++kb, ++it) {
            const int st = it % S;
            umma::mbar_wait(&full_bar[st], (it / S) & 1);
            umma::fence_proxy_async_smem();
            umma::tc_fence_after();
            const uint32_t aa = s0 + st * STAGE, bb = aa + A_BYTES;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              umma::mma_bf16_pair(d_tmem, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), IDESC,
                                  (kb | q) != 0);
            umma::mma_commit_pair_mc(&empty_bar[st], 0x3);
          }
          umma::mma_commit_pair_mc(&tfull_bar[acc], 0x3);
        } else {
          // ---------------------------------------------------- relay (peer): local rows landed -> leader
          for (int kb = 0; kb < nk; ++kb, ++it) {
            const int st = it % S;
            umma::mbar_wait(&full_bar[st], (it / S) & 1);
            umma::fence_proxy_async_smem();   // this CTA's cp.async rows -> the pair's tensor cores
            umma::mbar_arrive_remote(&full_bar[st], 0);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    int tcount = 0;
    for (int ct = cid; ct < a.num_ctiles; ct += ncl, ++tcount) {
      const TileInfo t = decode_tile(a, ct, crank, BN);
      const int m = t.m0 + r;
      const int opix = m < t.cnt ? out_pixel(a, t.phase, m) : -1;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      const int obase = t.g * a.nout_g + t.n0;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
        if (opix >= 0) {
          const int o = obase + cc;
          uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)opix * a.out_C + o);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t pk[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              float v0 = v[8 * i + 2 * jj], v1 = v[8 * i + 2 * jj + 1];
              if (bias) { v0 += bias[o + 8 * i + 2 * jj]; v1 += bias[o + 8 * i + 2 * jj + 1]; }
              __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
              pk[jj] = *reinterpret_cast<uint32_t*>(&b2);
            }
            dst[i] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      umma::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) umma::mbar_arrive(&tempty_bar[acc]);
        else umma::mbar_arrive_remote(&tempty_bar[acc], 0);
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::cluster_sync_all();   // no peer may still signal into this CTA
  if (warp == MMA_WARP) umma::tmem_dealloc_pair(tmem, 2 * BN);
}
#endif  // ORTH_EXPERIMENTAL

// W^T per tap for the adjoint: WT[(g ci_g + i) k^2 + t][o] = W[(g co_g + o) k^2 + t][i]
__global__ void __launch_bounds__(256) transpose_w_kernel(const __nv_bfloat16* __restrict__ w,
                                                          __nv_bfloat16* __restrict__ wt, int g, int co_g, int ci_g,
                                                          int taps) {
  __shared__ __nv_bfloat16 tile[32][34];
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const int gt = blockIdx.z;   // (group, tap)
  const int gi = gt / taps, t = gt - gi * taps;
  const int o0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int oo = e >> 5, ii = e & 31;
    const int o = o0 + oo, i = i0 + ii;
    tile[oo][ii] = (o < co_g && i < ci_g) ? w[(((int64_t)gi * co_g + o) * taps + t) * ci_g + i] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * 32; e += 256) {
    const int ii = e >> 5, oo = e & 31;
    const int o = o0 + oo, i = i0 + ii;
    if (o < co_g && i < ci_g) wt[(((int64_t)gi * ci_g + i) * taps + t) * co_g + o] = tile[oo][ii];
  }
  (void)g;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}


template <int BN, int S>
int launch_ws(const __nv_bfloat16* in, const __nv_bfloat16* w, int w_rows, const float* bias, __nv_bfloat16* out,
              const TcConvArgs& a0, cudaStream_t stream) {
  g_conv_variant = BN == 256 ? ORTH_CV_GATHER256 : BN == 128 ? ORTH_CV_GATHER128 : BN == 64 ? ORTH_CV_GATHER64 : ORTH_CV_GATHER32;
  TcConvArgs a = a0;
  size_t smem = 1024 + (size_t)S * (128 * 128 + BN * 128);
  // TMA-store epilogue for forward tiles (output = consecutive pixels), ORTH_CONV_NO_TMA_OUT=1 off
  static const bool no_tma_out = std::getenv("ORTH_CONV_NO_TMA_OUT") != nullptr;
  CUtensorMap ty;
  std::memset(&ty, 0, sizeof(ty));
  a.tma_out = 0;
  if (!no_tma_out && !a.transposed && BN >= 128 && a.cs == 1 && ((uintptr_t)out & 15) == 0 && a.out_C % 8 == 0 &&
      smem + 17 * 1024 <= 227 * 1024) {
    const size_t off = ((size_t)S * (128 * 128 + BN * 128) + 1023) & ~size_t(1023);
    auto enc = tensor_map_encoder();
    const cuuint64_t dims[2] = {(cuuint64_t)a.out_C, (cuuint64_t)a.N * a.Ho * a.Wo};
    const cuuint64_t strides[1] = {(cuuint64_t)a.out_C * 2};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    if (enc && enc(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      a.tma_out = 1;
      a.stage_off = (int)off;
      smem = 1024 + off + 16 * 1024;
    }
  }
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(conv_ws<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  const int ncl_max = num_sms() / a.cs;
  const int grid = (a.num_ctiles < ncl_max ? a.num_ctiles : ncl_max) * a.cs;
  CUtensorMap tm;
  if (!make_weight_tmap(&tm, w, w_rows, a.k * a.k, a.cr_g, BN / a.cs)) return (int)cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)a.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (pdl.h)
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const int e = (int)cudaLaunchKernelEx(&cfg, conv_ws<BN, S>, in, bias, out, a, tm, ty);
#ifdef ORTH_CONV_TRACE
  {
    cudaStreamSynchronize(stream);
    static unsigned long long h[160 * 8];
    cudaMemcpyFromSymbol(h, ws_trace, sizeof(h));
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (int c = 0; c < grid && c < 160; ++c) {
      s0 += h[c * 8]; s1 += h[c * 8 + 1]; s2 += h[c * 8 + 2]; s3 += h[c * 8 + 3]; s4 += h[c * 8 + 4];
    }
    std::printf("conv_ws<%d,%d> tiles=%d grid=%d kb/cta=%.0f: mma-thread total %.0f cyc, waits: full %.0f tempty %.0f; producer empty-wait %.0f cyc (per CTA avg)\n",
                BN, S, a.num_tiles, grid, s4 / grid, s3 / grid, s1 / grid, s2 / grid, s0 / grid);
    static unsigned long long z[160 * 8];
    cudaMemcpyToSymbol(ws_trace, z, sizeof(z));
  }
#endif
  return e;
}

#ifdef ORTH_EXPERIMENTAL
template <int BN, int S>
int launch_pair(const __nv_bfloat16* in, const __nv_bfloat16* w, int w_rows, const float* bias, __nv_bfloat16* out,
                const TcConvArgs& a, cudaStream_t stream) {
  g_conv_variant = ORTH_CV_GATHER_PAIR;
  const size_t smem = 1024 + (size_t)S * (128 * 128 + BN / 2 * 128) + (size_t)a.k * a.k * 128 * 4;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(conv_pair<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(conv_pair<BN, S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = smem;
  }
  const int ncl_max = num_sms() / 2;
  const int grid = (a.num_ctiles < ncl_max ? a.num_ctiles : ncl_max) * 2;
  CUtensorMap tm;
  if (!make_weight_tmap(&tm, w, w_rows, a.k * a.k, a.cr_g, BN / 2)) return (int)cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, conv_pair<BN, S>, in, bias, out, a, tm);
}
#endif  // ORTH_EXPERIMENTAL

// Split K into two half-tile items when it pays: few tiles (at most half the SMs: every SM gets work
// twice as fast), or when the halves fill the last wave better (cfg3 512@7: 196 tiles = 1.32 waves of
// full tiles but 2.65 of halves, i.e. 2 -> 1.5 full-tile times).
static bool splitk_pays(int64_t t) {
  const int64_t S = num_sms();
  if (2 * t <= S) return true;
  return (2 * t + S - 1) / S < 2 * ((t + S - 1) / S);
}

int launch_any(const __nv_bfloat16* in, const __nv_bfloat16* w, int w_rows, const float* bias, __nv_bfloat16* out,
               TcConvArgs& a, int groups, cudaStream_t s) {
  const int n = a.nout_g;
  for (int p = 0; p < a.nphase && p < MAX_PHASES; ++p) {   // contributing taps per phase (tap_valid)
    a.phase_nt[p] = 0;
    a.phase_taps[p] = 0;
    for (int tap = 0; tap < a.k * a.k; ++tap)
      if (tap_valid_calc(a, p, tap)) {
        ++a.phase_nt[p];
        if (tap < 32) a.phase_taps[p] |= 1u << tap;
      }
  }
  // widest N tile that still gives ~every SM a tile (every K=16 MMA shape costs ~125-150 cycles, so a
  // 128x256 tile does twice the work of a 128x128 one per MMA: narrower only pays when it fills
  // otherwise idle SMs -- or, with a partial workspace, split K in two instead, ORTH_CONV_NO_SPLITK=1 off)
  int bn = n % 256 == 0 ? 256 : n % 128 == 0 ? 128 : n % 64 == 0 ? 64 : 32;
  static const int bn_cap = std::getenv("ORTH_CONV_WS_BN") ? std::atoi(std::getenv("ORTH_CONV_WS_BN")) : 256;   // A/B switch
  while (bn > bn_cap && bn > 32) bn /= 2;
  static const bool no_split = std::getenv("ORTH_CONV_NO_SPLITK") != nullptr;
  a.ksplit = 1;
  const int64_t tiles256 = (int64_t)a.tiles_m * (n / 256) * groups;
  const int kblocks = ((a.cr_g + 63) / 64) * a.k * a.k / a.nphase;   // per tile (taps spread over the phases)
  if (!no_split && a.part && a.flags && bn == 256 && a.cr_g % 128 == 0 &&
      kblocks >= 64 &&   // measured: 72 K blocks 37.6 -> 33.6 us, 36 K blocks 23.6 -> 27.1 us
      splitk_pays(tiles256) && (size_t)tiles256 * 128 * 256 * 4 <= a.part_bytes && tiles256 <= 65536)
    a.ksplit = 2;   // two half-K items per 128x256 tile: twice the MMA work per instruction, same item count
  while (a.ksplit == 1 && bn > 128 && (int64_t)a.tiles_m * (n / bn) * groups < (num_sms() * 4) / 5 &&
         n % (bn / 2) == 0)
    bn /= 2;
  a.tiles_n = n / bn;
  a.num_tiles = a.tiles_m * a.tiles_n * groups;
  if (a.num_tiles == 0) return 0;
  // clusters along M share B (multicast): 4 when every phase has >= 8 M tiles, else 2 / 1
  static const int cs_env = std::getenv("ORTH_CONV_CLUSTER") ? std::atoi(std::getenv("ORTH_CONV_CLUSTER")) : -1;
  int min_tiles = 1 << 30;
  for (int p = 0; p < a.nphase; ++p)
    if (a.phase_cnt[p] > 0) min_tiles = std::min(min_tiles, a.phase_tile0[p + 1] - a.phase_tile0[p]);
  // measured on B200: clusters (B multicast) made every cfg2 layer slower -- the stage release then
  // waits for the slowest CTA of the cluster, and these layers are not L2-bandwidth bound -- so the
  // default stays 1 (ORTH_CONV_CLUSTER=2|4 for experiments)
  int cs = 1;
  if (cs_env >= 1 && cs_env <= 4 && (cs_env & (cs_env - 1)) == 0) cs = cs_env;
  while (cs > 1 && (bn / cs) % 8 != 0) cs /= 2;
  // 2-SM pair tiles (M = 256, cta_group::2) for the wide layers.  Correct (parity-tested) but measured
  // SLOWER on every cfg2 layer (e.g. 256@8: 28 -> 40 us): the two producers run in lockstep and the
  // peer's rows reach the leader through a relay; opt-in with ORTH_CONV_PAIR=1 for experiments
#ifdef ORTH_EXPERIMENTAL
  static const bool want_pair = std::getenv("ORTH_CONV_PAIR") != nullptr;
#else
  const bool want_pair = false;
#endif
  const bool pair = want_pair && cs_env < 0 && bn >= 128 && min_tiles >= 2 && a.k <= 7;
  if (pair) cs = 2;
  a.cs = cs;
  int c0 = 0;
  for (int p = 0; p < a.nphase; ++p) {
    a.phase_ctile0[p] = c0;
    c0 += (a.phase_tile0[p + 1] - a.phase_tile0[p] + cs - 1) / cs;
  }
  a.phase_ctile0[a.nphase] = c0;
  a.ctiles_m = c0;
  a.num_ctiles = a.ctiles_m * a.tiles_n * groups;
  a.base_ctiles = a.num_ctiles;
  if (a.ksplit > 1) {
    if (pair || cs > 1) a.ksplit = 1;
    else a.num_ctiles *= a.ksplit;
  }
#ifdef ORTH_EXPERIMENTAL
  if (pair) {   // stage = 16 KB A + BN/2 x 128 B of B
    if (bn == 256) return a.k <= 3 ? launch_pair<256, 6>(in, w, w_rows, bias, out, a, s)
                                   : launch_pair<256, 5>(in, w, w_rows, bias, out, a, s);
    return a.k <= 3 ? launch_pair<128, 8>(in, w, w_rows, bias, out, a, s)
                    : launch_pair<128, 6>(in, w, w_rows, bias, out, a, s);
  }
#endif
  switch (bn) {   // deepest ring that fits 227 KB (the producers keep no pixel table in shared memory)
    case 256: return launch_ws<256, 4>(in, w, w_rows, bias, out, a, s);
    case 128: return launch_ws<128, 6>(in, w, w_rows, bias, out, a, s);
    case 64: return launch_ws<64, 9>(in, w, w_rows, bias, out, a, s);
    default: return launch_ws<32, 8>(in, w, w_rows, bias, out, a, s);
  }
}

void base_args(TcConvArgs& a, const LayerInfo& L, int N, int H, int W, int Ho, int Wo) {
  a = TcConvArgs{};
  a.N = N; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
  a.k = L.k; a.s = L.s; a.d = L.d; a.pt = L.pt; a.pl = L.pl;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
}

}  // namespace

// Group packing: P consecutive groups with few channels (ci_g, co_g < 64) are
// fused into one "virtual" group with a block-diagonal kernel, so every A row
// is a full 128-byte (64-channel) SW128 row and the MMA N is P * co_g.  The
// extra zeros cost P-times the (cheap, here under-used) MMA work but turn the
// gather of a 32-channel grouped layer from half-empty into dense rows.
static int pack_factor(const LayerInfo& L, bool bwd) {
  const int cr = bwd ? L.co : L.ci, nout = bwd ? L.ci : L.co;
  int P = 1;
  while (P * 2 <= L.g && L.g % (P * 2) == 0 && cr * P * 2 <= 64) P *= 2;
  while (P > 1 && ((P * nout) % 32 != 0)) P /= 2;
  return P;
}

static LayerInfo packed(const LayerInfo& L, int P) {
  LayerInfo q = L;
  q.g = L.g / P; q.ci = L.ci * P; q.co = L.co * P;
  return q;
}

namespace {
// W'[(gp P co + p co + o) k^2 + t][q ci + i] = (p == q) ? W[((gp P + p) co + o) k^2 + t][i] : 0
__global__ void __launch_bounds__(256) pack_w_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wp,
                                                     int gpacks, int P, int co, int ci, int taps) {
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const int64_t rowlen = (int64_t)P * ci;
  const int64_t total = (int64_t)gpacks * P * co * taps * rowlen;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int64_t row = e / rowlen;
    const int col = (int)(e - row * rowlen);
    const int t = (int)(row % taps);
    const int64_t ro = row / taps;                 // gp * P * co + p * co + o
    const int o = (int)(ro % co), p = (int)((ro / co) % P);
    const int64_t gp = ro / ((int64_t)co * P);
    const int q = col / ci, i = col - q * ci;
    wp[e] = (p == q) ? w[(((gp * P + p) * co + o) * taps + t) * ci + i] : __float2bfloat16(0.f);
  }
}
}  // namespace

bool conv_fwd_tc_eligible(const LayerInfo& L) {
  const LayerInfo q = packed(L, pack_factor(L, false));
  return q.co % 32 == 0 && q.ci % 8 == 0 && L.ci_f % 8 == 0 && L.co_f % 8 == 0 && L.k * L.k <= MAX_TAPS &&
         pack_factor(L, false) <= 8;
}

bool conv_bwd_tc_eligible(const LayerInfo& L) {
  const LayerInfo q = packed(L, pack_factor(L, true));
  return q.ci % 32 == 0 && q.co % 8 == 0 && L.ci_f % 8 == 0 && L.co_f % 8 == 0 && L.k * L.k <= MAX_TAPS &&
         L.s * L.s <= MAX_PHASES && pack_factor(L, true) <= 8;
}

static int pack_weights(const LayerInfo& L, int P, const void* kernel, void* dst, cudaStream_t s) {
  const int taps = L.k * L.k;
  const int64_t total = (int64_t)L.co_f * taps * P * L.ci;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  launch_pdl(pack_w_kernel, dim3(blocks), dim3(256), 0, s, (const __nv_bfloat16*)kernel, (__nv_bfloat16*)dst, L.g / P, P, L.co, L.ci,
                                       taps);
  return (int)cudaGetLastError();
}

// split-K partial bytes / flags of one launch_any call (upper bound of its decision): 128 x 256 FP32 tile
// per 256-wide output tile, only when the grid has at most half the SMs' worth of such tiles
static int64_t splitk_need(int64_t tiles_m, int nout_g, int cr_g, int groups, int64_t* flags) {
  if (nout_g % 256 != 0 || cr_g % 128 != 0) return 0;
  const int64_t t256 = tiles_m * (nout_g / 256) * groups;
  if (!splitk_pays(t256)) return 0;
  *flags = std::max<int64_t>(*flags, t256);
  return t256 * 128 * 256 * 4;
}

int64_t conv_scratch_need(const LayerInfo& L, int N, int H, int W, int64_t* flags) {
  *flags = 0;
  if (N < 1 || H < 1 || W < 1 || L.cons == CONS_DENSE) return 0;
  const int Ho = (H + L.pt + L.pb - L.d * (L.k - 1) - 1) / L.s + 1;
  const int Wo = (W + L.pl + L.pr - L.d * (L.k - 1) - 1) / L.s + 1;
  if (Ho < 1 || Wo < 1) return 0;
  int64_t need = 0;
  static const bool tma_on = std::getenv("ORTH_CONV_TMA") != nullptr;   // experimental padded-copy kernel
  const int ext = L.d * (L.k - 1);
  {  // forward: TMA-window kernels on a padded copy, or the gather kernel with split-K
    const LayerInfo q = packed(L, pack_factor(L, false));
    need = std::max(need, conv_stack_pad_bytes(q, N, H, W, Ho, Wo));
    if (tma_on && q.s == 1) need = std::max(need, (int64_t)N * (Ho + ext) * (Wo + ext) * q.ci_f * 2);
    need = std::max(need, splitk_need(((int64_t)N * Ho * Wo + 127) / 128, q.co, q.ci, q.g, flags));
  }
  {  // adjoint: stride 1 as the tap-flipped forward conv of the transposed view, else polyphase tiles
    const LayerInfo q = packed(L, pack_factor(L, true));
    if (q.s == 1) {
      LayerInfo F = q;
      F.ci = q.co; F.co = q.ci; F.ci_f = q.co_f; F.co_f = q.ci_f;
      F.pt = ext - q.pt; F.pl = ext - q.pl; F.pb = ext - q.pb; F.pr = ext - q.pr;
      need = std::max(need, conv_stack_pad_bytes(F, N, Ho, Wo, H, W));
      if (tma_on) need = std::max(need, (int64_t)N * (H + ext) * (W + ext) * F.ci_f * 2);
    }
    int64_t tiles = 0;   // polyphase tiles, as launch_conv_bwd_tc builds them
    for (int p = 0; p < q.s * q.s; ++p) {
      const int ph = p / q.s, pw = p % q.s;
      const int64_t hp = H > ph ? (H - ph + q.s - 1) / q.s : 0, wp = W > pw ? (W - pw + q.s - 1) / q.s : 0;
      tiles += ((int64_t)N * hp * wp + 127) / 128;
    }
    need = std::max(need, splitk_need(tiles, q.ci, q.co, q.g, flags));
  }
  return need;
}

int launch_conv_fwd_tc(const LayerInfo& L0, const void* kernel, void* scratch, const float* bias, const void* x,
                       void* y, int N, int H, int W, int Ho, int Wo, void* stream) {
  const int P = pack_factor(L0, false);
  const LayerInfo L = packed(L0, P);
  if (P > 1) {
    if (int e = pack_weights(L0, P, kernel, scratch, (cudaStream_t)stream)) return e;
    kernel = scratch;
  }
  static const bool no_reuse = std::getenv("ORTH_CONV_NO_REUSE") != nullptr;   // A/B switch
  if (!no_reuse) {   // stride 1: TMA-window kernels (conv_stack.cu: >= 128 channels, conv_pad.cu: <= 64)
    int e = launch_conv_fwd_stack(L, kernel, bias, x, y, N, H, W, Ho, Wo, stream);
    if (e < 0) e = launch_conv_fwd_reuse(L, kernel, bias, x, y, N, H, W, Ho, Wo, stream);
    if (e < 0) e = launch_conv_fwd_tma(L, kernel, bias, x, y, N, H, W, Ho, Wo, stream);
    if (e >= 0) return e;
  }
  TcConvArgs a;
  base_args(a, L, N, H, W, Ho, Wo);
  a.part = static_cast<float*>(L0.pad_scratch); a.part_bytes = (size_t)L0.pad_bytes; a.flags = L0.conv_flags;
  a.transposed = 0;
  a.in_C = L.ci_f; a.out_C = L.co_f; a.cr_g = L.ci; a.nout_g = L.co;
  a.nphase = 1;
  a.phase_cnt[0] = N * Ho * Wo;
  a.phase_tile0[0] = 0;
  a.phase_tile0[1] = (a.phase_cnt[0] + 127) / 128;
  a.tiles_m = a.phase_tile0[1];
  return launch_any((const __nv_bfloat16*)x, (const __nv_bfloat16*)kernel, L.co_f, bias, (__nv_bfloat16*)y, a, L.g,
                    (cudaStream_t)stream);
}

int launch_conv_bwd_tc(const LayerInfo& L0, const void* kernel, void* wt_scratch, const float* bias, const void* y,
                       void* x, int N, int H, int W, int Ho, int Wo, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int taps = L0.k * L0.k;
  const int P = pack_factor(L0, true);
  const LayerInfo L = packed(L0, P);
  if (P > 1) {   // block-diagonal pack into the second half of the scratch, then transpose that
    void* pk = static_cast<__nv_bfloat16*>(wt_scratch) + (int64_t)8 * L0.kernel_numel;
    if (int e = pack_weights(L0, P, kernel, pk, s)) return e;
    kernel = pk;
  }
  dim3 tg((unsigned)((L.ci + 31) / 32), (unsigned)((L.co + 31) / 32), (unsigned)(L.g * taps));
  launch_pdl(transpose_w_kernel, tg, dim3(256), 0, s, (const __nv_bfloat16*)kernel, (__nv_bfloat16*)wt_scratch, L.g, L.co, L.ci,
                                        taps);
  if (int e = (int)cudaGetLastError()) return e;
  static const bool no_reuse = std::getenv("ORTH_CONV_NO_REUSE") != nullptr;   // A/B switch
  if (L.s == 1 && !no_reuse) {
    // Stride 1: x[h, w] = sum_{a,b} K[a,b]^T y[h + p_t - d a, w + p_l - d b] is the forward conv of y
    // with the tap-flipped transposed kernel and padding d(k-1) - p (mod H for circular, where the
    // grids coincide), so it runs on the padded-window kernel (conv_pad.cu).
    LayerInfo F = L;
    F.ci = L.co; F.co = L.ci; F.ci_f = L.co_f; F.co_f = L.ci_f;
    F.pt = L.d * (L.k - 1) - L.pt; F.pl = L.d * (L.k - 1) - L.pl;
    F.pb = L.d * (L.k - 1) - L.pb; F.pr = L.d * (L.k - 1) - L.pr;
    int e = launch_conv_fwd_stack(F, wt_scratch, bias, y, x, N, Ho, Wo, H, W, stream, 1);
    if (e < 0) e = launch_conv_fwd_reuse(F, wt_scratch, bias, y, x, N, Ho, Wo, H, W, stream, 1);
    if (e < 0) e = launch_conv_fwd_tma(F, wt_scratch, bias, y, x, N, Ho, Wo, H, W, stream, 1);
    if (e >= 0) return e;
  }
  TcConvArgs a;
  base_args(a, L, N, H, W, Ho, Wo);
  a.part = static_cast<float*>(L0.pad_scratch); a.part_bytes = (size_t)L0.pad_bytes; a.flags = L0.conv_flags;
  a.transposed = 1;
  a.in_C = L.co_f; a.out_C = L.ci_f; a.cr_g = L.co; a.nout_g = L.ci;
  a.nphase = L.s * L.s;
  int t0 = 0;
  for (int p = 0; p < a.nphase; ++p) {
    const int ph = p / L.s, pw = p % L.s;
    a.phase_hp[p] = H > ph ? (H - ph + L.s - 1) / L.s : 0;
    a.phase_wp[p] = W > pw ? (W - pw + L.s - 1) / L.s : 0;
    a.phase_cnt[p] = N * a.phase_hp[p] * a.phase_wp[p];
    a.phase_tile0[p] = t0;
    t0 += (a.phase_cnt[p] + 127) / 128;
  }
  a.phase_tile0[a.nphase] = t0;
  a.tiles_m = t0;
  return launch_any((const __nv_bfloat16*)y, (const __nv_bfloat16*)wt_scratch, L.ci_f, bias, (__nv_bfloat16*)x, a,
                    L.g, s);
}

}  // namespace orth
