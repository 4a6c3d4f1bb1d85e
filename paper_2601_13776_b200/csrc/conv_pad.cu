// a6 (forward orthogonal convolution) on the tensor cores for
// stride-1 layers with <= 64 output channels per group (>= 128: conv_stack.cu),
// with the input window brought in by TMA once per tile and reused by all taps.
//
// Output pixels of a tile are TH rows of one image at pitch P: window pixel
// r <-> output (h0 + r / P, r % P); columns past Wo are computed and dropped.
// Per 64-channel chunk the window is R = TH + d(k-1) input rows in the
// SWIZZLE_128B K-major layout (zero padding: one 4-D box, out-of-bounds filled;
// circular: the wrapped row pieces), in one of two layouts:
//   window  (default): one copy of pitch P = Wo + d(k-1); tap (a, b) starts at
//           window row d(aP + b) -- inside a 1024-byte swizzle atom, which the
//           tensor core handles at no cost (it swizzles on absolute address bits);
//   copies: k column-shifted copies of pitch round8(Wo) (ORTH_CONV_PAD_LAYOUT).
//
// Two MMA orientations:
//   SW (co_g = 64, default): D^T = W x^T, tcgen05 M = 64 channels x N = 256
//       window pixels (the weights are the A operand); the M = 64 accumulator is
//       read as 16x256b fragments and transposed by stmatrix into a SWIZZLE_128B
//       staging tile, one TMA tensor store per output row;
//   plain: M = 128 window pixels x N = BN channels, epilogue stores rows;
//   ROW (co_g = 64, k <= 4): M = 128 window pixels x N = k * 64 -- ONE MMA per kernel row a for all k
//       taps (a, b): B = the row's k weight tiles stacked (k x 64 rows), A = the window at tap (a, 0).
//       Column block b of the accumulator at window pixel r then holds tap (a, b)'s contribution to
//       output pixel r - d b (the taps of a row differ only by a d-pixel shift of the same window), so
//       the epilogue adds block b of pixel r + d b (a lane shuffle; across warps through shared
//       memory).  r + d b stays inside the tile for every valid output (the pitch P = Wo + d(k-1) ends
//       in d(k-1) junk columns).  The k-wide N amortises the window operand's shared-memory reads over
//       k taps: per K=16 step A 4 KB + B k x 2 KB, below the M128 x N(k 64) floor of k x 32 cycles.
// Weights of one (group, channel tile) stay resident in shared memory when they
// fit (each CTA then walks a contiguous tile range), else they stream per tap.
//
// Warp roles (256 threads, one CTA per SM, persistent over tiles):
//   warp 0      window producer (TMA)
//   warp 1      weight producer (TMA)
//   warp 2      TMEM allocation + the single-thread tcgen05.mma issuer
//   warps 4-7   epilogue
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "orth_internal.h"
#include "pdl.h"
#include "tma_host.h"
#include "umma.cuh"

#ifdef ORTH_CONV_TRACE
// diagnostics: per CTA, per tile (first 32) globaltimer stamps
//   [0] A issued, [1] MMA saw A landed, [2] epilogue saw accumulator, [3] epilogue done
__device__ unsigned long long conv_trace[160 * 32 * 4];
__device__ unsigned long long conv_trace_clk[160 * 32 * 4];
// per CTA: MMA-thread cycles waiting for a free accumulator, for landed windows, total, tiles
__device__ unsigned long long pad_mma_trace[160 * 4];
__device__ __forceinline__ void ctrace(int tcount, int q) {
  if (tcount < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    conv_trace[(blockIdx.x * 32 + tcount) * 4 + q] = t;
    conv_trace_clk[(blockIdx.x * 32 + tcount) * 4 + q] = clock64();
  }
}
#define CTRACE(tc, q) ctrace(tc, q)
#else
#define CTRACE(tc, q)
#endif

namespace orth {
namespace {

struct PadArgs {
  int N, H, W, Ho, Wo, k, d, pt, pl, pr, circ;
  int out_C, cr_g, nout_g;
  int P, TH, R;                  // padded pitch, output rows per tile, input rows per tile
  int tiles_h, tiles_m, tiles_n, num_tiles;
  int abuf_bytes, nabuf, sb;     // A ring (nabuf buffers), B ring stages
  int ncopy;                     // 1: one window, tap (a,b) at row d(aP + b); k: column-shifted copies per b
  int copy_bytes;                // one window / copy: R * P * 128
  int a_tx;                      // bytes landed per A buffer (ncopy windows)
  // circular padding: per window b, up to three row pieces (map index, input column start, smem column)
  int pc_map[3 * 7], pc_col[3 * 7], pc_dst[3 * 7], npc[7];
  int bres;                      // 1: all taps x chunks of one (group, n-tile) resident in smem
  int tiles_per_cta;             // resident mode: contiguous tile range per CTA (set-major order)
  int stage_off;                 // swapped mode: byte offset of the output staging area
  int stage_row;                 // swapped mode: bytes per staged output row (Wo x 128 B, 1024-aligned)
  int slack_bytes;               // the last taps read this far past a window (junk pixels only): the next
                                 // buffer / the B region must cover it, so buffers need no padding
  int flip;                      // 1: weight tap t read from row k^2-1-t (stride-1 adjoint as a forward conv)
};

constexpr int A_WARP = 0, B_WARP = 1, MMA_WARP = 2, EPI_WARP0 = 4;
constexpr int NTHREADS = 8 * 32;
constexpr int ROW_EPI = 8;   // ROW: two epilogue warps per TMEM lane quadrant, one per 32-channel half
constexpr int NTHREADS_ROW = (4 + ROW_EPI) * 32;
constexpr int MAX_SB = 16;
constexpr int MAX_AB = 4;

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// zero padding: [0] = the R x P window box; circular: one row box per distinct piece width
constexpr int MAX_MAPS = 8;
struct PadMaps {
  CUtensorMap m[MAX_MAPS];
};

// SW (swapped operands, co_g = 64): D^T = W x^T, one tcgen05.mma M=64 (channels) N=256 (pixels)
// per K step -- the weights are the 64-row A operand, the pixel window the 256-row B operand.  A
// 128x64 N=64 tile costs ~73 cycles per MMA on B200 (shared-memory bound), the 64x256 one ~128 for
// 4x the work.  The accumulator (M=64 layout: channel o in TMEM lane (o % 16) + 32 (o / 16)) is
// transposed through a shared-memory staging tile and written by TMA, one output row per store.
template <int BN, bool SW, bool ROW = false>
__global__ void __launch_bounds__(ROW ? NTHREADS_ROW : NTHREADS, 1)
    conv_pad(const float* __restrict__ bias, __nv_bfloat16* __restrict__ out, const __grid_constant__ PadArgs a,
             const __grid_constant__ PadMaps tmA, const __grid_constant__ CUtensorMap tmB,
             const __grid_constant__ CUtensorMap tmY) {
  extern __shared__ uint8_t smem_raw[];
  umma::griddep_launch_dependents();
  uint8_t* smem = umma::align1024_smem(smem_raw);
  constexpr int B_BYTES = BN * 128;
  __shared__ uint64_t a_full[MAX_AB], a_empty[MAX_AB], b_full[MAX_SB], b_empty[MAX_SB], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int SB = a.sb, NA = a.nabuf;
  constexpr int ACC_COLS = (SW || ROW) ? 256 : BN;   // TMEM columns per accumulator
  const int bst_bytes = ROW ? a.k * B_BYTES : B_BYTES;   // one streamed B stage: a tap, or a kernel row
  if (warp == MMA_WARP) umma::tmem_alloc(&tmem_base_sh, 2 * ACC_COLS);
  if (tid == 0) {
    for (int i = 0; i < NA; ++i) {
      umma::mbar_init(&a_full[i], 1);
      umma::mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < SB; ++i) {
      umma::mbar_init(&b_full[i], 1);
      umma::mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], ROW ? ROW_EPI * 32 : 128);
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  umma::griddep_wait();   // PDL: the previous kernel's outputs (x, weights) are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t abase = umma::smem_u32(smem);
  const uint32_t bbase = abase + NA * a.abuf_bytes;
  const int kk2 = a.k * a.k;

  auto decode = [&](int tile, int& n, int& h0, int& g, int& n0) {
    const int tm = tile % a.tiles_m, rest = tile / a.tiles_m;
    n0 = (rest % a.tiles_n) * BN;
    g = rest / a.tiles_n;
    n = tm / a.tiles_h;
    h0 = (tm - n * a.tiles_h) * a.TH;
  };
  // tile schedule: streaming B -> grid-stride; resident B -> a contiguous range per CTA
  const int t_begin = a.bres ? blockIdx.x * a.tiles_per_cta : blockIdx.x;
  const int t_end = a.bres ? min(a.num_tiles, t_begin + a.tiles_per_cta) : a.num_tiles;
  const int t_step = a.bres ? 1 : gridDim.x;
  const int bset_bytes = ((a.cr_g + 63) / 64) * kk2 * B_BYTES;

  if (warp == A_WARP) {
    // ---------------------------------------------------------- A producer (whole warp)
    // Circular windows are assembled from up to three TMA row pieces per input row; one thread
    // issuing them serially costs ~150 ns per piece (measured), so the rows are spread over the
    // 32 lanes (lane 0 posts the byte count first, then every lane issues its rows' pieces).
    if (lane == 0) umma::tma_prefetch_desc(&tmA.m[0]);
    int u = 0, tc_a = 0;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++tc_a) {
      int n, h0, g, n0;
      decode(tile, n, h0, g, n0);
      for (int c0 = 0; c0 < a.cr_g; c0 += 64, ++u) {
        const int ab = u % NA;
        if (u >= NA) umma::mbar_wait(&a_empty[ab], ((u / NA) - 1) & 1);
        if (c0 == 0 && lane == 0) CTRACE(tc_a, 0);
        const uint32_t dst = abase + ab * a.abuf_bytes;
        const int c = g * a.cr_g + c0;
        if (lane == 0) umma::mbar_arrive_expect_tx(&a_full[ab], (uint32_t)a.a_tx);
        __syncwarp();
        for (int b = 0; b < a.ncopy; ++b) {
          const uint32_t cb = dst + (uint32_t)(b * a.copy_bytes);
          if (!a.circ) {   // one box: R rows x P pixels x 64 channels; out of bounds -> 0
            if (lane == 0)
              umma::tma_load_4d(cb, &tmA.m[0], &a_full[ab], c, (a.ncopy > 1 ? a.d * b : 0) - a.pl, h0 - a.pt, n);
          } else {
            for (int y = lane; y < a.R; y += 32) {
              const int h = wrapi(h0 - a.pt + y, a.H);
              const uint32_t row = cb + (uint32_t)(y * a.P) * 128u;
              for (int pc = 0; pc < a.npc[b]; ++pc)
                umma::tma_load_4d(row + (uint32_t)a.pc_dst[3 * b + pc] * 128u, &tmA.m[a.pc_map[3 * b + pc]],
                                  &a_full[ab], c, a.pc_col[3 * b + pc], h, n);
            }
          }
        }
      }
    }
  } else if (warp == B_WARP) {
    if (lane == 0) {
      // ---------------------------------------------------------- B producer
      umma::tma_prefetch_desc(&tmB);
      int i = 0, cur = -1, loads = 0;
      for (int tile = t_begin; tile < t_end; tile += t_step) {
        int n, h0, g, n0;
        decode(tile, n, h0, g, n0);
        if (a.bres) {   // whole (group, n-tile) weight set, once per set change
          const int set = tile / a.tiles_m;
          if (set == cur) continue;
          if (loads > 0) umma::mbar_wait(&b_empty[0], (loads - 1) & 1);   // MMAs on the old set done
          cur = set;
          umma::mbar_arrive_expect_tx(&b_full[0], (uint32_t)bset_bytes);
          int j = 0;
          for (int c0 = 0; c0 < a.cr_g; c0 += 64)
            for (int tap = 0; tap < kk2; ++tap, ++j)
              umma::tma_load_3d(bbase + j * B_BYTES, &tmB, &b_full[0], c0, a.flip ? kk2 - 1 - tap : tap,
                                g * a.nout_g + n0);
          ++loads;
          continue;
        }
        if (ROW) {   // one stage per (chunk, kernel row): the row's k tap tiles back to back
          for (int c0 = 0; c0 < a.cr_g; c0 += 64)
            for (int ra = 0; ra < a.k; ++ra, ++i) {
              const int st = i % SB;
              if (i >= SB) umma::mbar_wait(&b_empty[st], ((i / SB) - 1) & 1);
              umma::mbar_arrive_expect_tx(&b_full[st], (uint32_t)bst_bytes);
              for (int b = 0; b < a.k; ++b) {
                const int tap = ra * a.k + b;
                umma::tma_load_3d(bbase + st * bst_bytes + b * B_BYTES, &tmB, &b_full[st], c0,
                                  a.flip ? kk2 - 1 - tap : tap, g * a.nout_g + n0);
              }
            }
          continue;
        }
        for (int c0 = 0; c0 < a.cr_g; c0 += 64)
          for (int tap = 0; tap < kk2; ++tap, ++i) {
            const int st = i % SB;
            if (i >= SB) umma::mbar_wait(&b_empty[st], ((i / SB) - 1) & 1);
            umma::mbar_arrive_expect_tx(&b_full[st], B_BYTES);
            umma::tma_load_3d(bbase + st * B_BYTES, &tmB, &b_full[st], c0, a.flip ? kk2 - 1 - tap : tap,
                              g * a.nout_g + n0);
          }
      }
    }
  } else if (ROW && (warp == MMA_WARP || warp == MMA_WARP + 1)) {
    // ------------------------------------------------------ MMA issuers (kernel-row form)
    // On sm_100a a tcgen05.mma is accepted only shortly before the tensor core can start it, so every
    // cycle the issuing thread spends between MMAs (an mbarrier wait, ~100 cycles even when the phase
    // has completed; descriptor arithmetic in vector registers, R2UR) adds to the tile time 1:1
    // (tools/micro/row_mma2.cu: a 200-cycle stall per 12-MMA tile costs 210 cycles).  Hence:
    //  * with one resident weight set, TWO issuing threads (warps 2 and 3) take alternate tiles --
    //    accumulator a = tile parity -- so one waits for its window / accumulator while the other's
    //    MMAs run;
    //  * the loop is specialised on resident-vs-streamed weights and on k, the descriptors are 64-bit
    //    values advanced by adds and the tile range is re-derived here from kernel parameters, which
    //    keeps the MMA operands in uniform registers (computed per MMA in vector registers, ptxas wraps
    //    each tcgen05.mma in an ELECT / R2UR.BROADCAST loop).
    const int wi = warp - MMA_WARP;
    const bool dual = a.bres && a.num_tiles <= a.tiles_m;   // a single resident weight set
    if (lane == 0 && (wi == 0 || dual)) {
      const int nw = dual ? 2 : 1, nch = (a.cr_g + 63) / 64;
      const uint32_t ubase = umma::smem_base1024_u32(smem_raw);
      const uint64_t a_desc0 = umma::sdesc_sw128(ubase), b_desc0 = a_desc0 + (uint32_t)a.nabuf * ((uint32_t)a.abuf_bytes >> 4);
      const uint32_t a_buf16 = (uint32_t)a.abuf_bytes >> 4, a_row16 = (uint32_t)(a.d * a.P) * 8u;
      const uint32_t b_row16 = (uint32_t)(a.k * B_BYTES) >> 4, b_set16 = (uint32_t)(kk2 * B_BYTES) >> 4;
      const uint32_t b_st16 = (uint32_t)bst_bytes >> 4;
      const uint32_t idesc_row = umma::idesc_bf16(128, a.k * 64);
#ifdef ORTH_CONV_TRACE
      const long long t_all0 = clock64();
#endif
      // WI (issuer index), BRES and K are compile-time so that the loop state is provably warp-uniform
      // (a value derived from threadIdx is not, to ptxas); K = 0: the kernel row count at run time
      auto issue = [&](auto wi_c, auto bres_c, auto k_c) {
        constexpr int WI = decltype(wi_c)::value;
        constexpr bool BRES = decltype(bres_c)::value;
        constexpr int KC = decltype(k_c)::value;
        const int K = KC ? KC : a.k;
        // the tile range is derived here, inside the issuing branch: computed before it (and shared with
        // the other roles) it reaches ptxas as a non-uniform value and the MMA operands with it
        const int tb = a.bres ? blockIdx.x * a.tiles_per_cta : blockIdx.x;
        const int te = a.bres ? min(a.num_tiles, tb + a.tiles_per_cta) : a.num_tiles;
        const int ts = a.bres ? 1 : gridDim.x;
        int ab = 0, aph = 0, st = 0, bph = 0, cur = -1, loads = 0, tcount = WI;
        auto adv_a = [&]() {
          if (++ab == NA) { ab = 0; aph ^= 1; }
        };
        for (int c = 0; c < WI * nch; ++c) adv_a();   // this issuer's first tile starts at chunk WI * nch
        for (int tile = tb + WI * ts; tile < te; tile += nw * ts, tcount += nw) {
          if (BRES) {
            const int set = tile / a.tiles_m;
            if (set != cur) {
              if (loads > 0) umma::mma_commit(&b_empty[0]);   // (single issuer only: dual has one set)
              umma::mbar_wait_uni(&b_full[0], loads & 1);
              cur = set;
              ++loads;
            }
          }
          const int acc = tcount & 1;
#ifdef ORTH_CONV_TRACE
          long long tq0 = clock64();
#endif
          umma::mbar_wait_uni(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
#ifdef ORTH_CONV_TRACE
          if (blockIdx.x < 160 && WI == 0) pad_mma_trace[blockIdx.x * 4 + 0] += clock64() - tq0;
#endif
          umma::tc_fence_after();
          const uint32_t d_tmem = tmem_base_sh + acc * ACC_COLS;
          uint64_t bset = b_desc0;
          for (int c0 = 0; c0 < a.cr_g; c0 += 64, bset += b_set16) {
#ifdef ORTH_CONV_TRACE
            tq0 = clock64();
#endif
            umma::mbar_wait_uni(&a_full[ab], aph);
#ifdef ORTH_CONV_TRACE
            if (blockIdx.x < 160 && WI == 0) pad_mma_trace[blockIdx.x * 4 + 1] += clock64() - tq0;
#endif
            umma::tc_fence_after();
            if (c0 == 0 && WI == 0) CTRACE(tcount, 1);
            uint64_t ad = a_desc0 + ab * a_buf16;
#pragma unroll
            for (int ra = 0; ra < K; ++ra, ad += a_row16) {
              uint64_t bd = bset + ra * b_row16;
              if (!BRES) {
                umma::mbar_wait_uni(&b_full[st], bph);
                umma::tc_fence_after();
                bd = b_desc0 + st * b_st16;
              }
              const uint32_t acc0 = (c0 | ra) != 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) umma::mma_bf16(d_tmem, ad + 2 * q, bd + 2 * q, idesc_row, acc0 | (q != 0));
              if (!BRES) {
                umma::mma_commit(&b_empty[st]);
                if (++st == SB) { st = 0; bph ^= 1; }
              }
            }
            umma::mma_commit(&a_empty[ab]);
            adv_a();
          }
          umma::mma_commit(&tfull_bar[acc]);
          for (int c = 0; c < (nw - 1) * nch; ++c) adv_a();   // the other issuer's tile
        }
      };
      using T = std::true_type;
      using F = std::false_type;
      using W0 = std::integral_constant<int, 0>;
      using W1 = std::integral_constant<int, 1>;
      using K0 = std::integral_constant<int, 0>;
      using K3 = std::integral_constant<int, 3>;
      if (!a.bres) {
        if (a.k == 3) issue(W0{}, F{}, K3{});
        else issue(W0{}, F{}, K0{});
      } else if (wi == 0) {
        if (a.k == 3) issue(W0{}, T{}, K3{});
        else issue(W0{}, T{}, K0{});
      } else {
        if (a.k == 3) issue(W1{}, T{}, K3{});
        else issue(W1{}, T{}, K0{});
      }
#ifdef ORTH_CONV_TRACE
      if (blockIdx.x < 160 && wi == 0) {
        pad_mma_trace[blockIdx.x * 4 + 2] += clock64() - t_all0;
        pad_mma_trace[blockIdx.x * 4 + 3] += (min(a.num_tiles, (int)blockIdx.x * a.tiles_per_cta + a.tiles_per_cta) - (int)blockIdx.x * a.tiles_per_cta + nw - 1) / nw;
      }
#endif
    }
    __syncwarp();
  } else if (!ROW && (warp == MMA_WARP || warp == MMA_WARP + 1)) {
    // ------------------------------------------------------ MMA issuers (one MMA chain per tap)
    // Same rules as the kernel-row issuers above: compile-time resident-vs-streamed weights, locally
    // derived bases and tile range, rings stepped, descriptors advanced by adds; two issuers on
    // alternate tiles when the CTA's tiles share one resident weight set.
    constexpr uint32_t IDESC = SW ? umma::idesc_bf16(64, 256) : umma::idesc_bf16(128, BN);
    const int wi = warp - MMA_WARP;
    const bool dual = a.bres && a.num_tiles <= a.tiles_m;
    if (lane == 0 && (wi == 0 || dual)) {
      const int nw = dual ? 2 : 1, nch = (a.cr_g + 63) / 64;
      const uint32_t ubase = umma::smem_base1024_u32(smem_raw);
      const uint64_t a_desc0 = umma::sdesc_sw128(ubase), b_desc0 = a_desc0 + (uint32_t)a.nabuf * ((uint32_t)a.abuf_bytes >> 4);
      const uint32_t a_buf16 = (uint32_t)a.abuf_bytes >> 4, row16 = (uint32_t)(a.d * a.P) * 8u, col16 = (uint32_t)a.d * 8u;
      const uint32_t copy16 = (uint32_t)a.copy_bytes >> 4, tap16 = (uint32_t)B_BYTES >> 4;
      const uint32_t set16 = (uint32_t)kk2 * tap16;
      const bool copies = a.ncopy > 1;
#ifdef ORTH_CONV_TRACE
      const long long t_all0 = clock64();
#endif
      auto issue = [&](auto wi_c, auto bres_c) {
        constexpr int WI = decltype(wi_c)::value;
        constexpr bool BRES = decltype(bres_c)::value;
        const int tb0 = a.bres ? blockIdx.x * a.tiles_per_cta : blockIdx.x;
        const int te = a.bres ? min(a.num_tiles, tb0 + a.tiles_per_cta) : a.num_tiles;
        const int ts = a.bres ? 1 : gridDim.x;
        int ab = 0, aph = 0, st = 0, bph = 0, cur = -1, loads = 0, tcount = WI;
        auto adv_a = [&]() {
          if (++ab == NA) { ab = 0; aph ^= 1; }
        };
        for (int c = 0; c < WI * nch; ++c) adv_a();
        for (int tile = tb0 + WI * ts; tile < te; tile += nw * ts, tcount += nw) {
          if (BRES) {
            const int set = tile / a.tiles_m;
            if (set != cur) {
              if (loads > 0) umma::mma_commit(&b_empty[0]);   // (single issuer only: dual has one set)
              umma::mbar_wait_uni(&b_full[0], loads & 1);
              cur = set;
              ++loads;
            }
          }
          const int acc = tcount & 1;
#ifdef ORTH_CONV_TRACE
          long long tq0 = clock64();
#endif
          umma::mbar_wait_uni(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
#ifdef ORTH_CONV_TRACE
          if (blockIdx.x < 160 && WI == 0) pad_mma_trace[blockIdx.x * 4 + 0] += clock64() - tq0;
#endif
          umma::tc_fence_after();
          const uint32_t d_tmem = tmem_base_sh + acc * ACC_COLS;
          uint64_t bset = b_desc0;
          for (int c0 = 0; c0 < a.cr_g; c0 += 64, bset += set16) {
#ifdef ORTH_CONV_TRACE
            tq0 = clock64();
#endif
            umma::mbar_wait_uni(&a_full[ab], aph);
#ifdef ORTH_CONV_TRACE
            if (blockIdx.x < 160 && WI == 0) pad_mma_trace[blockIdx.x * 4 + 1] += clock64() - tq0;
#endif
            umma::tc_fence_after();
            if (c0 == 0 && WI == 0) CTRACE(tcount, 1);
            const uint64_t abuf = a_desc0 + ab * a_buf16;
            uint64_t btap = bset;
            for (int ta = 0; ta < a.k; ++ta) {
              for (int tb = 0; tb < a.k; ++tb, btap += tap16) {
                const uint64_t aa = copies ? abuf + tb * copy16 + ta * row16 : abuf + ta * row16 + tb * col16;
                uint64_t bb = btap;
                if (!BRES) {
                  umma::mbar_wait_uni(&b_full[st], bph);
                  umma::tc_fence_after();
                  bb = b_desc0 + st * tap16;
                }
                const uint32_t acc0 = (c0 | ta | tb) != 0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  umma::mma_bf16(d_tmem, (SW ? bb : aa) + 2 * q, (SW ? aa : bb) + 2 * q, IDESC, acc0 | (q != 0));
                if (!BRES) {
                  umma::mma_commit(&b_empty[st]);
                  if (++st == SB) { st = 0; bph ^= 1; }
                }
              }
            }
            umma::mma_commit(&a_empty[ab]);
            adv_a();
          }
          umma::mma_commit(&tfull_bar[acc]);
          for (int c = 0; c < (nw - 1) * nch; ++c) adv_a();   // the other issuer's tile
        }
      };
      using T = std::true_type;
      using F = std::false_type;
      using W0 = std::integral_constant<int, 0>;
      using W1 = std::integral_constant<int, 1>;
      if (!a.bres) issue(W0{}, F{});
      else if (wi == 0) issue(W0{}, T{});
      else issue(W1{}, T{});
#ifdef ORTH_CONV_TRACE
      if (blockIdx.x < 160 && wi == 0) {
        pad_mma_trace[blockIdx.x * 4 + 2] += clock64() - t_all0;
        pad_mma_trace[blockIdx.x * 4 + 3] += (min(a.num_tiles, (int)blockIdx.x * a.tiles_per_cta + a.tiles_per_cta) - (int)blockIdx.x * a.tiles_per_cta + nw - 1) / nw;
      }
#endif
    }
    __syncwarp();
  } else if (SW && warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue (swapped)
    // Warp q reads TMEM lanes 32q .. 32q+15 (channels 16q .. 16q+15) as mma-style 8x8 fragments
    // (16x256b loads) and writes them transposed with stmatrix: 16 B = 8 channels of one pixel per row.
    // Staging: output row yy at S + yy * stage_row, pixel x at + 128 x, 16-B chunk c at position
    // c ^ (x & 7) (the TMA SWIZZLE_128B layout, conflict-free for 8 consecutive pixels); window
    // columns that are not outputs go to a per-lane dump slot after the rows.
    const int q = warp & 3;
    uint8_t* S = smem + a.stage_off;
    const uint32_t s_base = umma::smem_u32(S);
    const uint32_t dump = s_base + (uint32_t)(a.TH * a.stage_row) + (uint32_t)lane * 16u;
    const int m = lane >> 3, jrow = lane & 7;
    const uint32_t chunk = (uint32_t)(2 * q + (m & 1));
    int tcount = 0;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++tcount) {
      int n, h0, g, n0;
      decode(tile, n, h0, g, n0);
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      if (tid == EPI_WARP0 * 32) CTRACE(tcount, 2);
      if (tid == EPI_WARP0 * 32) umma::bulk_wait_read0();   // the previous tile's stores have read S
      umma::named_bar_sync(2, 128);
      const int ob = g * a.nout_g + n0 + 16 * q + (lane >> 2);
      const float b_lo = bias ? bias[ob] : 0.f, b_hi = bias ? bias[ob + 8] : 0.f;
      const int rows = min(a.TH, a.Ho - h0);
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        uint32_t r[16];
        umma::tmem_ld_16x256b_x4(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256 + c), r);
        umma::tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int w = c + 16 * h + 8 * (m >> 1) + jrow;   // window pixel this lane addresses
          const int y = w / a.P, x = w - y * a.P;
          const uint32_t dst = (y < rows && x < a.Wo)
                                   ? s_base + (uint32_t)(y * a.stage_row + x * 128) + ((chunk ^ (uint32_t)(x & 7)) << 4)
                                   : dump;
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float bb = (e & 1) ? b_hi : b_lo;
            __nv_bfloat162 v2 = __floats2bfloat162_rn(__uint_as_float(r[8 * h + 2 * e]) + bb,
                                                      __uint_as_float(r[8 * h + 2 * e + 1]) + bb);
            pk[e] = *reinterpret_cast<uint32_t*>(&v2);
          }
          umma::stmatrix_x4_trans(dst, pk[0], pk[1], pk[2], pk[3]);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
      umma::fence_proxy_async_smem();                   // staging writes -> TMA (async proxy) reads
      umma::named_bar_sync(2, 128);
#ifdef ORTH_CONV_EXP
      if (false) {
#else
      if (tid == EPI_WARP0 * 32) {
#endif
        for (int yy = 0; yy < rows; ++yy)   // one output row (Wo pixels x 64 ch) per store
          umma::tma_store_3d(&tmY, s_base + (uint32_t)(yy * a.stage_row), g * a.nout_g + n0, 0, n * a.Ho + h0 + yy);
        umma::bulk_commit();
        CTRACE(tcount, 3);
      }
    }
    if (tid == EPI_WARP0 * 32) umma::bulk_wait0();
  } else if (ROW && warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue (kernel-row MMAs)
    // Thread = window pixel r (TMEM lane).  y[r][o] = sum_b acc[r + d b][b 64 + o]: block b of lane
    // r + d b comes by shuffle from the same warp, or from the next warp through `xs` (the first
    // d (k-1) lanes of every warp publish their blocks, one barrier per tile among the four warps of a
    // 32-channel half); lanes past the tile only feed junk outputs.  Eight warps: warp 4 + 4h + q reads
    // lane quadrant q, channel half h.
    const int q = warp & 3, h = (warp - EPI_WARP0) >> 2;             // TMEM lane quadrant, channel half
    const int r = q * 32 + lane;
    const int y = r / a.P, x = r - y * a.P;
    const int xl = a.d * (a.k - 1);                       // lanes published per warp (< 32)
    const int reg = 4 * 3 * xl * 16;                      // floats per exchange region: [warp][b - 1][lane][16]
    float* xs = reinterpret_cast<float*>(smem + a.stage_off);   // regions [half][chunk][tile parity]
    int tcount = 0;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++tcount) {
      int n, h0, g, n0;
      decode(tile, n, h0, g, n0);
      const int opix = (y < a.TH && x < a.Wo && h0 + y < a.Ho) ? (n * a.Ho + h0 + y) * a.Wo + x : -1;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      if (q == 0 && lane == 0) CTRACE(tcount, 2);
      const int obase = g * a.nout_g + n0;
#pragma unroll 1
      for (int ci = 0; ci < 2; ++ci) {   // two 16-channel chunks of this warp's half
        const int cc = 32 * h + 16 * ci;
        uint32_t rv[4][16];   // the k column blocks of this chunk, all in flight, one wait
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (b < a.k) umma::tmem_ld16_nw(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 256 + b * 64 + cc), rv[b]);
        umma::tmem_ld_wait();
        // one region per (half, chunk, tile parity): a warp publishing the next use of a region has passed
        // the barrier of the use in between, which every reader of this use reached after reading
        float* xh = xs + ((h * 2 + ci) * 2 + (tcount & 1)) * reg;
        if (lane < xl) {
#pragma unroll
          for (int b = 1; b < 4; ++b)
            if (b < a.k && lane < a.d * b) {
              float4* d4 = reinterpret_cast<float4*>(xh + ((q * 3 + b - 1) * xl + lane) * 16);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                d4[e] = make_float4(__uint_as_float(rv[b][4 * e]), __uint_as_float(rv[b][4 * e + 1]),
                                    __uint_as_float(rv[b][4 * e + 2]), __uint_as_float(rv[b][4 * e + 3]));
            }
        }
        umma::named_bar_sync(3 + h, 128);   // the four warps of this half
        float s[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) s[e] = __uint_as_float(rv[0][e]);
#pragma unroll
        for (int b = 1; b < 4; ++b) {
          if (b >= a.k) break;
          const int sh = a.d * b, src = lane + sh - 32;   // src >= 0: the partner is lane src of warp q + 1
          float t[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) t[e] = __shfl_down_sync(0xffffffffu, __uint_as_float(rv[b][e]), sh);
          if (src >= 0) {   // the last d b lanes (divergent, short)
            if (q < 3) {
              const float4* s4 = reinterpret_cast<const float4*>(xh + (((q + 1) * 3 + b - 1) * xl + src) * 16);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float4 v4 = s4[e];
                t[4 * e] = v4.x; t[4 * e + 1] = v4.y; t[4 * e + 2] = v4.z; t[4 * e + 3] = v4.w;
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) t[e] = 0.f;   // past the tile: feeds junk outputs only
            }
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) s[e] += t[e];
        }
        if (opix >= 0) {
          const int o = obase + cc;
          uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)opix * a.out_C + o);
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            uint32_t pk[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              float v0 = s[8 * i + 2 * jj], v1 = s[8 * i + 2 * jj + 1];
              if (bias) { v0 += bias[o + 8 * i + 2 * jj]; v1 += bias[o + 8 * i + 2 * jj + 1]; }
              __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
              pk[jj] = *reinterpret_cast<uint32_t*>(&b2);
            }
            dst[i] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
      if (q == 0 && lane == 0) CTRACE(tcount, 3);
    }
  } else if (!SW && !ROW && warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int y = r / a.P, x = r - y * a.P;
    int tcount = 0;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++tcount) {
      int n, h0, g, n0;
      decode(tile, n, h0, g, n0);
      const int opix = (y < a.TH && x < a.Wo && h0 + y < a.Ho) ? (n * a.Ho + h0 + y) * a.Wo + x : -1;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      if (q == 0 && lane == 0) CTRACE(tcount, 2);
      const int obase = g * a.nout_g + n0;
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
      umma::mbar_arrive(&tempty_bar[acc]);
      if (q == 0 && lane == 0) CTRACE(tcount, 3);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) umma::tmem_dealloc(tmem, 2 * ACC_COLS);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr size_t kSmemMax = 227 * 1024 - 1024;   // opt-in dynamic limit minus the static barriers

// 4-D map over the NHWC activation (C, W, H, N): box 64 ch x bw pixels x bh rows x 1 image, SWIZZLE_128B
bool make_act_tmap(CUtensorMap* out, const void* x, int C, int W, int H, int N, int bw, int bh) {
  using Key = std::tuple<const void*, int, int, int, int, int, int>;
  static std::map<Key, CUtensorMap> cache;
  static std::mutex mu;
  const Key key{x, C, W, H, N, bw, bh};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return true;
    }
  }
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  const cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = m;
  *out = m;
  return true;
}

template <int BN, bool SW, bool ROW = false>
int launch_pad(const void* x, const __nv_bfloat16* w, int w_rows, const float* bias, __nv_bfloat16* out, PadArgs& a,
               int in_C, cudaStream_t stream) {
  const size_t fixed = 1024;
  // swapped mode: output staging rows; ROW: the cross-warp exchange of d (k-1) lanes x 32 floats per warp
  const size_t stage = SW ? (size_t)a.TH * a.stage_row + 1024
                          : ROW ? (size_t)8 * 4 * 3 * a.d * (a.k - 1) * 16 * 4 : 0;
  const size_t bst = (size_t)(ROW ? a.k : 1) * BN * 128;   // one streamed B stage
  const size_t bset = (size_t)((a.cr_g + 63) / 64) * a.k * a.k * BN * 128;
  size_t smem;
  if (a.bres) {   // resident weights + >= 2 A buffers
    if (fixed + 2 * (size_t)a.abuf_bytes + bset + stage > kSmemMax) return -1;
    int na = MAX_AB;
    while (na > 2 && fixed + (size_t)na * a.abuf_bytes + bset + stage > kSmemMax) --na;
    a.nabuf = na;
    a.sb = 1;
    const int grid0 = std::min(a.num_tiles, sm_count());
    a.tiles_per_cta = (a.num_tiles + grid0 - 1) / grid0;
    a.stage_off = (int)(na * (size_t)a.abuf_bytes + bset);
    smem = fixed + (size_t)na * a.abuf_bytes + bset + stage;
  } else {
    // A ring: as many buffers as leave room for >= 4 B stages (at least 2)
    int na = MAX_AB;
    while (na > 2 && fixed + (size_t)na * a.abuf_bytes + 4 * bst + stage > kSmemMax) --na;
    if (fixed + (size_t)na * a.abuf_bytes + 2 * bst + stage > kSmemMax) return -1;
    a.nabuf = na;
    a.sb = (int)std::min<size_t>(MAX_SB, (kSmemMax - fixed - stage - (size_t)na * a.abuf_bytes) / bst);
    a.stage_off = (int)(na * (size_t)a.abuf_bytes + (size_t)a.sb * bst);
    smem = fixed + (size_t)na * a.abuf_bytes + (size_t)a.sb * bst + stage;
  }
  if (smem - fixed - (size_t)a.nabuf * a.abuf_bytes < (size_t)a.slack_bytes) return -1;   // reads stay in smem
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(conv_pad<BN, SW, ROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return (int)cudaGetLastError();
    attr = smem;
  }
  PadMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  if (!a.circ) {
    if (!make_act_tmap(&maps.m[0], x, in_C, a.W, a.H, a.N, a.P, a.R)) return (int)cudaErrorInvalidValue;
  } else {   // one row box per distinct piece width
    int widths[MAX_MAPS], nw = 0;
    for (int b = 0; b < a.ncopy; ++b)
      for (int pc = 0; pc < a.npc[b]; ++pc) {
        const int w0 = a.pc_map[3 * b + pc];   // host stored the width here; replaced by the map index
        int m = 0;
        while (m < nw && widths[m] != w0) ++m;
        if (m == nw) {
          if (nw == MAX_MAPS) return -1;
          widths[nw++] = w0;
          if (!make_act_tmap(&maps.m[m], x, in_C, a.W, a.H, a.N, w0, 1)) return (int)cudaErrorInvalidValue;
        }
        a.pc_map[3 * b + pc] = m;
      }
  }
  CUtensorMap tm;
  if (!make_weight_tmap(&tm, w, w_rows, a.k * a.k, a.cr_g, BN)) return (int)cudaErrorInvalidValue;
  CUtensorMap ty;
  std::memset(&ty, 0, sizeof(ty));
  if (SW) {   // output (C, Wo, N*Ho): one output row (Wo pixels x 64 channels) per box, SWIZZLE_128B staging
    auto enc = tensor_map_encoder();
    const cuuint64_t dims[3] = {(cuuint64_t)a.out_C, (cuuint64_t)a.Wo, (cuuint64_t)a.N * a.Ho};
    const cuuint64_t strides[2] = {(cuuint64_t)a.out_C * 2, (cuuint64_t)a.Wo * a.out_C * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)a.Wo, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (!enc || enc(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, out, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return (int)cudaErrorInvalidValue;
  }
  const int grid = a.bres ? (a.num_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta
                          : (a.num_tiles < sm_count() ? a.num_tiles : sm_count());
  launch_pdl(conv_pad<BN, SW, ROW>, dim3(grid), dim3(ROW ? NTHREADS_ROW : NTHREADS), smem, stream, bias, out, a, maps,
             tm, ty);
#ifdef ORTH_CONV_TRACE
  {
    cudaStreamSynchronize(stream);
    static unsigned long long h[160 * 32 * 4];
    cudaMemcpyFromSymbol(h, conv_trace, sizeof(h));
    double d01 = 0, d12 = 0, d23 = 0, per = 0;
    int cnt = 0, cnt2 = 0;
    static unsigned long long hc[160 * 32 * 4];
    cudaMemcpyFromSymbol(hc, conv_trace_clk, sizeof(hc));
    double c12 = 0;
    for (int c = 0; c < grid && c < 160; ++c)
      for (int t = 1; t < 16; ++t) {
        const unsigned long long* r = &h[(c * 32 + t) * 4];
        const unsigned long long* r0 = &h[(c * 32 + t - 1) * 4];
        if (!r[0] || !r[3] || !r0[3]) continue;
        d01 += (double)(r[1] - r[0]); d12 += (double)(r[2] - r[1]); d23 += (double)(r[3] - r[2]);
        c12 += (double)(hc[(c * 32 + t) * 4 + 2] - hc[(c * 32 + t) * 4 + 1]);
        per += (double)(r[3] - r0[3]);
        ++cnt;
      }
    (void)cnt2;
    if (cnt)
      std::printf("conv_pad BN=%d bres=%d TH=%d P=%d R=%d na=%d sb=%d tiles=%d grid=%d: A issue->landed %.2f, ->acc ready %.2f, epi %.2f, per-tile %.2f us, MMA span %.0f cycles (%.0f MHz)\n",
                  BN, a.bres, a.TH, a.P, a.R, a.nabuf, a.sb, a.num_tiles, grid, d01 / cnt * 1e-3, d12 / cnt * 1e-3,
                  d23 / cnt * 1e-3, per / cnt * 1e-3, c12 / cnt, 1e3 * c12 / d12);
    {
      static unsigned long long hm[160 * 4];
      cudaMemcpyFromSymbol(hm, pad_mma_trace, sizeof(hm));
      double wt = 0, wa = 0, tot = 0, nt = 0;
      for (int c = 0; c < grid && c < 160; ++c) { wt += hm[4 * c]; wa += hm[4 * c + 1]; tot += hm[4 * c + 2]; nt += hm[4 * c + 3]; }
      if (nt > 0)
        std::printf("  MMA thread per tile: %.0f cycles total, waiting for a free accumulator %.0f, for the window %.0f\n",
                    tot / nt, wt / nt, wa / nt);
      static unsigned long long zm[160 * 4];
      cudaMemcpyToSymbol(pad_mma_trace, zm, sizeof(zm));
    }
    cudaMemset(conv_trace, 0, 0);
    static unsigned long long z[160 * 32 * 4];
    cudaMemcpyToSymbol(conv_trace, z, sizeof(z));
  }
#endif
  return (int)cudaGetLastError();
}

}  // namespace

int conv_sm_count() { return sm_count(); }
bool conv_act_tmap(CUtensorMap_st* out, const void* x, int C, int W, int H, int N, int bw, int bh) {
  return make_act_tmap(out, x, C, W, H, N, bw, bh);
}

// Plan the padded-row path for a (possibly group-packed) forward layer; false
// if it does not apply (stride != 1, rows wider than one tile, channel slices
// that would cross groups, circular padding that is not a single wrap, ...).
static bool pad_args(const LayerInfo& L, int N, int H, int W, int Ho, int Wo, int& bn, PadArgs& a, bool sw) {
  const int ext = L.d * (L.k - 1);
  static const int co_max = std::getenv("ORTH_CONV_PAD_COMAX") ? std::atoi(std::getenv("ORTH_CONV_PAD_COMAX")) : 64;
  if (L.s != 1 || Wo > 128 || Wo < 16 || L.k > 7 || L.co > (sw ? 64 : co_max)) return false;
  if (L.g > 1 && L.ci % 64 != 0) return false;          // a 64-channel box must stay inside the group
  if (L.ci_f % 8 != 0) return false;                     // TMA row stride: multiple of 16 bytes
  const bool circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  const int pr = ext - L.pl;
  if (circ && (L.pl < 0 || pr < 0 || Wo != W)) return false;
  const int n = L.co;
  bn = n % 256 == 0 ? 256 : n % 128 == 0 ? 128 : n % 64 == 0 ? 64 : n % 32 == 0 ? 32 : 0;
  if (!bn) return false;
  static const char* layout_env = std::getenv("ORTH_CONV_PAD_LAYOUT");   // "window" | "copies" (A/B)
  // (1) one window of pitch P = Wo + d(k-1), tap (a, b) at row d(aP + b) (descriptor starts inside a
  //     swizzle atom cost nothing, measured); (2) k column-shifted copies of pitch round8(Wo)
  const int MT = sw ? 256 : 128;   // pixels per tile (MMA N when swapped, M otherwise)
  const int stage_row = (Wo * 128 + 1023) & ~1023;
  if (sw && L.co != 64) return false;
  for (int layout = 0; layout < 2; ++layout) {
    const bool single = layout == 0;
    if (layout_env && std::strcmp(layout_env, single ? "window" : "copies") != 0) continue;
    if (!single && circ && W % 8 != 0) continue;
    const int P = single ? Wo + ext : (circ ? W : (Wo + 7) & ~7);
    if (P > 128 + ext || P > 256) continue;
    const int TH = std::min(Ho, MT / P);
    if (TH < 1 || TH * Wo < MT / 2) continue;
    const int R = TH + ext;
    if (R > 256) continue;
    const size_t stage = sw ? (size_t)TH * stage_row + 1024 : 0;   // staged output rows + dump slots
    const int ncopy = single ? 1 : L.k;
    const int copy_bytes = R * P * 128;
    // the last window's taps read rows up to d(k-1)(P + single) + 127 past its start
    const int reach = single ? ext * (P + 1) + MT : ext * P + MT;
    const int slack_rows = std::max(0, reach - R * P);
    const size_t abuf = ((size_t)ncopy * copy_bytes + 1023) & ~size_t(1023);
    const size_t kc = (size_t)(L.ci + 63) / 64;
    int bres_bn = 0;
    for (int b = 128; b >= 64 && b * 4 >= n; b /= 2)   // N = 32 MMAs cost as much as N = 128 ones
      if (n % b == 0 && 1024 + 2 * abuf + kc * L.k * L.k * b * 128 + stage <= kSmemMax) { bres_bn = b; break; }
    static const bool no_res = std::getenv("ORTH_CONV_NO_BRES") != nullptr;   // A/B switch
    int bnl = bn;
    if (bres_bn && !no_res) bnl = bres_bn;
    if (!bres_bn || no_res) {   // streaming B needs two A buffers + a few B stages
      if (1024 + 2 * abuf + 2 * (size_t)bnl * 128 + stage > kSmemMax) continue;
    }
    bn = bnl;
    a = PadArgs{};
    a.bres = (bres_bn && !no_res) ? 1 : 0;
    a.N = N; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
    a.k = L.k; a.d = L.d; a.pt = L.pt; a.pl = L.pl; a.pr = pr;
    a.circ = circ;
    a.out_C = L.co_f; a.cr_g = L.ci; a.nout_g = L.co;
    a.P = P; a.TH = TH; a.R = R;
    a.stage_row = stage_row;
    a.slack_bytes = slack_rows * 128;
    a.tiles_h = (Ho + TH - 1) / TH;
    a.tiles_m = N * a.tiles_h;
    a.tiles_n = n / bn;
    a.num_tiles = a.tiles_m * a.tiles_n * L.g;
    a.ncopy = ncopy;
    a.copy_bytes = copy_bytes;
    a.abuf_bytes = (int)abuf;
    // bytes the window's TMA loads deliver: circular single windows fill only W + d(k-1) columns of a
    // (possibly alignment-padded) pitch P, the rest is junk that feeds junk outputs only
    a.a_tx = (circ && single) ? R * (W + ext) * 128 : ncopy * copy_bytes;
    if (circ) {
      for (int b = 0; b < ncopy; ++b) {
        int np = 0;
        if (single) {   // row = x[W - p_l, W) | x[0, W) | x[0, p_r)
          if (L.pl) { a.pc_col[3 * b + np] = W - L.pl; a.pc_dst[3 * b + np] = 0; a.pc_map[3 * b + np] = L.pl; ++np; }
          a.pc_col[3 * b + np] = 0; a.pc_dst[3 * b + np] = L.pl; a.pc_map[3 * b + np] = W; ++np;
          if (pr) { a.pc_col[3 * b + np] = 0; a.pc_dst[3 * b + np] = L.pl + W; a.pc_map[3 * b + np] = pr; ++np; }
        } else {        // copy b covers input columns (x - p_l + d b) mod W: pieces [s, W) then [0, s)
          const int s0 = ((L.d * b - L.pl) % W + W) % W;
          a.pc_col[3 * b] = s0; a.pc_dst[3 * b] = 0; a.pc_map[3 * b] = W - s0; ++np;   // pc_map: width for now
          if (s0 > 0) { a.pc_col[3 * b + 1] = 0; a.pc_dst[3 * b + 1] = W - s0; a.pc_map[3 * b + 1] = s0; ++np; }
        }
        a.npc[b] = np;
      }
    }
    return true;
  }
  return false;
}

// returns -1 when the padded-row path does not apply (caller falls back), else 0 / a CUDA error.
// flip = 1: L is the forward view of a stride-1 adjoint (see launch_conv_bwd_reuse).
int launch_conv_fwd_reuse(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                          int H, int W, int Ho, int Wo, void* stream, int flip) {
  if (((uintptr_t)x & 15) != 0 || ((uintptr_t)y & 15) != 0) return -1;
  const auto* w = static_cast<const __nv_bfloat16*>(kernel);
  auto* out = static_cast<__nv_bfloat16*>(y);
  cudaStream_t s = (cudaStream_t)stream;
  static const bool no_swap = std::getenv("ORTH_CONV_NO_SWAP") != nullptr;   // A/B switch
  // kernel-row MMAs (co_g = 64, 2 <= k <= 4, one window layout): M = 128 pixels x N = k 64.  Opt-in since
  // the issuers were made uniform: the swapped / one-chain-per-tap forms are then faster (64@56^2, batch
  // 256: 76 / 72 us vs 90 us, the kernel-row epilogue's cross-lane sums being the limit)
  static const bool use_row = std::getenv("ORTH_CONV_ROW") != nullptr;       // A/B switch
  int bn = 0;
  PadArgs a;
  if (use_row && L.co == 64 && L.k >= 2 && L.k <= 4 && L.d * (L.k - 1) < 32 &&
      pad_args(L, N, H, W, Ho, Wo, bn, a, false) && bn == 64 && a.ncopy == 1) {
    if (a.num_tiles == 0) return 0;
    a.flip = flip;
    g_conv_variant = ORTH_CV_WINDOW_ROW;
    const int e = launch_pad<64, false, true>(x, w, L.co_f, bias, out, a, L.ci_f, s);
    if (e >= 0) return e;
  }
  if (!no_swap && pad_args(L, N, H, W, Ho, Wo, bn, a, true) && bn == 64) {   // 64 channels x 256 pixels per MMA
    if (a.num_tiles == 0) return 0;
    a.flip = flip;
    g_conv_variant = ORTH_CV_WINDOW_SWAP;
    const int e = launch_pad<64, true>(x, w, L.co_f, bias, out, a, L.ci_f, s);
    if (e >= 0) return e;
  }
  if (!pad_args(L, N, H, W, Ho, Wo, bn, a, false)) return -1;
  if (a.num_tiles == 0) return 0;
  a.flip = flip;
  g_conv_variant = ORTH_CV_WINDOW;
  switch (bn) {
    case 32: return launch_pad<32, false>(x, w, L.co_f, bias, out, a, L.ci_f, s);
    case 64: return launch_pad<64, false>(x, w, L.co_f, bias, out, a, L.ci_f, s);
    case 128: return launch_pad<128, false>(x, w, L.co_f, bias, out, a, L.ci_f, s);
    default: return launch_pad<256, false>(x, w, L.co_f, bias, out, a, L.ci_f, s);
  }
}

}  // namespace orth
