// a6 (forward orthogonal convolution) for stride-1 layers with
// >= 128 output channels per group, on the tensor cores with the operands
// swapped: D^T[o][w] = sum_{c,a,b} K[o, a, b, c] * window[w + d(aP + b)][c], one
// tcgen05.mma M = 128 output channels x N = 256 window pixels x K = 16.
//
// Window.  The padded images of the batch form one stream of padded rows g = n Hp + y (Hp = Ho + d(k-1)
// rows of P = Wo + d(k-1) pixels).  A tile is TH consecutive padded rows (TH P <= 256 window pixels); its
// input window is those rows plus the d(k-1) below, one 64-channel chunk at a time, R = TH + d(k-1)
// rows x P pixels x 64 channels, SWIZZLE_128B K-major, loaded straight from the NHWC input: every padded
// row is one TMA box (zero padding: out-of-bounds columns / rows / images fill zeros) or three row pieces
// (circular: x[W - p_l, W) | x[0, W) | x[0, p_r) of the wrapped input row), the rows spread over the
// window warp's 32 lanes.  (Round 1 materialised a padded copy first; the extra pass cost ~23 us per
// cfg3 128@28 layer, ~25 % of the layer.)  The B operand of tap (a, b) is the 256 window pixels starting
// at d(aP + b) (a descriptor may start inside a swizzle atom: the tensor core
// swizzles on absolute address bits).  Window pixel w = yl P + x of padded row
// g0 + yl = n Hp + y is output (n, y, x) when y < Ho and x < Wo; other columns
// are computed and dropped.  Small images are therefore batched into one MMA
// instead of one image per tile (4x4 images: 7 per tile).
//
// Weights: the A operand, 128 output channels x 64 input channels per (chunk,
// tap) stage, streamed through a TMA ring (per tile the whole 128-channel block
// is re-read from L2; the CTA walks tiles in window-row-major order so that
// concurrently running CTAs read the same block).
//
// Epilogue: TMEM lane = output channel.  Warp q reads lanes 32q .. 32q+31 as
// mma-style 8x8 fragments (tcgen05.ld 16x256b) and writes them transposed with
// stmatrix (16 B = 8 channels of one pixel per row) into a SWIZZLE_128B staging
// area of valid output rows, two 64-channel halves; one TMA tensor store per
// (output row, half).
//
// Warp roles (256 threads, one CTA per SM, persistent over tiles):
//   warp 0 window TMA, warp 1 weight TMA, warp 2 TMEM alloc + MMA issuer,
//   warps 4-7 epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "orth_internal.h"
#include "tma_host.h"
#include "umma.cuh"

#ifdef ORTH_STACK_TRACE
// diagnostics: per CTA {MMA start, MMA end, ns waiting for windows, ns waiting for weights, epilogue end}
__device__ unsigned long long stack_trace[160 * 5];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define STRACE(...) __VA_ARGS__
#else
#define STRACE(...)
#endif

namespace orth {
namespace {

struct StackArgs {
  int N, H, W, Ho, Wo, k, d, pt, pl, circ;
  int Hp, P, TH, R;               // padded rows per image, window pitch, output rows per tile, window rows
  int in_C, out_C, cr_g, nout_g;  // input / output channels (whole tensor), per group
  int tiles_m, tiles_n, num_tiles;
  int abuf_bytes, nabuf, sb;      // window ring, weight ring stages
  int stage_off, stage_row, stage_half, slots;
  int flip;                       // weight tap t read from row k^2-1-t (stride-1 adjoint, forward form)
  // window rows straight from the unpadded NHWC input (no padded copy): per padded row, npc TMA row
  // pieces (map pc_map, input column pc_col, window column pc_dst); circular: the wrapped halves
  int npc, pc_map[3], pc_col[3], pc_dst[3];
};
struct StackMaps {
  CUtensorMap m[3];   // 4-D (C, W, H, N) maps, box 64 ch x width x 1 row x 1 image, one per piece width
};

constexpr int NTHREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int MAX_AB = 4;
constexpr int MAX_SB = 8;
constexpr int W_BYTES = 128 * 128;   // one weight stage: 128 output channels x 64 input channels
constexpr size_t kSmemMax = 227 * 1024 - 1024;

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// padded[n][yy][xx][c] = x~[n][yy - p_t][xx - p_l][c] (circular: mod H, W; zeros outside), 8 channels
// (16 B) per thread; rows of the whole batch back to back
// one CTA per padded row (n, yy): its source row is resolved once (32-bit math per 16-byte element,
// no 64-bit divisions), the P x C/8 16-byte chunks of the row are stored contiguously (coalesced)
__global__ void __launch_bounds__(256) pad_kernel(const uint4* __restrict__ x, uint4* __restrict__ out, int N, int H,
                                                  int W, int C8, int Hp, int P, int pt, int pl, int circ) {
  const int64_t row = blockIdx.x;                 // n * Hp + yy
  const int n = (int)(row / Hp), yy = (int)(row - (int64_t)n * Hp);
  int h = yy - pt;
  bool hok = true;
  if (circ) h = wrapi(h, H);
  else hok = h >= 0 && h < H;
  const uint4* src = x + ((int64_t)n * H + (hok ? h : 0)) * W * C8;
  uint4* dst = out + row * (int64_t)P * C8;
  const int per = P * C8;
  for (int e = threadIdx.x; e < per; e += 256) {
    const int xx = e / C8, c = e - xx * C8;
    int w = xx - pl;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (circ) {
      w = wrapi(w, W);
      v = __ldg(src + w * C8 + c);
    } else if (hok && w >= 0 && w < W) {
      v = __ldg(src + w * C8 + c);
    }
    dst[e] = v;
  }
}

// valid output rows in padded rows [0, g)
__device__ __forceinline__ int valid_before(int g, int Hp, int Ho) { return (g / Hp) * Ho + min(g % Hp, Ho); }

__global__ void __launch_bounds__(NTHREADS, 1)
    conv_stack(const float* __restrict__ bias, const __grid_constant__ StackArgs a,
               const __grid_constant__ StackMaps tmA, const __grid_constant__ CUtensorMap tmW,
               const __grid_constant__ CUtensorMap tmY) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t a_full[MAX_AB], a_empty[MAX_AB], b_full[MAX_SB], b_empty[MAX_SB], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NA = a.nabuf, SB = a.sb;
  if (warp == 2) umma::tmem_alloc(&tmem_base_sh, 512);
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
      umma::mbar_init(&tempty_bar[i], 128);
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t abase = umma::smem_u32(smem);
  const uint32_t wbase = abase + NA * a.abuf_bytes;
  const int kk2 = a.k * a.k;
  // tile -> (first padded row, 128-channel block, group); window-row tiles fastest
  auto decode = [&](int tile, int& g0, int& n0, int& grp) {
    const int tm = tile % a.tiles_m, rest = tile / a.tiles_m;
    n0 = (rest % a.tiles_n) * 128;
    grp = rest / a.tiles_n;
    g0 = tm * a.TH;
  };

  if (warp == 0) {
    // -------------------------------------------------------------- window producer (whole warp)
    // R padded rows x P pixels x 64 channels straight from the NHWC input: padded row g = n Hp + yy is
    // input row yy - p_t (circular: wrapped; zeros / past the batch: out of bounds -> zero fill), each as
    // its npc row pieces; the rows are spread over the 32 lanes (lane 0 posts the byte count first).
    if (lane < a.npc) umma::tma_prefetch_desc(&tmA.m[a.pc_map[lane]]);
    int u = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      int g0, n0, grp;
      decode(tile, g0, n0, grp);
      for (int c0 = 0; c0 < a.cr_g; c0 += 64, ++u) {
        const int ab = u % NA;
        if (lane == 0) {
          if (u >= NA) umma::mbar_wait(&a_empty[ab], ((u / NA) - 1) & 1);
          umma::mbar_arrive_expect_tx(&a_full[ab], (uint32_t)(a.R * a.P * 128));
        }
        __syncwarp();
        const uint32_t dst = abase + ab * a.abuf_bytes;
        const int c = grp * a.cr_g + c0;
        for (int y = lane; y < a.R; y += 32) {
          const int g = g0 + y, n = g / a.Hp, yy = g - n * a.Hp;
          int h = yy - a.pt;
          if (a.circ) { h %= a.H; if (h < 0) h += a.H; }
          const uint32_t row = dst + (uint32_t)(y * a.P) * 128u;
          for (int pc = 0; pc < a.npc; ++pc)
            umma::tma_load_4d(row + (uint32_t)a.pc_dst[pc] * 128u, &tmA.m[a.pc_map[pc]], &a_full[ab], c, a.pc_col[pc],
                              h, n);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ weight producer
      umma::tma_prefetch_desc(&tmW);
      int i = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        int g0, n0, grp;
        decode(tile, g0, n0, grp);
        for (int c0 = 0; c0 < a.cr_g; c0 += 64)
          for (int tap = 0; tap < kk2; ++tap, ++i) {
            const int st = i % SB;
            if (i >= SB) umma::mbar_wait(&b_empty[st], ((i / SB) - 1) & 1);
            umma::mbar_arrive_expect_tx(&b_full[st], W_BYTES);
            umma::tma_load_3d(wbase + st * W_BYTES, &tmW, &b_full[st], c0, a.flip ? kk2 - 1 - tap : tap,
                              grp * a.nout_g + n0);
          }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      // Kept warp-uniform for ptxas (see conv_pad.cu, ROW issuers): bases and the tile range derived
      // here, rings stepped, descriptors advanced by adds (16-byte units).
      constexpr uint32_t IDESC = umma::idesc_bf16(128, 256);
      const uint32_t ubase = umma::smem_base1024_u32(smem_raw);
      const uint64_t a_desc0 = umma::sdesc_sw128(ubase);
      const uint64_t w_desc0 = a_desc0 + (uint32_t)a.nabuf * ((uint32_t)a.abuf_bytes >> 4);
      const uint32_t abuf16 = (uint32_t)a.abuf_bytes >> 4, row16 = (uint32_t)(a.d * a.P) * 8u, col16 = (uint32_t)a.d * 8u;
      int ab = 0, aph = 0, st = 0, bph = 0, tcount = 0;
      STRACE(unsigned long long wa = 0, wb = 0; const unsigned long long t_start = gtime();)
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
        const int acc = tcount & 1;
        umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
        umma::tc_fence_after();
        const uint32_t d_tmem = tmem_base_sh + acc * 256;
        for (int c0 = 0; c0 < a.cr_g; c0 += 64) {
          STRACE(const unsigned long long t0a = gtime();)
          umma::mbar_wait(&a_full[ab], aph);
          STRACE(wa += gtime() - t0a;)
          umma::tc_fence_after();
          uint64_t brow = a_desc0 + ab * abuf16;   // window row of kernel row ta
          for (int ta = 0; ta < a.k; ++ta, brow += row16) {
            uint64_t bw = brow;
            for (int tb = 0; tb < a.k; ++tb, bw += col16) {
              STRACE(const unsigned long long t0b = gtime();)
              umma::mbar_wait(&b_full[st], bph);
              STRACE(wb += gtime() - t0b;)
              umma::tc_fence_after();
              const uint64_t aw = w_desc0 + st * (uint32_t)(W_BYTES >> 4);
              const uint32_t acc0 = (c0 | ta | tb) != 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) umma::mma_bf16(d_tmem, aw + 2 * q, bw + 2 * q, IDESC, acc0 | (q != 0));
              umma::mma_commit(&b_empty[st]);
              if (++st == SB) { st = 0; bph ^= 1; }
            }
          }
          umma::mma_commit(&a_empty[ab]);
          if (++ab == NA) { ab = 0; aph ^= 1; }
        }
        umma::mma_commit(&tfull_bar[acc]);
      }
      STRACE(stack_trace[blockIdx.x * 5 + 0] = t_start; stack_trace[blockIdx.x * 5 + 1] = gtime();
             stack_trace[blockIdx.x * 5 + 2] = wa; stack_trace[blockIdx.x * 5 + 3] = wb;)
    }
    __syncwarp();
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const uint32_t s_base = umma::smem_u32(smem + a.stage_off);
    const uint32_t dump = s_base + (uint32_t)(2 * a.stage_half) + (uint32_t)lane * 16u;
    const int m = lane >> 3, jrow = lane & 7;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
      int g0, n0, grp;
      decode(tile, g0, n0, grp);
      const int acc = tcount & 1;
      const int v0 = valid_before(g0, a.Hp, a.Ho);
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      if (tid == EPI_WARP0 * 32) umma::bulk_wait_read0();   // the previous tile's stores have read the staging
      umma::named_bar_sync(2, 128);
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {   // TMEM lanes 32q + 16 hf .. + 15 = channels
        const int ch0 = 32 * q + 16 * hf;
        const int ob = grp * a.nout_g + n0 + ch0 + (lane >> 2);
        const float b_lo = bias ? bias[ob] : 0.f, b_hi = bias ? bias[ob + 8] : 0.f;
        const uint32_t chunk = (uint32_t)(((ch0 >> 3) + (m & 1)) & 7);   // 16-B chunk in the 128-B half row
        const uint32_t half_off = (uint32_t)((ch0 >> 6) * a.stage_half);
#pragma unroll 1
        for (int c = 0; c < 256; c += 32) {
          uint32_t r[16];
          umma::tmem_ld_16x256b_x4(tmem + ((uint32_t)(32 * q + 16 * hf) << 16) + (uint32_t)(acc * 256 + c), r);
          umma::tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int w = c + 16 * h + 8 * (m >> 1) + jrow;   // window pixel this lane addresses
            const int yl = w / a.P, x = w - yl * a.P;
            const int gg = g0 + yl, n = gg / a.Hp, y = gg - n * a.Hp;
            uint32_t dst = dump;
            if (yl < a.TH && x < a.Wo && y < a.Ho && n < a.N) {
              const int slot = valid_before(gg, a.Hp, a.Ho) - v0;
              dst = s_base + half_off + (uint32_t)(slot * a.stage_row + x * 128) + ((chunk ^ (uint32_t)(x & 7)) << 4);
            }
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
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
      umma::fence_proxy_async_smem();   // staging writes -> TMA (async proxy) reads
      umma::named_bar_sync(2, 128);
      if (tid == EPI_WARP0 * 32) {
        for (int yl = 0; yl < a.TH; ++yl) {   // one store per (valid output row, 64-channel half)
          const int gg = g0 + yl, n = gg / a.Hp, y = gg - n * a.Hp;
          if (y >= a.Ho || n >= a.N) continue;
          const uint32_t src = s_base + (uint32_t)((valid_before(gg, a.Hp, a.Ho) - v0) * a.stage_row);
          umma::tma_store_3d(&tmY, src, grp * a.nout_g + n0, 0, n * a.Ho + y);
          umma::tma_store_3d(&tmY, src + (uint32_t)a.stage_half, grp * a.nout_g + n0 + 64, 0, n * a.Ho + y);
        }
        umma::bulk_commit();
      }
    }
    if (tid == EPI_WARP0 * 32) umma::bulk_wait0();
    STRACE(if (tid == EPI_WARP0 * 32) stack_trace[blockIdx.x * 5 + 4] = gtime();)
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 2) umma::tmem_dealloc(tmem, 512);
}

// host: plan one layer; false = not applicable
bool stack_args(const LayerInfo& L, int N, int H, int W, int Ho, int Wo, StackArgs& a) {
  const int ext = L.d * (L.k - 1);
  if (L.s != 1 || L.k > 7 || L.co % 128 != 0) return false;
  if (L.g > 1 && L.ci % 64 != 0) return false;   // a 64-channel box must stay inside the group
  if (L.ci_f % 8 != 0 || L.co_f % 8 != 0) return false;
  const bool circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  const int pr = ext - L.pl;
  if (circ && (L.pl < 0 || pr < 0 || Wo != W || Ho != H)) return false;
  if (L.pt < 0 || L.pl < 0) return false;
  const int P = Wo + ext;
  if (P > 256 || Wo < 1) return false;
  if (L.ci_f % 8 != 0) return false;
  const int TH = 256 / P;
  const int Hp = Ho + ext;
  a = StackArgs{};
  a.N = N; a.H = H; a.W = W; a.Ho = Ho; a.Wo = Wo;
  a.k = L.k; a.d = L.d; a.pt = L.pt; a.pl = L.pl; a.circ = circ;
  a.Hp = Hp; a.P = P; a.TH = TH; a.R = TH + ext;
  if (W > 256) return false;   // TMA box width
  // window row pieces (pc_map holds the piece width here; launch_conv_fwd_stack turns it into a map index)
  a.npc = 0;
  if (circ) {   // row = x[W - p_l, W) | x[0, W) | x[0, p_r)
    if (L.pl) { a.pc_col[a.npc] = W - L.pl; a.pc_dst[a.npc] = 0; a.pc_map[a.npc] = L.pl; ++a.npc; }
    a.pc_col[a.npc] = 0; a.pc_dst[a.npc] = L.pl; a.pc_map[a.npc] = W; ++a.npc;
    if (pr) { a.pc_col[a.npc] = 0; a.pc_dst[a.npc] = L.pl + W; a.pc_map[a.npc] = pr; ++a.npc; }
  } else {      // one P-wide box from column -p_l: the padding columns are out of bounds (zero fill)
    a.pc_col[0] = -L.pl; a.pc_dst[0] = 0; a.pc_map[0] = P; a.npc = 1;
  }
  a.in_C = L.ci_f; a.out_C = L.co_f; a.cr_g = L.ci; a.nout_g = L.co;
  const long long rows = (long long)N * Hp;
  a.tiles_m = (int)((rows + TH - 1) / TH);
  a.tiles_n = L.co / 128;
  const long long nt = (long long)a.tiles_m * a.tiles_n * L.g;
  if (nt > (1LL << 30)) return false;
  a.num_tiles = (int)nt;
  // staging: valid output rows of one tile (max over the Hp-periodic tile offsets), 1024-aligned rows
  int slots = 0;
  for (int g0 = 0; g0 < Hp * TH && g0 < Hp * 256; g0 += TH) {
    auto vb = [&](int g) { return (g / Hp) * Ho + std::min(g % Hp, Ho); };
    slots = std::max(slots, vb(g0 + TH) - vb(g0));
  }
  a.slots = slots;
  a.stage_row = (Wo * 128 + 1023) & ~1023;
  a.stage_half = slots * a.stage_row;
  // shared memory: window ring + weight ring + two staging halves + dump slots
  a.abuf_bytes = (a.R * P * 128 + 1023) & ~1023;
  const size_t stage = (size_t)2 * a.stage_half + 1024;
  const size_t slack = (size_t)std::max(0, ext * (P + 1) + 256 - a.R * P) * 128;   // last taps read past a window
  // the weight ring is the latency-critical stream (a whole 128-channel block per tile): give it up to
  // MAX_SB stages first (measured: 2 stages starve the MMA at ~25 GB/s per SM), then extra window buffers
  if (1024 + 2 * (size_t)a.abuf_bytes + 2 * (size_t)W_BYTES + stage > kSmemMax) return false;
  const size_t room = kSmemMax - 1024 - stage - 2 * (size_t)a.abuf_bytes;
  a.sb = (int)std::min<size_t>(MAX_SB, room / W_BYTES);
  int na = 2;
  while (na < MAX_AB && (size_t)(na - 1) * a.abuf_bytes + (size_t)a.sb * W_BYTES <= room) ++na;
  a.nabuf = na;
  a.stage_off = na * a.abuf_bytes + a.sb * W_BYTES;
  if ((size_t)a.sb * W_BYTES + stage < slack) return false;   // the last window's over-read stays in smem
  return true;
}

}  // namespace

// padded copy of x (N x Hp x P x C, rows of the whole batch back to back) into the layer's scratch;
// -1 if it does not fit
int launch_pad_input(const LayerInfo& L, const void* x, int N, int H, int W, int Hp, int P, void* stream) {
  const int64_t elems = (int64_t)N * Hp * P * L.ci_f;
  if (!L.pad_scratch || elems * 2 > L.pad_bytes || L.ci_f % 8 != 0) return -1;
  pad_kernel<<<(unsigned)((int64_t)N * Hp), 256, 0, (cudaStream_t)stream>>>((const uint4*)x, (uint4*)L.pad_scratch, N, H, W, L.ci_f / 8,
                                                      Hp, P, L.pt, L.pl,
                                                      L.desc.padding_mode == ORTH_PAD_CIRCULAR ? 1 : 0);
  return (int)cudaGetLastError();
}

static bool stack_rule(const LayerInfo& L, int Ho, int Wo) {
  static const bool force = std::getenv("ORTH_CONV_STACK") != nullptr;
  static const bool off = std::getenv("ORTH_CONV_NO_STACK") != nullptr;
  if (off) return false;
  return force || (L.co == 128 && Wo >= 16 && Ho >= 16);
}

// the windows come straight from the input (TMA row pieces): no padded copy, no scratch
int64_t conv_stack_pad_bytes(const LayerInfo&, int, int, int, int, int) { return 0; }

int launch_conv_fwd_stack(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                          int H, int W, int Ho, int Wo, void* stream, int flip) {
  // Default where it measured faster than the gather conv: 128 output channels per group on images
  // >= 16 px (B200, no padded copy: cfg3 128@28 75 vs 98 us, cfg2 128@16 41-43 vs 45 us); 256 / 512
  // channels on small images lose (cfg3 256@14 80 vs 59 us, cfg2 512@4 63 vs 35 us: padded columns waste
  // MMA work).  ORTH_CONV_STACK=1 forces it wherever it applies, ORTH_CONV_NO_STACK=1 turns it off.
  if (!stack_rule(L, Ho, Wo)) return -1;
  if (((uintptr_t)x & 15) != 0 || ((uintptr_t)y & 15) != 0) return -1;
  StackArgs a;
  if (!stack_args(L, N, H, W, Ho, Wo, a)) return -1;
  if (a.num_tiles == 0) return 0;
  a.flip = flip;
  g_conv_variant = ORTH_CV_STACK;
  cudaStream_t s = (cudaStream_t)stream;
  StackMaps ta;   // one (C, W, H, N) map per distinct piece width: box 64 ch x width x 1 row x 1 image
  std::memset(&ta, 0, sizeof(ta));
  {
    int widths[3], nw = 0;
    for (int pc = 0; pc < a.npc; ++pc) {
      const int w0 = a.pc_map[pc];
      int m = 0;
      while (m < nw && widths[m] != w0) ++m;
      if (m == nw) {
        widths[nw++] = w0;
        if (!conv_act_tmap(&ta.m[m], x, a.in_C, W, H, N, w0, 1)) return (int)cudaErrorInvalidValue;
      }
      a.pc_map[pc] = m;
    }
  }
  CUtensorMap tw;
  if (!make_weight_tmap(&tw, kernel, L.co_f, L.k * L.k, L.ci, 128)) return (int)cudaErrorInvalidValue;
  CUtensorMap ty;
  {   // output (C, Wo, N*Ho): one output row x 64 channels per box, SWIZZLE_128B staging
    auto enc = tensor_map_encoder();
    const cuuint64_t dims[3] = {(cuuint64_t)a.out_C, (cuuint64_t)Wo, (cuuint64_t)N * Ho};
    const cuuint64_t strides[2] = {(cuuint64_t)a.out_C * 2, (cuuint64_t)Wo * a.out_C * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)Wo, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    std::memset(&ty, 0, sizeof(ty));
    if (!enc || enc(&ty, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return (int)cudaErrorInvalidValue;
  }
  const size_t smem = 1024 + (size_t)a.stage_off + 2 * (size_t)a.stage_half + 1024;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(conv_stack, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return (int)cudaGetLastError();
    attr = smem;
  }
  const int grid = std::min(a.num_tiles, conv_sm_count());
  conv_stack<<<grid, NTHREADS, smem, s>>>(bias, a, ta, tw, ty);
#ifdef ORTH_STACK_TRACE
  {
    cudaStreamSynchronize(s);
    static unsigned long long h[160 * 5];
    cudaMemcpyFromSymbol(h, stack_trace, sizeof(h));
    unsigned long long t0 = ~0ull, t1 = 0, t2 = 0;
    double wa = 0, wb = 0, span = 0;
    for (int c = 0; c < grid && c < 160; ++c) {
      t0 = std::min(t0, h[c * 5]);
      t1 = std::max(t1, h[c * 5 + 1]);
      t2 = std::max(t2, h[c * 5 + 4]);
      wa += h[c * 5 + 2];
      wb += h[c * 5 + 3];
      span += h[c * 5 + 1] - h[c * 5];
    }
    std::printf("conv_stack tiles=%d grid=%d TH=%d P=%d R=%d na=%d sb=%d: MMA-thread span %.1f us (wait windows %.1f, "
                "weights %.1f), last MMA %.1f, last epilogue %.1f us after first start\n", a.num_tiles, grid, a.TH, a.P,
                a.R, a.nabuf, a.sb, span / grid * 1e-3, wa / grid * 1e-3, wb / grid * 1e-3, (t1 - t0) * 1e-3,
                (t2 - t0) * 1e-3);
  }
#endif
  return (int)cudaGetLastError();
}

}  // namespace orth
