// a6 (forward orthogonal convolution) for stride-1 layers as an
// implicit GEMM whose operands are loaded ONLY by TMA.
//
// The input is first copied padded (circular wrap or zeros, `launch_pad_input`)
// into the plan's conv scratch as a (C, P, Hp, N) tensor, P = Wo + d(k-1),
// Hp = Ho + d(k-1).  A tile is M = 128 output pixels = NI images x TH rows x Wo
// columns; for tap (a, b) and 64-channel chunk c its im2col A block is then the
// single 4-D box {64 ch, Wo, TH, NI} at (c, d b, y0 + d a, n0) of the padded
// tensor, which lands in shared memory exactly as the 128-row SWIZZLE_128B
// K-major operand (row = ((i TH) + y) Wo + x).  The weight tile of the tap is
// one 3-D box {64, 1, BN}.  So one thread issues two TMA loads per K block where
// the gather kernel (conv_tc.cu) has 8 producer warps issuing 1024 16-byte
// cp.async (its MMA warp waits 34% of the time) -- yet the layer times came out
// the same: both are bound by the shared-memory port.  Opt-in (see below).
//
// Warp roles (256 threads, one CTA per SM, persistent): warp 0 TMA producer,
// warp 1 TMEM owner + MMA issuer (M = 128, N = BN, two TMEM accumulators),
// warps 4-7 epilogue (thread = output pixel row, BN channels as 16-byte stores).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "orth_internal.h"
#include "pdl.h"
#include "tma_host.h"
#include "umma.cuh"

#ifdef ORTH_EXPERIMENTAL   // measured no faster than conv_ws: built only with ORTH_EXPERIMENTAL=1
namespace orth {
namespace {

struct TmaConvArgs {
  int N, Ho, Wo, k, d;
  int NI, TH;                     // images and output rows per tile (NI * TH * Wo <= 128)
  int out_C, cr_g, nout_g;
  int tiles_y, tiles_m, tiles_n, num_tiles;
  int sb, flip;
};

constexpr int NTHREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int MAX_SB = 8;
constexpr size_t kSmemMax = 227 * 1024 - 1024;

template <int BN>
__global__ void __launch_bounds__(NTHREADS, 1)
    conv_tma(const float* __restrict__ bias, __nv_bfloat16* __restrict__ out, const __grid_constant__ TmaConvArgs a,
             const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  umma::griddep_launch_dependents();
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t full_bar[MAX_SB], empty_bar[MAX_SB], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int SB = a.sb;
  if (warp == 1) umma::tmem_alloc(&tmem_base_sh, 2 * BN);
  if (tid == 0) {
    for (int i = 0; i < SB; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
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
  umma::griddep_wait();   // PDL: the padded input and the weights are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int kk2 = a.k * a.k;
  const int mrows = a.NI * a.TH * a.Wo;
  auto decode = [&](int tile, int& n0, int& y0, int& c_n0, int& g) {
    const int tm = tile % a.tiles_m, rest = tile / a.tiles_m;
    c_n0 = (rest % a.tiles_n) * BN;
    g = rest / a.tiles_n;
    n0 = (tm / a.tiles_y) * a.NI;
    y0 = (tm % a.tiles_y) * a.TH;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      umma::tma_prefetch_desc(&tmA);
      umma::tma_prefetch_desc(&tmB);
      int i = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
        int n0, y0, c_n0, g;
        decode(tile, n0, y0, c_n0, g);
        for (int c0 = 0; c0 < a.cr_g; c0 += 64)
          for (int tap = 0; tap < kk2; ++tap, ++i) {
            const int st = i % SB;
            if (i >= SB) umma::mbar_wait(&empty_bar[st], ((i / SB) - 1) & 1);
            const int ta = tap / a.k, tb = tap - ta * a.k;
            const uint32_t sa = s0 + st * STAGE;
            umma::mbar_arrive_expect_tx(&full_bar[st], (uint32_t)(mrows * 128 + B_BYTES));
            umma::tma_load_4d(sa, &tmA, &full_bar[st], g * a.cr_g + c0, a.d * tb, y0 + a.d * ta, n0);
            umma::tma_load_3d(sa + A_BYTES, &tmB, &full_bar[st], c0, a.flip ? kk2 - 1 - tap : tap,
                              g * a.nout_g + c_n0);
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = umma::idesc_bf16(128, BN);
      int i = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
        const int acc = tcount & 1;
        umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
        umma::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int c0 = 0; c0 < a.cr_g; c0 += 64)
          for (int tap = 0; tap < kk2; ++tap, ++i) {
            const int st = i % SB;
            umma::mbar_wait(&full_bar[st], (i / SB) & 1);
            umma::tc_fence_after();
            const uint32_t sa = s0 + st * STAGE;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              umma::mma_bf16(d_tmem, umma::sdesc_sw128(sa + 32 * q), umma::sdesc_sw128(sa + A_BYTES + 32 * q), IDESC,
                             (c0 | tap | q) != 0);
            umma::mma_commit(&empty_bar[st]);
          }
        umma::mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------------------ epilogue: thread = output pixel row
    const int q = warp & 3, r = q * 32 + lane;
    const int per_img = a.TH * a.Wo;
    const int ii = r / per_img, rem = r - ii * per_img, yy = rem / a.Wo, xx = rem - yy * a.Wo;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
      int n0, y0, c_n0, g;
      decode(tile, n0, y0, c_n0, g);
      const int n = n0 + ii, y = y0 + yy;
      const int64_t opix = (r < mrows && n < a.N && y < a.Ho) ? ((int64_t)n * a.Ho + y) * a.Wo + xx : -1;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      const int obase = g * a.nout_g + c_n0;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
        if (opix >= 0) {
          const int o = obase + cc;
          uint4* dst = reinterpret_cast<uint4*>(out + opix * a.out_C + o);
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
            dst[i4] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tmem, 2 * BN);
}

template <int BN>
int launch_tma(const LayerInfo& L, const void* kernel, const float* bias, void* y, TmaConvArgs& a, int Hp, int P,
               cudaStream_t s) {
  constexpr size_t STAGE = 128 * 128 + (size_t)BN * 128;
  a.sb = (int)std::min<size_t>(MAX_SB, (kSmemMax - 1024) / STAGE);
  if (a.sb < 2) return -1;
  const size_t smem = 1024 + (size_t)a.sb * STAGE;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(conv_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return (int)cudaGetLastError();
    attr = smem;
  }
  CUtensorMap ta;   // padded input (C, P, Hp, N): box 64 ch x Wo x TH x NI, SWIZZLE_128B
  {
    auto enc = tensor_map_encoder();
    const cuuint64_t dims[4] = {(cuuint64_t)L.ci_f, (cuuint64_t)P, (cuuint64_t)Hp, (cuuint64_t)a.N};
    const cuuint64_t strides[3] = {(cuuint64_t)L.ci_f * 2, (cuuint64_t)P * L.ci_f * 2,
                                   (cuuint64_t)Hp * P * L.ci_f * 2};
    const cuuint32_t box[4] = {64, (cuuint32_t)a.Wo, (cuuint32_t)a.TH, (cuuint32_t)a.NI};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    std::memset(&ta, 0, sizeof(ta));
    if (!enc || enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, L.pad_scratch, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return (int)cudaErrorInvalidValue;
  }
  CUtensorMap tb;
  if (!make_weight_tmap(&tb, kernel, L.co_f, L.k * L.k, L.ci, BN)) return (int)cudaErrorInvalidValue;
  const int grid = std::min(a.num_tiles, conv_sm_count());
  return (int)launch_pdl(conv_tma<BN>, dim3(grid), dim3(NTHREADS), smem, s, bias, (__nv_bfloat16*)y, a, ta, tb);
}

}  // namespace

int launch_conv_fwd_tma(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                        int H, int W, int Ho, int Wo, void* stream, int flip) {
  // Opt-in (ORTH_CONV_TMA=1): measured on B200 it matches the gather kernel on 128@16, 512@7 and
  // 512@4 and loses on 256@8 / 256@14 (31.6 vs 25.9, 81.8 vs 62.7 us) -- removing the gather producers
  // did not move the MMA rate, which is bound by the shared-memory port (operand reads + TMA writes).
  static const bool on = std::getenv("ORTH_CONV_TMA") != nullptr;
  if (!on || !L.pad_scratch) return -1;
  if (L.s != 1 || L.k > 7 || Wo > 128 || Wo < 1 || Ho < 1) return -1;
  if (L.g > 1 && L.ci % 64 != 0) return -1;       // a 64-channel box must stay inside the group
  if (L.ci_f % 8 != 0 || L.co_f % 8 != 0 || ((uintptr_t)y & 15) != 0) return -1;
  const int BN = L.co % 256 == 0 ? 256 : L.co % 128 == 0 ? 128 : 0;
  if (!BN) return -1;
  if (L.desc.padding_mode == ORTH_PAD_CIRCULAR && (Ho != H || Wo != W)) return -1;
  const int ext = L.d * (L.k - 1);
  const int P = Wo + ext, Hp = Ho + ext;
  TmaConvArgs a{};
  a.N = N; a.Ho = Ho; a.Wo = Wo; a.k = L.k; a.d = L.d; a.flip = flip;
  if (Ho * Wo >= 128) { a.NI = 1; a.TH = std::max(1, 128 / Wo); }
  else { a.TH = Ho; a.NI = std::max(1, 128 / (Ho * Wo)); }
  if (a.NI * a.TH * a.Wo < 64) return -1;          // mostly empty tiles: leave it to the gather kernel
  a.out_C = L.co_f; a.cr_g = L.ci; a.nout_g = L.co;
  a.tiles_y = (Ho + a.TH - 1) / a.TH;
  a.tiles_m = ((N + a.NI - 1) / a.NI) * a.tiles_y;
  a.tiles_n = L.co / BN;
  const long long nt = (long long)a.tiles_m * a.tiles_n * L.g;
  if (nt > (1LL << 30)) return -1;
  a.num_tiles = (int)nt;
  if (a.num_tiles == 0) return 0;
  if (int e = launch_pad_input(L, x, N, H, W, Hp, P, stream)) return e < 0 ? -1 : e;
  g_conv_variant = ORTH_CV_TMA;
  cudaStream_t s = (cudaStream_t)stream;
  return BN == 256 ? launch_tma<256>(L, kernel, bias, y, a, Hp, P, s) : launch_tma<128>(L, kernel, bias, y, a, Hp, P, s);
}

}  // namespace orth
#else
namespace orth {
int launch_conv_fwd_tma(const LayerInfo&, const void*, const float*, const void*, void*, int, int, int, int, int,
                        void*, int) {
  return -1;
}
}  // namespace orth
#endif

