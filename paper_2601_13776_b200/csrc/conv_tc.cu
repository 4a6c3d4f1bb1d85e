// a6 on the 5th-generation tensor cores: implicit-GEMM conv forward, BF16 in,
// FP32 accumulation in TMEM, BF16 out (P:122 forward "single call", P:332-338
// stride / dilation / groups; circular or zero padding, reading R11).
//
// GEMM view per group g: D[M = N*Ho*Wo pixels, N = co_g] = A[M, K] B[N, K]^T with
// K = (tap, channel), A[m, (a,b,c)] = x~[n, s*u + d*a - p_t, s*v + d*b - p_l, g*ci_g + c]
// and B = the BF16 GEMM-layout kernel (C_o, k, k, C_i/g), already K-major.
//
// Persistent, warp-specialised kernel (one CTA per SM, 416 threads):
//   warps 0-7   producers.  Per tile they first build a (tap, row) -> input
//               pixel table in shared memory (-1 = zero padding; circular
//               padding wraps here), so the per-stage gather is a table read
//               plus a 16-byte cp.async per (row, 8-channel chunk) into an
//               S-stage SWIZZLE_128B ring (zero-fill for padding / tails).
//               After cp.async.wait_group + fence.proxy.async they arrive on
//               the stage's `full` mbarrier, LAG stages behind.
//   warp 8      TMEM allocation + one thread issuing tcgen05.mma (M=128, N=BN,
//               K=16, x4 per stage) into one of two TMEM accumulators,
//               committing to the stage's `empty` barrier and, per tile, `tfull`.
//   warps 9-12  epilogue: tcgen05.ld of their 32-lane quarter, bias, RNE to
//               BF16, NHWC stores; arrive on `tempty`.
// The accumulator is double-buffered, so the epilogue of tile t overlaps the
// mainloop of tile t+1.  (Measured: a single producer warp per SM sub-partition
// was instruction-latency bound at ~2.5k cycles per stage; the table cuts the
// per-row work to a load, a compare and an address multiply.)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "orth_internal.h"
#include "umma.cuh"
#include "tma_host.h"

namespace orth {
namespace {

struct TcConvArgs {
  int N, H, W, Ci, Co, ci_g, co_g, k, s, d, pt, pl, Ho, Wo, circ;
  int tiles_m, tiles_n, num_tiles;
};

constexpr int NPROD = 256;                 // producer threads (warps 0-7)
constexpr int MMA_WARP = 8;
constexpr int NTHREADS = NPROD + 32 + 128;
constexpr int MAX_TAPS = 49;               // k <= 7

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

template <int BN, int S>
__global__ void __launch_bounds__(NTHREADS, 1)
    conv_fwd_ws(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                const float* __restrict__ bias, __nv_bfloat16* __restrict__ y, TcConvArgs a,
                const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int A_BYTES = 128 * 128, B_BYTES = BN * 128, STAGE = A_BYTES + B_BYTES;
  constexpr int LAG = S - 2;   // stages of cp.async kept in flight per producer thread
  int* tab = reinterpret_cast<int*>(smem + S * STAGE);   // [taps][128] input pixel index, -1 = padding
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == MMA_WARP) umma::tmem_alloc(&tmem_base_sh, 2 * BN);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], NPROD + 1);   // + the TMA issuer's expect_tx arrival
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
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int kc = (a.ci_g + 63) / 64;
  const int kk2 = a.k * a.k;
  const int nk = kk2 * kc;
  const int M = a.N * a.Ho * a.Wo;
  const int hw = a.Ho * a.Wo;

  if (warp < MMA_WARP) {
    // ------------------------------------------------------------ producers
    const int c = tid & 7, rbase = tid >> 3;   // A rows rbase + 32 i
    if (tid == 0) umma::tma_prefetch_desc(&tmB);
    const uint32_t tab_s = umma::smem_u32(tab);
    int it = 0, st = 0, ph = 0;                // ring position of k-block `it`
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x) {
      const int tm = tile % a.tiles_m, rest = tile / a.tiles_m;
      const int tn = rest % a.tiles_n, g = rest / a.tiles_n;
      const int m0 = tm * 128, n0 = tn * BN;
      umma::named_bar_sync(1, NPROD);          // everyone is done reading the previous table
      for (int e = tid; e < 128 * kk2; e += NPROD) {
        const int r = e & 127, t = e >> 7;
        const int m = m0 + r;
        int v = -1;
        if (m < M) {
          const int n = m / hw, rr = m - n * hw;
          const int u = rr / a.Wo, vv = rr - u * a.Wo;
          int h = u * a.s - a.pt + a.d * (t / a.k), ww = vv * a.s - a.pl + a.d * (t % a.k);
          bool ok = true;
          if (a.circ) {
            h = wrapi(h, a.H);
            ww = wrapi(ww, a.W);
          } else {
            ok = h >= 0 && h < a.H && ww >= 0 && ww < a.W;
          }
          if (ok) v = (n * a.H + h) * a.W + ww;
        }
        tab[t * 128 + r] = v;
      }
      umma::named_bar_sync(1, NPROD);
      const __nv_bfloat16* xg = x + (int64_t)g * a.ci_g + c * 8;
      const uint32_t off_r[4] = {umma::sw128_off(rbase, c), umma::sw128_off(rbase + 32, c),
                                 umma::sw128_off(rbase + 64, c), umma::sw128_off(rbase + 96, c)};
      for (int tap = 0; tap < kk2; ++tap) {
        const uint32_t trow = tab_s + (uint32_t)(tap * 128 + rbase) * 4u;
        int pix[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pix[i] = umma::ld_shared_s32(trow + 128u * i);
        for (int c0 = 0; c0 < a.ci_g; c0 += 64, ++it) {
          umma::mbar_wait(&empty_bar[st], ph ^ 1);
          const uint32_t sa = s0 + st * STAGE;
          if (tid == 0) {   // B tile (BN x 64 channels of this tap) by TMA, SWIZZLE_128B, OOB -> 0
            umma::mbar_arrive_expect_tx(&full_bar[st], B_BYTES);
            umma::tma_load_3d(sa + A_BYTES, &tmB, &full_bar[st], c0, tap, g * a.co_g + n0);
          }
          const bool cok = c0 + c * 8 < a.ci_g;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool ok = cok && pix[i] >= 0;
            umma::cp_async16(sa + off_r[i], ok ? xg + (int64_t)pix[i] * a.Ci + c0 : x, ok);
          }
          umma::cp_async_commit();
          if (it >= LAG) {
            umma::cp_async_wait<LAG>();
            umma::fence_proxy_async_smem();
            int sp = st - LAG;
            sp += sp < 0 ? S : 0;
            umma::mbar_arrive(&full_bar[sp]);
          }
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
    umma::cp_async_wait<0>();
    umma::fence_proxy_async_smem();
    for (int j = it - LAG < 0 ? 0 : it - LAG; j < it; ++j) umma::mbar_arrive(&full_bar[j % S]);
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = umma::idesc_bf16(128, BN);
      int it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
        const int acc = tcount & 1;
        umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) & 1) ^ 1);
        umma::tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int st = it % S;
          umma::mbar_wait(&full_bar[st], (it / S) & 1);
          umma::tc_fence_after();
          const uint32_t aa = s0 + st * STAGE, bb = aa + A_BYTES;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            umma::mma_bf16(d_tmem, umma::sdesc_sw128(aa + 32 * q), umma::sdesc_sw128(bb + 32 * q), IDESC,
                           (kb | q) != 0);
          umma::mma_commit(&empty_bar[st]);
        }
        umma::mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;               // TMEM lane quarter of this warp (warps 9..12 -> 1,2,3,0)
    const int r = q * 32 + lane;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < a.num_tiles; tile += gridDim.x, ++tcount) {
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
      const int tm = tile % a.tiles_m, rest = tile / a.tiles_m;
      const int tn = rest % a.tiles_n, g = rest / a.tiles_n;
      const int m = tm * 128 + r;
      const int obase = g * a.co_g + tn * BN;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + cc), v);
        if (m < M) {
          const int o = obase + cc;
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float v0 = v[2 * i], v1 = v[2 * i + 1];
            if (bias) { v0 += bias[o + 2 * i]; v1 += bias[o + 2 * i + 1]; }
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
            pk[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          uint4* dst = reinterpret_cast<uint4*>(y + (int64_t)m * a.Co + o);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      umma::tc_fence_before();
      umma::mbar_arrive(&tempty_bar[acc]);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) umma::tmem_dealloc(tmem, 2 * BN);
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
int launch_ws(const __nv_bfloat16* x, const __nv_bfloat16* w, const float* bias, __nv_bfloat16* y, TcConvArgs a,
              cudaStream_t stream) {
  const size_t smem = 1024 + (size_t)S * (128 * 128 + BN * 128) + (size_t)MAX_TAPS * 128 * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv_fwd_ws<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int grid = a.num_tiles < num_sms() ? a.num_tiles : num_sms();
  CUtensorMap tm;
  if (!make_weight_tmap(&tm, w, a.Co, a.k * a.k, a.ci_g, BN)) return (int)cudaErrorInvalidValue;
  conv_fwd_ws<BN, S><<<grid, NTHREADS, smem, stream>>>(x, w, bias, y, a, tm);
  return (int)cudaGetLastError();
}

}  // namespace

bool conv_fwd_tc_eligible(const LayerInfo& L) {
  return L.co % 64 == 0 && L.ci % 8 == 0 && L.ci_f % 8 == 0 && L.co_f % 8 == 0 && L.k * L.k <= MAX_TAPS;
}

int launch_conv_fwd_tc(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                       int H, int W, int Ho, int Wo, void* stream) {
  TcConvArgs a;
  a.N = N; a.H = H; a.W = W; a.Ci = L.ci_f; a.Co = L.co_f; a.ci_g = L.ci; a.co_g = L.co;
  a.k = L.k; a.s = L.s; a.d = L.d; a.pt = L.pt; a.pl = L.pl; a.Ho = Ho; a.Wo = Wo;
  a.circ = L.desc.padding_mode == ORTH_PAD_CIRCULAR;
  const int64_t M = (int64_t)N * Ho * Wo;
  a.tiles_m = (int)((M + 127) / 128);
  auto xs = (const __nv_bfloat16*)x;
  auto ws = (const __nv_bfloat16*)kernel;
  auto ys = (__nv_bfloat16*)y;
  cudaStream_t s = (cudaStream_t)stream;
  if (L.co % 256 == 0) {
    a.tiles_n = L.co / 256; a.num_tiles = a.tiles_m * a.tiles_n * L.g;
    return launch_ws<256, 4>(xs, ws, bias, ys, a, s);
  }
  if (L.co % 128 == 0) {
    a.tiles_n = L.co / 128; a.num_tiles = a.tiles_m * a.tiles_n * L.g;
    return launch_ws<128, 5>(xs, ws, bias, ys, a, s);
  }
  a.tiles_n = L.co / 64; a.num_tiles = a.tiles_m * a.tiles_n * L.g;
  return launch_ws<64, 7>(xs, ws, bias, ys, a, s);
}

}  // namespace orth
