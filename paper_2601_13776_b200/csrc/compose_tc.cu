// a4/a5 on the 5th-generation tensor cores (BF16 / BF16X3 construction modes):
// the BCOP projector chain and RKO (*) BCOP (P:321-326, P:351 footnote), each
// contraction through the 3-pass hi/lo split (hi*hi + hi*lo + lo*hi, FP32
// accumulation in TMEM), so the composed kernel stays FP32-accurate to ~1e-5
// and orthogonal far inside the 1e-3 bar (reading R16).
//
//   cvt    : ortho (FP32, user buffer) -> BF16 hi/lo copies of Q, U and the
//            RKO matrix split by spatial phase, R_ab[o, j] = R[o, j s^2 + a s + b]
//   proj   : P_j = U_j U_j^T, epilogue also writes I - P_j           (a4)
//   chain  : per substep and output tap  K'[t] = K[t] P + K[t-1] (I - P)
//            along the vertical, then the horizontal axis (block_orth, R5)
//   aoc    : K[p,q] = sum_{a,b} R_ab Kb[p-a, q-b]                     (a5, R7)
// Every GEMM reads BF16 K-major rows (16-byte cp.async, SWIZZLE_128B ring);
// epilogues write FP32 into the same composition workspace layout as the
// SIMT path (so the emit kernel is shared) plus the BF16 copies the next
// phase consumes (row-major, and transposed for the AOC's B operand).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "orth_internal.h"
#include "pdl.h"
#include "tma_host.h"
#include "umma.cuh"

namespace orth {

struct TcgSeg {
  const __nv_bfloat16 *ah, *al, *bh, *bl;
  int32_t lda, ldb;
};
struct TcgDesc {
  int32_t M, N, K, seg_begin, seg_count, tile_begin, tiles_n;
  float alpha, diag, alpha2, diag2;
  float* f;                      // fp32 output (nullable)
  int32_t ldf, ldo, ldt, pad_;
  __nv_bfloat16 *oh, *ol;        // row-major bf16 output (nullable)
  __nv_bfloat16 *o2h, *o2l;      // second row-major output alpha2*acc + diag2*I (nullable)
  __nv_bfloat16 *th, *tl;        // transposed bf16 output (nullable)
};
struct CvtItem {
  int64_t src_off;               // fp32 offset in ortho
  int32_t m, n, ld, mode;        // mode 0: row-major copy; 1: RKO phase split with s2 = phases
  int32_t s2, pad_;
  __nv_bfloat16 *dh, *dl;
};
struct TcgPhase {
  std::vector<TcgDesc> d;
  std::vector<TcgSeg> s;
  int tiles = 0;
  TcgDesc* dd = nullptr;
  TcgSeg* ds = nullptr;
  void* dmaps = nullptr;   // per segment 4 TMA maps {A hi, B hi, A lo, B lo}, then the tile -> desc table
  int* dtile = nullptr;
};
// dataflow composition: one (desc, tile) item of any phase, in claim order, with the per-unit counter it
// waits on (the unit's previous phase complete) and the one it bumps
struct TcgItem {
  int32_t desc, local;        // index into the combined descriptor array, tile inside the descriptor
  int32_t wait_ctr;           // -1: none
  uint32_t wait_target;
  int32_t done_ctr, pad_[3];
};

struct TcComposePlan {
  void* arena = nullptr;
  std::vector<CvtItem> cvt;
  CvtItem* dcvt = nullptr;
  TcgPhase proj, aoc;
  std::vector<TcgPhase> chain;
  std::vector<int> proj_unit, aoc_unit;       // unit index of every descriptor (dataflow dependencies)
  std::vector<std::vector<int>> chain_unit;
  // dataflow: every phase in ONE persistent launch (combined descriptors, segments' TMA maps, items)
  void* flow_mem = nullptr;
  TcgDesc* fdesc = nullptr;
  TcgItem* fitems = nullptr;
  CUtensorMap* fmaps = nullptr;
  unsigned* fctr = nullptr;                   // [0] claim counter, then per (unit, phase) completion counters
  int n_fitems = 0, n_fctr = 0;
};

namespace {

__device__ __forceinline__ void split(float x, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  l = __float2bfloat16_rn(x - __bfloat162float(h));
}

__device__ __forceinline__ int find_tcg(const TcgDesc* __restrict__ d, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int S = 3;

__global__ void __launch_bounds__(256, 1) tcg_kernel(const TcgDesc* __restrict__ descs, int ndesc,
                                                     const TcgSeg* __restrict__ segs) {
  constexpr int TILE = 128 * 128, STAGE = 4 * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t empty_bar[S];
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const TcgDesc d = descs[find_tcg(descs, ndesc, blockIdx.x)];
  const int local = blockIdx.x - d.tile_begin;
  const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;
  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, 128);
  if (tid == 32) {
    for (int i = 0; i < S; ++i) umma::mbar_init(&empty_bar[i], 1);
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);
  const int nkb = (d.K + 63) / 64;
  const int nk = nkb * d.seg_count;   // 0 for an empty product (rank-0 projector): acc = 0
  const int c = tid & 7;
  for (int kb = 0; kb < nk + S - 1; ++kb) {
    if (kb < nk) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const TcgSeg sg = segs[d.seg_begin + kb / nkb];
      const int kc = (kb % nkb) * 64 + c * 8;
      const bool kok = kc < d.K;
      const uint32_t sa = s0 + st * STAGE;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i;
        const uint32_t off = umma::sw128_off(r, c);
        const bool aok = kok && m0 + r < d.M, bok = kok && n0 + r < d.N;
        const int64_t ao = (int64_t)(m0 + r) * sg.lda + kc, bo = (int64_t)(n0 + r) * sg.ldb + kc;
        umma::cp_async16(sa + off, aok ? sg.ah + ao : sg.ah, aok);
        umma::cp_async16(sa + TILE + off, bok ? sg.bh + bo : sg.bh, bok);
        umma::cp_async16(sa + 2 * TILE + off, aok ? sg.al + ao : sg.al, aok);
        umma::cp_async16(sa + 3 * TILE + off, bok ? sg.bl + bo : sg.bl, bok);
      }
    }
    umma::cp_async_commit();
    const int j = kb - (S - 1);
    if (j >= 0) {
      umma::cp_async_wait<S - 1>();
      umma::fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        umma::tc_fence_after();
        const int st = j % S;
        const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, (j | q) != 0);
          umma::mma_bf16(tmem, umma::sdesc_sw128(ah + 32 * q), umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
          umma::mma_bf16(tmem, umma::sdesc_sw128(al + 32 * q), umma::sdesc_sw128(bh + 32 * q), IDESC, 1);
        }
        umma::mma_commit(&empty_bar[st]);
      }
    }
  }
  if (tid == 0) umma::mma_commit(&done_bar);
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();
  // epilogue through a smem tile (row stride 129 floats: conflict-free both ways)
  float* St = reinterpret_cast<float*>(smem);
  constexpr int LDS = 129;
  {
    const int q = warp & 3, half = warp >> 2, r = q * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < 64; cc += 32) {
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * 64 + cc), v);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) St[r * LDS + half * 64 + cc + jj] = nk > 0 ? v[jj] : 0.f;
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  for (int e = tid; e < 128 * 128; e += 256) {
    const int r = e >> 7, cl = e & 127, i = m0 + r, jn = n0 + cl;
    const float acc = St[r * LDS + cl];
    float o = 0.f, o2 = 0.f;
    if (i < d.M && jn < d.N) {
      o = d.alpha * acc + (i == jn ? d.diag : 0.f);
      o2 = d.alpha2 * acc + (i == jn ? d.diag2 : 0.f);
      if (d.f) d.f[(int64_t)i * d.ldf + jn] = o;
    }
    St[r * LDS + cl] = o;
    if (i < d.M && jn < d.ldo) {
      __nv_bfloat16 h, l;
      if (d.oh) {
        split(o, h, l);
        d.oh[(int64_t)i * d.ldo + jn] = h;
        d.ol[(int64_t)i * d.ldo + jn] = l;
      }
      if (d.o2h) {
        split(o2, h, l);
        d.o2h[(int64_t)i * d.ldo + jn] = h;
        d.o2l[(int64_t)i * d.ldo + jn] = l;
      }
    }
  }
  if (d.th) {
    __syncthreads();
    for (int e = tid; e < 128 * 128; e += 256) {
      const int cl = e >> 7, r = e & 127, i = m0 + r, jn = n0 + cl;
      if (jn < d.N && i < d.ldt) {
        __nv_bfloat16 h, l;
        split(St[r * LDS + cl], h, l);
        d.th[(int64_t)jn * d.ldt + i] = h;
        d.tl[(int64_t)jn * d.ldt + i] = l;
      }
    }
  }
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 128);
}

// TMA version of the composition GEMM (one 128x128 output tile per CTA):
// tid 0 streams {A hi, B hi, A lo, B lo} 128x64 boxes of each segment by TMA
// into a 3-stage SWIZZLE_128B ring, tid 32 issues the 3-pass tcgen05.mma, all
// 256 threads run a vectorised epilogue (two 64-column halves through a
// padded smem tile; row outputs as float4 / packed BF16x4, the transposed
// output by a column pass).
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void split4(float a, float b, float c, float d, uint2& hi, uint2& lo) {
  hi.x = pack2(a, b);
  hi.y = pack2(c, d);
  lo.x = pack2(a - __uint_as_float(hi.x << 16), b - __uint_as_float(hi.x & 0xFFFF0000u));
  lo.y = pack2(c - __uint_as_float(hi.y << 16), d - __uint_as_float(hi.y & 0xFFFF0000u));
}

__global__ void __launch_bounds__(256, 1) tcg_tma_kernel(const TcgDesc* __restrict__ descs,
                                                         const int* __restrict__ tile_desc,
                                                         const CUtensorMap* __restrict__ maps) {
  constexpr int TILE = 128 * 128, STAGE = 4 * TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  __shared__ uint64_t full_bar[S], empty_bar[S], done_bar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  umma::griddep_launch_dependents();
  const TcgDesc d = descs[tile_desc[blockIdx.x]];   // plan constants: readable before the PDL wait
  const int local = blockIdx.x - d.tile_begin;
  const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;
  if (warp == 0) umma::tmem_alloc(&tmem_base_sh, 128);
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
    }
    umma::mbar_init(&done_bar, 1);
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  umma::griddep_wait();   // PDL: the previous phase's outputs are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  const int nkb = (d.K + 63) / 64;
  const int nk = nkb * d.seg_count;   // 0 for an empty product (rank-0 projector): acc = 0
  if (tid == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      if (kb >= S) umma::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
      const CUtensorMap* mp = maps + 4 * (d.seg_begin + kb / nkb);
      const int k0 = (kb % nkb) * 64;
      const uint32_t sa = s0 + st * STAGE;
      umma::mbar_arrive_expect_tx(&full_bar[st], STAGE);
      umma::tma_load_2d(sa, mp + 0, &full_bar[st], k0, m0);
      umma::tma_load_2d(sa + TILE, mp + 1, &full_bar[st], k0, n0);
      umma::tma_load_2d(sa + 2 * TILE, mp + 2, &full_bar[st], k0, m0);
      umma::tma_load_2d(sa + 3 * TILE, mp + 3, &full_bar[st], k0, n0);
    }
  } else if (tid == 32) {
    constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % S;
      umma::mbar_wait(&full_bar[st], (kb / S) & 1);
      umma::tc_fence_after();
      const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t dah = umma::sdesc_sw128(ah + 32 * q), dbh = umma::sdesc_sw128(bh + 32 * q);
        umma::mma_bf16(tmem, dah, dbh, IDESC, (kb | q) != 0);
        umma::mma_bf16(tmem, dah, umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
        umma::mma_bf16(tmem, umma::sdesc_sw128(al + 32 * q), dbh, IDESC, 1);
      }
      umma::mma_commit(&empty_bar[st]);
    }
    umma::mma_commit(&done_bar);
  }
  umma::mbar_wait(&done_bar, 0);
  umma::tc_fence_after();
  // ---- epilogue: two 64-column halves
  constexpr int LDF = 68;
  float* Sf = reinterpret_cast<float*>(smem);   // [128][68]
  const bool fvec = d.f && (d.ldf & 3) == 0;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    {
      const int q = warp & 3, sub = warp >> 2, r = q * 32 + lane;
      float v[32];
      umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 64 + sub * 32), v);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        *reinterpret_cast<float4*>(Sf + r * LDF + sub * 32 + 4 * t) =
            nk > 0 ? make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    umma::tc_fence_before();
    __syncthreads();
#pragma unroll 2
    for (int u = 0; u < 8; ++u) {
      const int e = tid + 256 * u, r = e >> 4, c4 = (e & 15) * 4;
      const int i = m0 + r, j0 = n0 + h * 64 + c4;
      const float4 a = *reinterpret_cast<const float4*>(Sf + r * LDF + c4);
      const float acc[4] = {a.x, a.y, a.z, a.w};
      float o[4], o2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = i < d.M && j0 + k < d.N;
        const float dg = (i == j0 + k) ? 1.f : 0.f;
        o[k] = ok ? fmaf(d.alpha, acc[k], d.diag * dg) : 0.f;
        o2[k] = ok ? fmaf(d.alpha2, acc[k], d.diag2 * dg) : 0.f;
      }
      if (d.f && i < d.M && j0 < d.N) {
        float* dst = d.f + (int64_t)i * d.ldf + j0;
        if (fvec && j0 + 3 < d.N) {
          *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (j0 + k < d.N) dst[k] = o[k];
        }
      }
      if (i < d.M && j0 < d.ldo) {   // ldo % 8 == 0: the 4-group lies inside the padded row
        const int64_t bo = (int64_t)i * d.ldo + j0;
        uint2 hv, lv;
        if (d.oh) {
          split4(o[0], o[1], o[2], o[3], hv, lv);
          *reinterpret_cast<uint2*>(d.oh + bo) = hv;
          *reinterpret_cast<uint2*>(d.ol + bo) = lv;
        }
        if (d.o2h) {
          split4(o2[0], o2[1], o2[2], o2[3], hv, lv);
          *reinterpret_cast<uint2*>(d.o2h + bo) = hv;
          *reinterpret_cast<uint2*>(d.o2l + bo) = lv;
        }
      }
      if (d.th) *reinterpret_cast<float4*>(Sf + r * LDF + c4) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();
    if (d.th) {   // transposed rows: lane -> column (conflict-free Sf column reads), 8 rows -> one 16-byte store
#pragma unroll 1
      for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u, cl = e & 63, i8 = (e >> 6) * 8;
        const int jn = n0 + h * 64 + cl, i0 = m0 + i8;
        float x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) x[t] = Sf[(i8 + t) * LDF + cl];
        if (jn < d.N && i0 < d.ldt) {
          uint2 h0, l0, h1, l1;
          split4(x[0], x[1], x[2], x[3], h0, l0);
          split4(x[4], x[5], x[6], x[7], h1, l1);
          const int64_t o = (int64_t)jn * d.ldt + i0;
          *reinterpret_cast<uint4*>(d.th + o) = make_uint4(h0.x, h0.y, h1.x, h1.y);
          *reinterpret_cast<uint4*>(d.tl + o) = make_uint4(l0.x, l0.y, l1.x, l1.y);
        }
      }
      __syncthreads();
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tmem, 128);
}

// Persistent, pipelined version of tcg_tma_kernel (default): grid <= #SMs, each
// CTA walks tiles tile = blockIdx.x + i * gridDim.x.  Warp 0 = TMA producer
// (3-stage ring of {A, B} x {hi, lo} 64-deep K blocks), warp 1 = TMEM owner +
// single-thread MMA issuer into one of two 128-column accumulators, warps 2-9 =
// epilogue (the same FP32 / hi-lo / second / transposed outputs as above, in
// four 32-column passes through an 18 KB staging tile).  The epilogue of tile i
// overlaps the loads and MMAs of tile i+1 (the 1-tile-per-CTA kernel paid the
// CTA launch, prologue and a serial epilogue per tile).
constexpr int kTcpThreads = 320;
constexpr int kTcpSf = 128 * 36;   // floats of the staging tile [128][32 + 4]

__global__ void __launch_bounds__(kTcpThreads, 1) tcg_tma_persist(const TcgDesc* __restrict__ descs,
                                                                  const int* __restrict__ tile_desc, int ntiles,
                                                                  const CUtensorMap* __restrict__ maps) {
  constexpr int TILE = 128 * 128, STAGE = 4 * TILE;
  extern __shared__ uint8_t smem_raw[];
  umma::griddep_launch_dependents();
  uint8_t* smem = umma::align1024_smem(smem_raw);
  float* Sf = reinterpret_cast<float*>(smem + S * STAGE);
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 1) umma::tmem_alloc(&tmem_base_sh, 256);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], 8);   // one arrival per epilogue warp
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  umma::griddep_wait();   // PDL: the previous phase's outputs are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  if (warp == 0) {
    // ---------------------------------------------------------------- producer (lanes 0-3)
    // the four boxes of a K block are issued by four lanes: one thread issuing TMA loads back to back
    // pays ~150 ns per load (measured on the conv window loads)
    if (lane < 4) {
      int kb_all = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TcgDesc& d = descs[tile_desc[tile]];
        const int local = tile - d.tile_begin;
        const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;
        const int nkb = (d.K + 63) / 64, nk = nkb * d.seg_count;
        for (int kb = 0; kb < nk; ++kb, ++kb_all) {
          const int st = kb_all % S;
          if (kb_all >= S) umma::mbar_wait(&empty_bar[st], ((kb_all / S) - 1) & 1);
          const CUtensorMap* mp = maps + 4 * (d.seg_begin + kb / nkb);
          const int k0 = (kb % nkb) * 64;
          const uint32_t sa = s0 + st * STAGE;
          if (lane == 0) umma::mbar_arrive_expect_tx(&full_bar[st], STAGE);
          __syncwarp(0xFu);
          umma::tma_load_2d(sa + lane * TILE, mp + lane, &full_bar[st], k0, (lane & 1) ? n0 : m0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);
      int kb_all = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
        const TcgDesc& d = descs[tile_desc[tile]];
        const int nk = ((d.K + 63) / 64) * d.seg_count;   // 0: empty product (rank-0 projector), acc = 0
        const int acc = tcount & 1;
        if (tcount >= 2) umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) - 1) & 1);
        umma::tc_fence_after();
        const uint32_t dt = tmem + acc * 128;
        for (int kb = 0; kb < nk; ++kb, ++kb_all) {
          const int st = kb_all % S;
          umma::mbar_wait(&full_bar[st], (kb_all / S) & 1);
          umma::tc_fence_after();
          const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t dah = umma::sdesc_sw128(ah + 32 * q), dbh = umma::sdesc_sw128(bh + 32 * q);
            umma::mma_bf16(dt, dah, dbh, IDESC, (kb | q) != 0);
            umma::mma_bf16(dt, dah, umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
            umma::mma_bf16(dt, umma::sdesc_sw128(al + 32 * q), dbh, IDESC, 1);
          }
          umma::mma_commit(&empty_bar[st]);
        }
        umma::mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-9)
    const int ew = warp - 2, etid = tid - 64;
    const int q = warp & 3, sub = ew >> 2, r_own = q * 32 + lane;   // TMEM lane quarter = warp % 4
    constexpr int LDF = 36;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
      const TcgDesc d = descs[tile_desc[tile]];
      const int local = tile - d.tile_begin;
      const int m0 = (local / d.tiles_n) * 128, n0 = (local % d.tiles_n) * 128;
      const int nk = ((d.K + 63) / 64) * d.seg_count;
      const bool fvec = d.f && (d.ldf & 3) == 0;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {   // 32-column passes
        {
          float v[16];
          umma::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 128 + h * 32 + sub * 16), v);
#pragma unroll
          for (int t = 0; t < 4; ++t)
            *reinterpret_cast<float4*>(Sf + r_own * LDF + sub * 16 + 4 * t) =
                nk > 0 ? make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (h == 3) {   // accumulator drained: release it to the MMA warp
          umma::tc_fence_before();
          __syncwarp();
          if (lane == 0) umma::mbar_arrive(&tempty_bar[acc]);
        }
        umma::named_bar_sync(1, 256);
#pragma unroll 2
        for (int u = 0; u < 4; ++u) {
          const int e = etid + 256 * u, r = e >> 3, c4 = (e & 7) * 4;
          const int i = m0 + r, j0 = n0 + h * 32 + c4;
          const float4 a = *reinterpret_cast<const float4*>(Sf + r * LDF + c4);
          const float accv[4] = {a.x, a.y, a.z, a.w};
          float o[4], o2[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool ok = i < d.M && j0 + k < d.N;
            const float dg = (i == j0 + k) ? 1.f : 0.f;
            o[k] = ok ? fmaf(d.alpha, accv[k], d.diag * dg) : 0.f;
            o2[k] = ok ? fmaf(d.alpha2, accv[k], d.diag2 * dg) : 0.f;
          }
          if (d.f && i < d.M && j0 < d.N) {
            float* dst = d.f + (int64_t)i * d.ldf + j0;
            if (fvec && j0 + 3 < d.N) {
              *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (j0 + k < d.N) dst[k] = o[k];
            }
          }
          if (i < d.M && j0 < d.ldo) {   // ldo % 8 == 0: the 4-group lies inside the padded row
            const int64_t bo = (int64_t)i * d.ldo + j0;
            uint2 hv, lv;
            if (d.oh) {
              split4(o[0], o[1], o[2], o[3], hv, lv);
              *reinterpret_cast<uint2*>(d.oh + bo) = hv;
              *reinterpret_cast<uint2*>(d.ol + bo) = lv;
            }
            if (d.o2h) {
              split4(o2[0], o2[1], o2[2], o2[3], hv, lv);
              *reinterpret_cast<uint2*>(d.o2h + bo) = hv;
              *reinterpret_cast<uint2*>(d.o2l + bo) = lv;
            }
          }
          if (d.th) *reinterpret_cast<float4*>(Sf + r * LDF + c4) = make_float4(o[0], o[1], o[2], o[3]);
        }
        umma::named_bar_sync(1, 256);
        if (d.th) {   // transposed rows: lane -> column, 8 rows -> one 16-byte store
#pragma unroll 1
          for (int u = 0; u < 2; ++u) {
            const int e = etid + 256 * u, cl = e & 31, i8 = (e >> 5) * 8;
            const int jn = n0 + h * 32 + cl, i0 = m0 + i8;
            float x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = Sf[(i8 + t) * LDF + cl];
            if (jn < d.N && i0 < d.ldt) {
              uint2 h0, l0, h1, l1;
              split4(x[0], x[1], x[2], x[3], h0, l0);
              split4(x[4], x[5], x[6], x[7], h1, l1);
              const int64_t o = (int64_t)jn * d.ldt + i0;
              *reinterpret_cast<uint4*>(d.th + o) = make_uint4(h0.x, h0.y, h1.x, h1.y);
              *reinterpret_cast<uint4*>(d.tl + o) = make_uint4(l0.x, l0.y, l1.x, l1.y);
            }
          }
          umma::named_bar_sync(1, 256);
        }
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tmem, 256);
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All composition phases (projectors, every chain substep, RKO (*) BCOP) in ONE persistent launch:
// (desc, tile) items in phase-major claim order; a tile's producer waits until its unit's previous
// phase is complete (per-unit monotonic counters, relaxed polls + one acquire fence), the epilogue
// publishes with a release reduction after the proxy fence.  Units therefore advance independently --
// the per-phase launches made every phase wait for the slowest unit of the previous one.  The tile
// pipeline (TMA boxes, 3-pass MMA, 8 epilogue warps) is tcg_tma_persist's.
__global__ void __launch_bounds__(kTcpThreads, 1) tcg_flow(const TcgDesc* __restrict__ descs,
                                                           const TcgItem* __restrict__ items, int n_items,
                                                           const CUtensorMap* __restrict__ maps,
                                                           unsigned* __restrict__ ctr) {
  constexpr int TILE = 128 * 128, STAGE = 4 * TILE;
  extern __shared__ uint8_t smem_raw[];
  umma::griddep_launch_dependents();
  uint8_t* smem = umma::align1024_smem(smem_raw);
  float* Sf = reinterpret_cast<float*>(smem + S * STAGE);
  __shared__ uint64_t full_bar[S], empty_bar[S], tfull_bar[2], tempty_bar[2], qfull[8], qempty[8];
  __shared__ int qslot[8];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 1) umma::tmem_alloc(&tmem_base_sh, 256);
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], 8);
    }
    for (int i = 0; i < 8; ++i) {
      umma::mbar_init(&qfull[i], 1);
      umma::mbar_init(&qempty[i], 8);   // the 8 epilogue warps are the last readers of a queue slot
    }
    umma::fence_mbar_init();
  }
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  umma::griddep_wait();   // PDL: the cvt kernel's copies and counter reset are complete
  const uint32_t tmem = tmem_base_sh;
  const uint32_t s0 = umma::smem_u32(smem);
  if (warp == 0) {
    // ---------------------------------------------------------------- claim + producer (lanes 0-3)
    if (lane < 4) {
      int kb_all = 0;
      for (int kq = 0;; ++kq) {
        const int slot = kq & 7;
        int idx = 0;
        if (lane == 0) {
          if (kq >= 8) umma::mbar_wait(&qempty[slot], ((kq >> 3) - 1) & 1);
          idx = (int)atomicAdd(ctr, 1u);
          if (idx < n_items) {
            const TcgItem it = items[idx];
            if (it.wait_ctr >= 0) {   // the unit's previous phase is complete
              while (ld_relaxed_u32(ctr + it.wait_ctr) < it.wait_target) __nanosleep(32);
              asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
          }
          qslot[slot] = idx < n_items ? idx : -1;
          umma::mbar_arrive(&qfull[slot]);
        }
        idx = __shfl_sync(0xFu, idx, 0);
        if (idx >= n_items) break;
        asm volatile("fence.proxy.async.global;" ::: "memory");   // other CTAs' generic writes -> TMA reads
        const TcgItem it = items[idx];
        const TcgDesc& d = descs[it.desc];
        const int m0 = (it.local / d.tiles_n) * 128, n0 = (it.local % d.tiles_n) * 128;
        const int nkb = (d.K + 63) / 64, nk = nkb * d.seg_count;
        for (int kb = 0; kb < nk; ++kb, ++kb_all) {
          const int st = kb_all % S;
          if (kb_all >= S) umma::mbar_wait(&empty_bar[st], ((kb_all / S) - 1) & 1);
          const CUtensorMap* mp = maps + 4 * (d.seg_begin + kb / nkb);
          const int k0 = (kb % nkb) * 64;
          const uint32_t sa = s0 + st * STAGE;
          if (lane == 0) umma::mbar_arrive_expect_tx(&full_bar[st], STAGE);
          __syncwarp(0xFu);
          umma::tma_load_2d(sa + lane * TILE, mp + lane, &full_bar[st], k0, (lane & 1) ? n0 : m0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = umma::idesc_bf16(128, 128);
      int kb_all = 0, tcount = 0;
      for (int kq = 0;; ++kq, ++tcount) {
        const int slot = kq & 7;
        umma::mbar_wait(&qfull[slot], (kq >> 3) & 1);
        const int idx = qslot[slot];
        if (idx < 0) break;
        const TcgDesc& d = descs[items[idx].desc];
        const int nk = ((d.K + 63) / 64) * d.seg_count;
        const int acc = tcount & 1;
        if (tcount >= 2) umma::mbar_wait(&tempty_bar[acc], ((tcount >> 1) - 1) & 1);
        umma::tc_fence_after();
        const uint32_t dt = tmem + acc * 128;
        for (int kb = 0; kb < nk; ++kb, ++kb_all) {
          const int st = kb_all % S;
          umma::mbar_wait(&full_bar[st], (kb_all / S) & 1);
          umma::tc_fence_after();
          const uint32_t ah = s0 + st * STAGE, bh = ah + TILE, al = ah + 2 * TILE, bl = ah + 3 * TILE;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t dah = umma::sdesc_sw128(ah + 32 * q), dbh = umma::sdesc_sw128(bh + 32 * q);
            umma::mma_bf16(dt, dah, dbh, IDESC, (kb | q) != 0);
            umma::mma_bf16(dt, dah, umma::sdesc_sw128(bl + 32 * q), IDESC, 1);
            umma::mma_bf16(dt, umma::sdesc_sw128(al + 32 * q), dbh, IDESC, 1);
          }
          umma::mma_commit(&empty_bar[st]);
        }
        umma::mma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-9)
    const int ew = warp - 2, etid = tid - 64;
    const int q = warp & 3, sub = ew >> 2, r_own = q * 32 + lane;
    constexpr int LDF = 36;
    for (int kq = 0, tcount = 0;; ++kq, ++tcount) {
      const int slot = kq & 7;
      umma::mbar_wait(&qfull[slot], (kq >> 3) & 1);
      const int idx = qslot[slot];
      if (idx < 0) break;
      const TcgItem it = items[idx];
      const TcgDesc d = descs[it.desc];
      const int m0 = (it.local / d.tiles_n) * 128, n0 = (it.local % d.tiles_n) * 128;
      const int nk = ((d.K + 63) / 64) * d.seg_count;
      const bool fvec = d.f && (d.ldf & 3) == 0;
      const int acc = tcount & 1;
      umma::mbar_wait(&tfull_bar[acc], (tcount >> 1) & 1);
      umma::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        {
          float v[16];
          umma::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 128 + h * 32 + sub * 16), v);
#pragma unroll
          for (int t = 0; t < 4; ++t)
            *reinterpret_cast<float4*>(Sf + r_own * LDF + sub * 16 + 4 * t) =
                nk > 0 ? make_float4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (h == 3) {
          umma::tc_fence_before();
          __syncwarp();
          if (lane == 0) umma::mbar_arrive(&tempty_bar[acc]);
        }
        umma::named_bar_sync(1, 256);
#pragma unroll 2
        for (int u = 0; u < 4; ++u) {
          const int e = etid + 256 * u, r = e >> 3, c4 = (e & 7) * 4;
          const int i = m0 + r, j0 = n0 + h * 32 + c4;
          const float4 a = *reinterpret_cast<const float4*>(Sf + r * LDF + c4);
          const float accv[4] = {a.x, a.y, a.z, a.w};
          float o[4], o2[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool ok = i < d.M && j0 + k < d.N;
            const float dg = (i == j0 + k) ? 1.f : 0.f;
            o[k] = ok ? fmaf(d.alpha, accv[k], d.diag * dg) : 0.f;
            o2[k] = ok ? fmaf(d.alpha2, accv[k], d.diag2 * dg) : 0.f;
          }
          if (d.f && i < d.M && j0 < d.N) {
            float* dst = d.f + (int64_t)i * d.ldf + j0;
            if (fvec && j0 + 3 < d.N) {
              *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (j0 + k < d.N) dst[k] = o[k];
            }
          }
          if (i < d.M && j0 < d.ldo) {
            const int64_t bo = (int64_t)i * d.ldo + j0;
            uint2 hv, lv;
            if (d.oh) {
              split4(o[0], o[1], o[2], o[3], hv, lv);
              *reinterpret_cast<uint2*>(d.oh + bo) = hv;
              *reinterpret_cast<uint2*>(d.ol + bo) = lv;
            }
            if (d.o2h) {
              split4(o2[0], o2[1], o2[2], o2[3], hv, lv);
              *reinterpret_cast<uint2*>(d.o2h + bo) = hv;
              *reinterpret_cast<uint2*>(d.o2l + bo) = lv;
            }
          }
          if (d.th) *reinterpret_cast<float4*>(Sf + r * LDF + c4) = make_float4(o[0], o[1], o[2], o[3]);
        }
        umma::named_bar_sync(1, 256);
        if (d.th) {
#pragma unroll 1
          for (int u = 0; u < 2; ++u) {
            const int e = etid + 256 * u, cl = e & 31, i8 = (e >> 5) * 8;
            const int jn = n0 + h * 32 + cl, i0 = m0 + i8;
            float x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = Sf[(i8 + t) * LDF + cl];
            if (jn < d.N && i0 < d.ldt) {
              uint2 h0, l0, h1, l1;
              split4(x[0], x[1], x[2], x[3], h0, l0);
              split4(x[4], x[5], x[6], x[7], h1, l1);
              const int64_t o = (int64_t)jn * d.ldt + i0;
              *reinterpret_cast<uint4*>(d.th + o) = make_uint4(h0.x, h0.y, h1.x, h1.y);
              *reinterpret_cast<uint4*>(d.tl + o) = make_uint4(l0.x, l0.y, l1.x, l1.y);
            }
          }
          umma::named_bar_sync(1, 256);
        }
      }
      // ---- item done: publish this tile's writes, bump the unit's counter, free the queue slot
      asm volatile("fence.proxy.async.global;" ::: "memory");
      umma::named_bar_sync(1, 256);
      if (ew == 0 && lane == 0)   // release (cumulative over the barrier) orders every epilogue warp's writes
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + it.done_ctr) : "memory");
      if (lane == 0) umma::mbar_arrive(&qempty[slot]);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tmem, 256);
}

// FP32 ortho -> BF16 hi/lo copies (row-major padded, or the RKO phase split).
// CTA = rows r = blockIdx.x + k gridDim.x of item blockIdx.y; 32-bit index math.
__global__ void __launch_bounds__(256) cvt_kernel(const CvtItem* __restrict__ items, const float* __restrict__ ortho,
                                                  unsigned* __restrict__ zero, int nzero) {
  if (zero && blockIdx.x == 0 && blockIdx.y == 0)   // re-arm the dataflow counters of the launch that follows
    for (int i = threadIdx.x; i < nzero; i += blockDim.x) zero[i] = 0u;
  umma::griddep_launch_dependents();
  umma::griddep_wait();
  const CvtItem it = items[blockIdx.y];
  for (int r = blockIdx.x; r < it.m; r += gridDim.x) {
    const float* src = ortho + it.src_off + (int64_t)r * it.n;
    if (it.mode == 0) {
      __nv_bfloat16* dh = it.dh + (int64_t)r * it.ld;
      __nv_bfloat16* dl = it.dl + (int64_t)r * it.ld;
      if (it.n <= 128) {   // short rows: one warp per row, 8 rows per CTA pass (the block loop below
        continue;          // would leave most of the 256 threads idle); handled after this loop
      }
      for (int c = threadIdx.x; c < it.n; c += 256) {
        __nv_bfloat16 h, l;
        split(__ldg(src + c), h, l);
        dh[c] = h;
        dl[c] = l;
      }
    } else {   // R[o, j s^2 + ph] -> block ph, row o, column j
      const int nj = it.n / it.s2;
      if (it.s2 == 4 && ((it.src_off + (int64_t)r * it.n) & 3) == 0) {   // the 4 phases of j: one float4
        for (int j = threadIdx.x; j < nj; j += 256) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src) + j);
          const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int ph = 0; ph < 4; ++ph) {
            __nv_bfloat16 h, l;
            split(x[ph], h, l);
            const int64_t o = ((int64_t)ph * it.m + r) * it.ld + j;
            it.dh[o] = h;
            it.dl[o] = l;
          }
        }
      } else {
        for (int j = threadIdx.x; j < nj; j += 256)
          for (int ph = 0; ph < it.s2; ++ph) {
            __nv_bfloat16 h, l;
            split(__ldg(src + j * it.s2 + ph), h, l);
            const int64_t o = ((int64_t)ph * it.m + r) * it.ld + j;
            it.dh[o] = h;
            it.dl[o] = l;
          }
      }
    }
  }
  if (it.mode == 0 && it.n <= 128) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = blockIdx.x * 8 + warp; r < it.m; r += gridDim.x * 8) {
      const float* src = ortho + it.src_off + (int64_t)r * it.n;
      __nv_bfloat16* dh = it.dh + (int64_t)r * it.ld;
      __nv_bfloat16* dl = it.dl + (int64_t)r * it.ld;
      for (int c = lane; c < it.n; c += 32) {
        __nv_bfloat16 h, l;
        split(__ldg(src + c), h, l);
        dh[c] = h;
        dl[c] = l;
      }
    }
  }
}

int launch_phase(const TcgPhase& ph, cudaStream_t s) {
  if (!ph.tiles) return 0;
  const size_t smem = 1024 + (size_t)S * 4 * 128 * 128;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tcg_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  static const bool one_tile = std::getenv("ORTH_COMPOSE_ONE_TILE") != nullptr;   // A/B: 1 tile per CTA
  if (ph.dmaps && !one_tile) {
    const size_t smem_p = 1024 + (size_t)S * 4 * 128 * 128 + (size_t)kTcpSf * 4;
    static bool attr_p = false;
    if (!attr_p) {
      cudaFuncSetAttribute(tcg_tma_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
      attr_p = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(ph.tiles, sms);
    launch_pdl(tcg_tma_persist, dim3(grid), dim3(kTcpThreads), smem_p, s, (const TcgDesc*)ph.dd,
               (const int*)ph.dtile, ph.tiles, reinterpret_cast<const CUtensorMap*>(ph.dmaps));
  } else if (ph.dmaps)
    launch_pdl(tcg_tma_kernel, dim3(ph.tiles), dim3(256), smem, s, ph.dd, ph.dtile,
               reinterpret_cast<const CUtensorMap*>(ph.dmaps));
  else
    tcg_kernel<<<ph.tiles, 256, smem, s>>>(ph.dd, (int)ph.d.size(), ph.ds);
  return (int)cudaGetLastError();
}

// TMA maps of every segment operand (K extent x rows, row stride ld) plus the
// tile -> descriptor table; phases whose operands cannot be described by TMA
// (misaligned pointer or stride) keep the cp.async kernel.
bool host_phase_maps(const TcgPhase& ph, std::vector<CUtensorMap>& maps) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  maps.assign(4 * ph.s.size(), CUtensorMap{});
  std::vector<int> seg_desc(ph.s.size(), -1);
  for (size_t di = 0; di < ph.d.size(); ++di)
    for (int k = 0; k < ph.d[di].seg_count; ++k) seg_desc[ph.d[di].seg_begin + k] = (int)di;
  for (size_t si = 0; si < ph.s.size(); ++si) {
    const TcgSeg& g = ph.s[si];
    const int di = seg_desc[si];
    const TcgDesc& d = ph.d[di < 0 ? 0 : di];
    const __nv_bfloat16* ptr[4] = {g.ah, g.bh, g.al, g.bl};
    const int rows[4] = {d.M, d.N, d.M, d.N}, ld[4] = {g.lda, g.ldb, g.lda, g.ldb};
    for (int q = 0; q < 4; ++q) {
      if (((uintptr_t)ptr[q] & 15) || (ld[q] % 8) || d.K < 1) return false;
      const cuuint64_t dims[2] = {(cuuint64_t)d.K, (cuuint64_t)std::max(rows[q], 1)};
      const cuuint64_t strides[1] = {(cuuint64_t)ld[q] * 2};
      const cuuint32_t box[2] = {64, 128};
      const cuuint32_t es[2] = {1, 1};
      std::memset(&maps[4 * si + q], 0, sizeof(CUtensorMap));
      if (enc(&maps[4 * si + q], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(ptr[q]), dims, strides,
              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
  }
  return true;
}

bool build_phase_maps(TcgPhase& ph) {
  if (!ph.tiles) return true;
  std::vector<CUtensorMap> maps;
  if (!host_phase_maps(ph, maps)) return false;
  std::vector<int> tile;
  for (size_t di = 0; di < ph.d.size(); ++di) {
    const TcgDesc& d = ph.d[di];
    for (int t = 0; t < ((d.M + 127) / 128) * d.tiles_n; ++t) tile.push_back((int)di);
  }
  const size_t mb = maps.size() * sizeof(CUtensorMap);
  if (cudaMalloc(&ph.dmaps, mb + tile.size() * sizeof(int) + 64) != cudaSuccess) {
    ph.dmaps = nullptr;
    return false;
  }
  ph.dtile = reinterpret_cast<int*>(static_cast<char*>(ph.dmaps) + mb);
  if (!maps.empty()) cudaMemcpy(ph.dmaps, maps.data(), mb, cudaMemcpyHostToDevice);
  cudaMemcpy(ph.dtile, tile.data(), tile.size() * sizeof(int), cudaMemcpyHostToDevice);
  return true;
}

void finish(TcgPhase& ph) {
  int t = 0;
  for (auto& d : ph.d) {
    d.tile_begin = t;
    d.tiles_n = (d.N + 127) / 128;
    t += ((d.M + 127) / 128) * d.tiles_n;
  }
  ph.tiles = t;
}

TcgDesc mkdesc(int M, int N, int K) {
  TcgDesc d{};
  d.M = M; d.N = N; d.K = K;
  d.alpha = 1.0f;
  return d;
}

}  // namespace

// The dataflow composition (tcg_flow): every phase's descriptors, segments' TMA maps and tiles combined,
// items in phase-major order (inside a phase the units with the most K work first), one completion
// counter per (unit, phase).  Phase order: projectors, chain substeps, RKO (*) BCOP.  A chain substep of
// a unit waits for all of the unit's tiles of the previous stage (its projectors for substep 0), the AOC
// tiles for the unit's last substep.  Leaves T.flow_mem null (per-phase launches) if a map cannot be built.
static void build_compose_flow(Plan& P, TcComposePlan& T) {
  std::vector<const TcgPhase*> phs;
  std::vector<const std::vector<int>*> units;
  phs.push_back(&T.proj); units.push_back(&T.proj_unit);
  for (size_t t = 0; t < T.chain.size(); ++t) { phs.push_back(&T.chain[t]); units.push_back(&T.chain_unit[t]); }
  phs.push_back(&T.aoc); units.push_back(&T.aoc_unit);
  const int nph = (int)phs.size(), nu = (int)P.comp_units.size();
  std::vector<TcgDesc> desc;
  std::vector<CUtensorMap> maps;
  std::vector<int> desc0(nph, 0);
  int seg0 = 0;
  for (int p = 0; p < nph; ++p) {
    desc0[p] = (int)desc.size();
    std::vector<CUtensorMap> m;
    if (phs[p]->tiles && !host_phase_maps(*phs[p], m)) return;
    for (TcgDesc d : phs[p]->d) { d.seg_begin += seg0; desc.push_back(d); }
    maps.insert(maps.end(), m.begin(), m.end());
    seg0 += (int)phs[p]->s.size();
    if (phs[p]->tiles && (int)m.size() != 4 * (int)phs[p]->s.size()) return;
  }
  if (desc.empty()) return;
  // tiles per (unit, phase), the last phase index with tiles per unit (chain depth differs across units)
  std::vector<int> cnt((size_t)nu * nph, 0);
  for (int p = 0; p < nph; ++p)
    for (size_t di = 0; di < phs[p]->d.size(); ++di) {
      const TcgDesc& d = phs[p]->d[di];
      cnt[(size_t)(*units[p])[di] * nph + p] += ((d.M + 127) / 128) * ((d.N + 127) / 128);
    }
  auto ctr_of = [&](int u, int p) { return 1 + u * nph + p; };
  std::vector<TcgItem> items;
  for (int p = 0; p < nph; ++p) {
    std::vector<int> order(phs[p]->d.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (int64_t)phs[p]->d[a].K * phs[p]->d[a].seg_count > (int64_t)phs[p]->d[b].K * phs[p]->d[b].seg_count;
    });
    for (int di : order) {
      const TcgDesc& d = phs[p]->d[di];
      const int u = (*units[p])[di];
      int wp = -1;   // the unit's previous phase with tiles
      for (int q = p - 1; q >= 0; --q)
        if (cnt[(size_t)u * nph + q] > 0) { wp = q; break; }
      const int nt = ((d.M + 127) / 128) * ((d.N + 127) / 128);
      for (int t = 0; t < nt; ++t) {
        TcgItem it{};
        it.desc = desc0[p] + di;
        it.local = t;
        it.wait_ctr = wp >= 0 ? ctr_of(u, wp) : -1;
        it.wait_target = wp >= 0 ? (uint32_t)cnt[(size_t)u * nph + wp] : 0u;
        it.done_ctr = ctr_of(u, p);
        items.push_back(it);
      }
    }
  }
  for (auto& d : desc) d.tiles_n = (d.N + 127) / 128;
  const int nctr = 1 + nu * nph;
  const size_t bd = desc.size() * sizeof(TcgDesc), bi = items.size() * sizeof(TcgItem);
  const size_t bm = maps.size() * sizeof(CUtensorMap), bc = (size_t)nctr * sizeof(unsigned);
  auto al = [](size_t x) { return (x + 127) / 128 * 128; };
  char* mem = nullptr;
  if (cudaMalloc(&mem, al(bm) + al(bd) + al(bi) + al(bc)) != cudaSuccess) { cudaGetLastError(); return; }
  T.fmaps = reinterpret_cast<CUtensorMap*>(mem);
  T.fdesc = reinterpret_cast<TcgDesc*>(mem + al(bm));
  T.fitems = reinterpret_cast<TcgItem*>(mem + al(bm) + al(bd));
  T.fctr = reinterpret_cast<unsigned*>(mem + al(bm) + al(bd) + al(bi));
  cudaMemcpy(T.fmaps, maps.data(), bm, cudaMemcpyHostToDevice);
  cudaMemcpy(T.fdesc, desc.data(), bd, cudaMemcpyHostToDevice);
  cudaMemcpy(T.fitems, items.data(), bi, cudaMemcpyHostToDevice);
  cudaMemset(T.fctr, 0, bc);
  T.flow_mem = mem;
  T.n_fitems = (int)items.size();
  T.n_fctr = nctr;
}

orth_status_t build_compose_tc(Plan& P) {
  auto* T = new TcComposePlan();
  P.tcc = T;
  // ---- bf16 workspace layout (element offsets), then one allocation
  int64_t off = 0;
  auto take = [&](int64_t n) { const int64_t o = off; off += pad_up(n, kPadBF16); return o; };
  struct MatB { int64_t h = -1, l = -1; int ld = 0; };
  std::vector<MatB> mb(P.mats.size()), pb(P.mats.size()), qb(P.mats.size());   // copies, P, I - P
  struct UnitB { int64_t ping_h, ping_l, pong_h, pong_l, tr_h, tr_l; int ld, ldt; };
  std::vector<UnitB> ub(P.comp_units.size());
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    const LayerInfo& L = P.layers[u.layer];
    const int base = L.first_mat + u.group * L.mats_per_group;
    if (u.ping >= 0) {   // BCOP chain: Q, U copies, projectors, tap buffers
      for (int j = 0; j < 1 + 2 * (L.kp - 1); ++j) {
        const MatInfo& M = P.mats[base + j];
        const int ld = (int)pad_up(M.n, 8);
        mb[base + j].ld = ld;
        mb[base + j].h = take(M.m * ld);
        mb[base + j].l = take(M.m * ld);
        if (j > 0) {
          const int ldc = (int)pad_up(M.m, 8);
          pb[base + j].ld = qb[base + j].ld = ldc;
          pb[base + j].h = take(M.m * ldc); pb[base + j].l = take(M.m * ldc);
          qb[base + j].h = take(M.m * ldc); qb[base + j].l = take(M.m * ldc);
        }
      }
      UnitB b{};
      b.ld = (int)pad_up(u.c, 8);
      const int64_t tap = (int64_t)u.rows * b.ld;
      b.ping_h = take(tap * L.kp * L.kp); b.ping_l = take(tap * L.kp * L.kp);
      b.pong_h = take(tap * L.kp * L.kp); b.pong_l = take(tap * L.kp * L.kp);
      b.ldt = (int)pad_up(u.rows, 8);
      b.tr_h = b.tr_l = -1;
      if (L.cons == CONS_AOC) {
        b.tr_h = take((int64_t)u.c * b.ldt * L.kp * L.kp);
        b.tr_l = take((int64_t)u.c * b.ldt * L.kp * L.kp);
      }
      ub[ui] = b;
    }
    if (L.cons == CONS_AOC) {   // RKO phase split
      const MatInfo& R = P.mats[base + L.mats_per_group - 1];
      const int ld = (int)pad_up(L.c_mid, 8);
      mb[base + L.mats_per_group - 1].ld = ld;
      mb[base + L.mats_per_group - 1].h = take((int64_t)L.s * L.s * R.m * ld);
      mb[base + L.mats_per_group - 1].l = take((int64_t)L.s * L.s * R.m * ld);
    }
  }
  // descriptors are sized before allocation; pointers resolved after
  if (cudaMalloc(&T->arena, (size_t)std::max<int64_t>(off, 64) * 2) != cudaSuccess) {
    cudaGetLastError();
    set_error("compose workspace allocation failed");
    return ORTH_ERR_OUT_OF_MEMORY;
  }
  cudaMemset(T->arena, 0, (size_t)std::max<int64_t>(off, 64) * 2);   // zero padding of every bf16 row
  auto bf = [&](int64_t o) { return reinterpret_cast<__nv_bfloat16*>(T->arena) + o; };
  float* comp = P.d_comp;
  // ---- cvt items
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    const LayerInfo& L = P.layers[u.layer];
    const int base = L.first_mat + u.group * L.mats_per_group;
    for (int j = 0; j < L.mats_per_group; ++j) {
      const MatB& b = mb[base + j];
      if (b.h < 0) continue;
      const MatInfo& M = P.mats[base + j];
      if (M.m == 0 || M.n == 0) continue;
      CvtItem c{};
      c.src_off = M.off; c.m = (int)M.m; c.n = (int)M.n; c.ld = b.ld;
      c.mode = (M.role == ROLE_R) ? 1 : 0;
      c.s2 = L.s * L.s;
      c.dh = bf(b.h); c.dl = bf(b.l);
      T->cvt.push_back(c);
    }
  }
  // ---- projectors P = U U^T and I - P
  std::vector<int> unit_of_mat(P.mats.size(), -1);
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const LayerInfo& L = P.layers[P.comp_units[ui].layer];
    const int base = L.first_mat + P.comp_units[ui].group * L.mats_per_group;
    for (int j = 0; j < L.mats_per_group; ++j) unit_of_mat[base + j] = (int)ui;
  }
  for (size_t i = 0; i < P.mats.size(); ++i) {
    if (pb[i].h < 0) continue;
    T->proj_unit.push_back(unit_of_mat[i]);
    const MatInfo& U = P.mats[i];
    const int c = (int)U.m;
    TcgDesc d = mkdesc(c, c, (int)U.n);
    d.seg_begin = (int)T->proj.s.size(); d.seg_count = 1;
    T->proj.s.push_back(TcgSeg{bf(mb[i].h), bf(mb[i].l), bf(mb[i].h), bf(mb[i].l), mb[i].ld, mb[i].ld});
    d.ldo = pb[i].ld;
    d.oh = bf(pb[i].h); d.ol = bf(pb[i].l);
    d.o2h = bf(qb[i].h); d.o2l = bf(qb[i].l);
    d.alpha2 = -1.0f; d.diag2 = 1.0f;
    if (U.n == 0) { d.K = 0; d.seg_count = 0; }   // rank-0 projector: P = 0, I - P = I
    T->proj.d.push_back(d);
  }
  // ---- chain substeps
  int max_sub = 0;
  for (auto& u : P.comp_units)
    if (u.ping >= 0) max_sub = std::max(max_sub, 2 * (P.layers[u.layer].kp - 1));
  T->chain.assign(max_sub, TcgPhase{});
  T->chain_unit.assign(max_sub, std::vector<int>());
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    if (u.ping < 0) continue;
    const LayerInfo& L = P.layers[u.layer];
    const int base = L.first_mat + u.group * L.mats_per_group;
    const UnitB& b = ub[ui];
    const int r = u.rows, c = u.c, ld = b.ld;
    const int64_t tapb = (int64_t)r * ld, tapf = (int64_t)r * c;
    int kh = 1, kw = 1;
    const __nv_bfloat16 *in_h = bf(mb[base].h), *in_l = bf(mb[base].l);   // Q rows [:r]
    const int nsub = 2 * (L.kp - 1);
    for (int t = 0; t < nsub; ++t) {
      const bool vert = (t % 2) == 0;
      const int uidx = base + 1 + t;
      const int oh = vert ? kh + 1 : kh, ow = vert ? kw : kw + 1;
      const bool to_ping = (t % 2) == 0;
      const int64_t out_f = to_ping ? u.ping : u.pong;
      __nv_bfloat16* out_h = bf(to_ping ? b.ping_h : b.pong_h);
      __nv_bfloat16* out_l = bf(to_ping ? b.ping_l : b.pong_l);
      TcgPhase& ph = T->chain[t];
      for (int p = 0; p < oh; ++p)
        for (int q = 0; q < ow; ++q) {
          const bool has_cur = vert ? (p < kh) : (q < kw);
          const bool has_prev = vert ? (p >= 1) : (q >= 1);
          const int cur = p * kw + q, prev = vert ? (p - 1) * kw + q : p * kw + q - 1;
          TcgDesc d = mkdesc(r, c, c);
          d.seg_begin = (int)ph.s.size();
          if (has_cur)
            ph.s.push_back(TcgSeg{in_h + cur * tapb, in_l + cur * tapb, bf(pb[uidx].h), bf(pb[uidx].l), ld, pb[uidx].ld});
          if (has_prev)
            ph.s.push_back(TcgSeg{in_h + prev * tapb, in_l + prev * tapb, bf(qb[uidx].h), bf(qb[uidx].l), ld, qb[uidx].ld});
          d.seg_count = (int)ph.s.size() - d.seg_begin;
          const int o = p * ow + q;
          // FP32 chain taps are read only by the emit of a BCOP unit's final step; every other step's
          // consumer (the next step, the AOC) reads the BF16 hi/lo copies -- skipping the FP32 stores cuts a
          // third of the bytes of these store-bound epilogues (~55 GB/s per SM, tools/micro/tma_store_bw.cu)
          if (t == nsub - 1 && L.cons != CONS_AOC) { d.f = comp + out_f + o * tapf; d.ldf = c; }
          d.oh = out_h + o * tapb; d.ol = out_l + o * tapb; d.ldo = ld;
          if (t == nsub - 1 && b.tr_h >= 0) {
            d.th = bf(b.tr_h) + (int64_t)o * c * b.ldt;
            d.tl = bf(b.tr_l) + (int64_t)o * c * b.ldt;
            d.ldt = b.ldt;
          }
          ph.d.push_back(d);
          T->chain_unit[t].push_back((int)ui);
        }
      kh = oh; kw = ow;
      in_h = out_h; in_l = out_l;
    }
  }
  // ---- AOC: K[p,q] = sum_ab R_ab Kb[p-a, q-b]
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    const LayerInfo& L = P.layers[u.layer];
    if (L.cons != CONS_AOC) continue;
    const int base = L.first_mat + u.group * L.mats_per_group;
    const MatB& rb = mb[base + L.mats_per_group - 1];
    const UnitB& b = ub[ui];
    const int s = L.s, kp = L.kp, k = L.k;
    const int64_t rblk = (int64_t)L.co * rb.ld;          // one phase block of the split R
    const int64_t ttap = (int64_t)u.c * b.ldt;            // one transposed chain tap
    for (int p = 0; p < k; ++p)
      for (int q = 0; q < k; ++q) {
        TcgDesc d = mkdesc(L.co, L.ci, L.c_mid);
        d.seg_begin = (int)T->aoc.s.size();
        for (int a = 0; a < s; ++a)
          for (int bb = 0; bb < s; ++bb) {
            const int ta = p - a, tb = q - bb;
            if (ta < 0 || tb < 0 || ta >= kp || tb >= kp) continue;
            const int ph = a * s + bb, t = ta * kp + tb;
            T->aoc.s.push_back(TcgSeg{bf(rb.h) + ph * rblk, bf(rb.l) + ph * rblk, bf(b.tr_h) + t * ttap,
                                      bf(b.tr_l) + t * ttap, rb.ld, b.ldt});
          }
        d.seg_count = (int)T->aoc.s.size() - d.seg_begin;
        d.f = comp + u.fin + (int64_t)(p * k + q) * L.co * L.ci;
        d.ldf = L.ci;
        T->aoc.d.push_back(d);
        T->aoc_unit.push_back((int)ui);
      }
  }
  // ---- upload descriptors
  finish(T->proj);
  finish(T->aoc);
  for (auto& ph : T->chain) finish(ph);
  cudaError_t e = cudaSuccess;
  auto up = [&](auto& vec, auto*& dptr) {
    using V = typename std::remove_reference<decltype(vec)>::type::value_type;
    if (vec.empty() || e != cudaSuccess) return;
    e = cudaMalloc((void**)&dptr, vec.size() * sizeof(V));
    if (e == cudaSuccess) e = cudaMemcpy(dptr, vec.data(), vec.size() * sizeof(V), cudaMemcpyHostToDevice);
  };
  up(T->cvt, T->dcvt);
  for (TcgPhase* ph : {&T->proj, &T->aoc}) { up(ph->d, ph->dd); up(ph->s, ph->ds); }
  for (auto& ph : T->chain) { up(ph.d, ph.dd); up(ph.s, ph.ds); }
  if (e != cudaSuccess) {
    set_error("compose descriptor upload failed: %s", cudaGetErrorString(e));
    return ORTH_ERR_CUDA;
  }
  static const bool no_tma = std::getenv("ORTH_COMPOSE_NO_TMA") != nullptr;   // A/B switch
  if (!no_tma) {
    for (TcgPhase* ph : {&T->proj, &T->aoc})
      if (!build_phase_maps(*ph)) { if (ph->dmaps) cudaFree(ph->dmaps); ph->dmaps = nullptr; }
    for (auto& ph : T->chain)
      if (!build_phase_maps(ph)) { if (ph.dmaps) cudaFree(ph.dmaps); ph.dmaps = nullptr; }
  }
  static const bool no_flow = std::getenv("ORTH_COMPOSE_PHASED") != nullptr;   // A/B: per-phase launches
  if (!no_tma && !no_flow) build_compose_flow(P, *T);
  return ORTH_OK;
}

void free_compose_tc(Plan& P) {
  TcComposePlan* T = P.tcc;
  if (!T) return;
  if (T->arena) cudaFree(T->arena);
  if (T->dcvt) cudaFree(T->dcvt);
  if (T->flow_mem) cudaFree(T->flow_mem);
  for (TcgPhase* ph : {&T->proj, &T->aoc}) {
    if (ph->dd) cudaFree(ph->dd);
    if (ph->ds) cudaFree(ph->ds);
    if (ph->dmaps) cudaFree(ph->dmaps);
  }
  for (auto& ph : T->chain) {
    if (ph.dd) cudaFree(ph.dd);
    if (ph.ds) cudaFree(ph.ds);
    if (ph.dmaps) cudaFree(ph.dmaps);
  }
  delete T;
  P.tcc = nullptr;
}

int launch_compose_tc(Plan& P, const float* ortho, void* stream) {
  TcComposePlan* T = P.tcc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!T->cvt.empty()) {
    int maxm = 1;
    for (auto& c : T->cvt) maxm = std::max(maxm, c.m);
    dim3 grid((unsigned)std::min(maxm, 32), (unsigned)T->cvt.size());   // fewer, fuller CTAs
    launch_pdl(cvt_kernel, grid, dim3(256), 0, s, (const CvtItem*)T->dcvt, ortho, T->fctr, T->n_fctr);
    P.launches++;
    if (int e = (int)cudaGetLastError()) return e;
  }
  if (T->flow_mem) {   // every phase in one dataflow launch
    const size_t smem_p = 1024 + (size_t)S * 4 * 128 * 128 + (size_t)kTcpSf * 4;
    static bool attr_f = false;
    if (!attr_f) {
      cudaFuncSetAttribute(tcg_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
      attr_f = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(T->n_fitems, sms);
    if (T->cvt.empty()) cudaMemsetAsync(T->fctr, 0, (size_t)T->n_fctr * sizeof(unsigned), s);
    launch_pdl(tcg_flow, dim3(grid), dim3(kTcpThreads), smem_p, s, (const TcgDesc*)T->fdesc,
               (const TcgItem*)T->fitems, T->n_fitems, (const CUtensorMap*)T->fmaps, T->fctr);
    P.launches++;
    return (int)cudaGetLastError();
  }
  int e = launch_phase(T->proj, s);
  P.launches += T->proj.tiles ? 1 : 0;
  for (auto& ph : T->chain) {
    if (e) return e;
    e = launch_phase(ph, s);
    P.launches += ph.tiles ? 1 : 0;
  }
  if (!e) {
    e = launch_phase(T->aoc, s);
    P.launches += T->aoc.tiles ? 1 : 0;
  }
  return e;
}

}  // namespace orth
