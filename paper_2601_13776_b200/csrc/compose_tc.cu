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
#include <type_traits>
#include <vector>

#include "orth_internal.h"
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
};
struct TcComposePlan {
  void* arena = nullptr;
  std::vector<CvtItem> cvt;
  CvtItem* dcvt = nullptr;
  TcgPhase proj, aoc;
  std::vector<TcgPhase> chain;
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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

// FP32 ortho -> BF16 hi/lo copies (row-major padded, or the RKO phase split)
__global__ void __launch_bounds__(256) cvt_kernel(const CvtItem* __restrict__ items, const float* __restrict__ ortho) {
  const CvtItem it = items[blockIdx.y];
  const int64_t total = (int64_t)it.m * it.n;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int r = (int)(e / it.n), col = (int)(e - (int64_t)r * it.n);
    __nv_bfloat16 h, l;
    split(ortho[it.src_off + e], h, l);
    int64_t o;
    if (it.mode == 0) o = (int64_t)r * it.ld + col;
    else {
      const int ph = col % it.s2, j = col / it.s2;   // R[o, j s^2 + ab] -> block ab, row o, column j
      o = ((int64_t)ph * it.m + r) * it.ld + j;
    }
    it.dh[o] = h;
    it.dl[o] = l;
  }
}

int launch_phase(const TcgPhase& ph, cudaStream_t s) {
  if (!ph.tiles) return 0;
  const size_t smem = 1024 + (size_t)S * 4 * 128 * 128;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  tcg_kernel<<<ph.tiles, 256, smem, s>>>(ph.dd, (int)ph.d.size(), ph.ds);
  return (int)cudaGetLastError();
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
  for (size_t i = 0; i < P.mats.size(); ++i) {
    if (pb[i].h < 0) continue;
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
          d.f = comp + out_f + o * tapf; d.ldf = c;
          d.oh = out_h + o * tapb; d.ol = out_l + o * tapb; d.ldo = ld;
          if (t == nsub - 1 && b.tr_h >= 0) {
            d.th = bf(b.tr_h) + (int64_t)o * c * b.ldt;
            d.tl = bf(b.tr_l) + (int64_t)o * c * b.ldt;
            d.ldt = b.ldt;
          }
          ph.d.push_back(d);
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
  return ORTH_OK;
}

void free_compose_tc(Plan& P) {
  TcComposePlan* T = P.tcc;
  if (!T) return;
  if (T->arena) cudaFree(T->arena);
  if (T->dcvt) cudaFree(T->dcvt);
  for (TcgPhase* ph : {&T->proj, &T->aoc}) { if (ph->dd) cudaFree(ph->dd); if (ph->ds) cudaFree(ph->ds); }
  for (auto& ph : T->chain) { if (ph.dd) cudaFree(ph.dd); if (ph.ds) cudaFree(ph.ds); }
  delete T;
  P.tcc = nullptr;
}

int launch_compose_tc(Plan& P, const float* ortho, void* stream) {
  TcComposePlan* T = P.tcc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!T->cvt.empty()) {
    int64_t maxe = 1;
    for (auto& c : T->cvt) maxe = std::max<int64_t>(maxe, (int64_t)c.m * c.n);
    dim3 grid((unsigned)std::min<int64_t>(64, (maxe + 255) / 256), (unsigned)T->cvt.size());
    cvt_kernel<<<grid, 256, 0, s>>>(T->dcvt, ortho);
    P.launches++;
    if (int e = (int)cudaGetLastError()) return e;
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
