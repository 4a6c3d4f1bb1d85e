// Persistent tensor-core Bjorck / Newton-Schulz (a3; residual form
// R16): ALL T iterations of all matrices in ONE cooperative launch.
//
// Why: the per-phase kernels (ns_tc.cu) pay a launch, a TMEM allocation, a
// barrier setup and a cold pipeline for every one of the 2T phases, and a
// phase waits for the slowest tile of ANY matrix.  Here every matrix (or a
// bundle of small matrices) belongs to a GROUP of G co-resident CTAs that
// runs its 2T phases on its own, synchronising only its own CTAs between
// phases (a global-memory barrier; nothing when G = 1).  Groups never wait
// for each other.  Host-side partition: plan.cpp/build_ns_persist (cost
// model + LPT).
//
// CTA roles (kThreads = 320 threads, one CTA per SM, kSlots x 32 KB ring +
// 96 KB epilogue staging):
//   warp 0  TMA producer: 128x64 BF16 operand tiles (K-major rows of X / R,
//           or MN-major columns of row-major X) into a kSlots (= 4) ring of
//           32 KB slots (a 1-pass k-block takes one slot, a 3-pass hi/lo
//           k-block two)
//   warp 1  TMEM allocation + the single-thread tcgen05.mma issuer, FP32
//           accumulators double-buffered in TMEM (2 x 128 columns; 2 x 256
//           for the 128 x 256 update tiles of the phase-synchronous kernel)
//   warps 2-9  epilogue (kEpiWarps = 8: lane quarter x column half): TMEM ->
//           registers -> per-warp smem transpose -> coalesced FP32 / BF16 row
//           stores (Gram: R = I - acc; update: X' = C + beta acc), overlapping
//           the next tile's mainloop.
// Two schedules share this tile pipeline: ns_persist_kernel (phase-synchronous
// CTA groups: epilogue writes -> proxy fence -> group barrier -> a monotonic
// smem counter that releases the producer into the next phase) and
// ns_flow_kernel (dataflow: (phase, matrix, tile) items claimed in one global
// order, each waiting on its matrix's per-phase counter).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <numeric>
#include <vector>

#include "orth_internal.h"
#include "umma.cuh"
#include "tma_host.h"

// Device-side tracing (per-phase / per-tile globaltimer stamps) is compiled in
// only with -DORTH_NSP_TRACE (diagnostics builds: ORTH_NVCC_FLAGS=-DORTH_NSP_TRACE).
#ifdef ORTH_NSP_TRACE
#define NSP_TRACE(x) x
#else
#define NSP_TRACE(x)
#endif

namespace orth {

struct NspBufs {
  float* X[2];
  float* R;
  __nv_bfloat16 *xh[2], *xl[2], *rh, *rl;
};

struct NspPhases {
  uint8_t f[kNspMaxPhases];   // bit0 gram, bit1 3-pass, bit2 parity of X read, bit3 write lo, bit4 write fp32 R
  int32_t n;
  unsigned long long* trace;  // diagnostics (ORTH_NS_TRACE): per CTA, globaltimer at start and at each phase end
  unsigned long long* ttrace; // diagnostics: per tile {slot counter, then 4 words per record}
};

namespace {

constexpr int kThreads = 320;    // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int kSlot = 32768;
#ifdef ORTH_NS_SLOTS
constexpr int kSlots = ORTH_NS_SLOTS;
#else
constexpr int kSlots = 4;
#endif
constexpr int kEpiWarps = 8;
// per epilogue warp: the accumulator chunk Sw (32 x 32 fp32) and the C tile of
// both chunks Sc[2] (32 x 32 fp32 each), float4 slots XOR-swizzled by row
constexpr int kStageFloats = kEpiWarps * 3 * 32 * 32;
constexpr size_t kSmem = 1024 + (size_t)kSlots * kSlot + (size_t)kStageFloats * 4;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <class T>
__device__ __forceinline__ T pick(T const (&a)[2], int i) { return i ? a[1] : a[0]; }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {   // low half = a
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= target, then acquire.  The polls are relaxed: an ld.acquire.gpu
// compiles to a load + CCTL.IVALL, and a producer spinning on it invalidates the
// SM's L1 every few tens of ns, stalling the epilogue warps' shared/global traffic.
// One fence after the observed value gives the same acquire ordering.
__device__ __forceinline__ void wait_geq_acquire(const unsigned* p, unsigned target, bool sleep) {
  while (ld_relaxed_gpu(p) < target)
    if (sleep) __nanosleep(32);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire_cta_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(umma::smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(umma::smem_u32(p)), "r"(v) : "memory");
}

// Group barrier over G co-resident CTAs: a monotonic arrival counter per
// group (zeroed by the scale kernel that precedes every launch); barrier k
// completes when the counter reaches k * G.  One release-reduction per CTA,
// acquire polls (measured 1.2 us for 148 CTAs vs 2.7 us for count+generation).
__device__ __forceinline__ void group_sync(unsigned* bar, unsigned target) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
  wait_geq_acquire(bar, target, false);
}

__device__ __forceinline__ void load_operand(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int k0, int mn0,
                                             int kind) {
  if (kind == 3) {          // columns of row-major X, 3-D map (64 MN, K, MN / 64): both 64-wide blocks in one box
    umma::tma_load_3d(dst, map, bar, 0, k0, mn0 >> 6);
  } else if (kind == 1) {   // columns of row-major X: two 64 (MN) x 64 (K) boxes
    umma::tma_load_2d(dst, map, bar, mn0, k0);
    umma::tma_load_2d(dst + 8192, map, bar, mn0 + 64, k0);
  } else {                  // rows: one 64 (K) x 128 box
    umma::tma_load_2d(dst, map, bar, k0, mn0);
  }
}
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int q, int mn_major) {
  return mn_major ? umma::sdesc_sw128_mn(base + 2048 * q, 8192) : umma::sdesc_sw128(base + 32 * q);
}

__global__ void __launch_bounds__(kThreads, 1)
    ns_persist_kernel(const NsDesc* __restrict__ dg, const NsDesc* __restrict__ du, const NsTile* __restrict__ tiles,
                      const NsGroup* __restrict__ ctas, unsigned* bars,
                      NspBufs bufs, const CUtensorMap* __restrict__ maps, const __grid_constant__ NspPhases ph) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  float* stage = reinterpret_cast<float*>(smem + kSlots * kSlot);
  __shared__ uint64_t full_bar[kSlots], empty_bar[kSlots], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int phase_done;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's ranges live in shared memory and are re-read where used (keeps
  // them out of the register budget: 10 warps cap the kernel at 168 registers)
  __shared__ NsGroup grp_sh;
  __shared__ __align__(16) uint32_t desc_sh[kEpiWarps][32];
  if (tid == 0) grp_sh = ctas[blockIdx.x];
  const volatile NsGroup& grp = grp_sh;

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], kEpiWarps);
    }
    phase_done = 0;
    umma::fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc(&tmem_base_sh, 512);   // two 256-column accumulators (wide update tiles)
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t ring = umma::smem_u32(smem);
  NSP_TRACE(if (ph.trace && tid == 0) {
    const unsigned long long t = gtimer();
    ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1)] = t;
    for (int q = 0; q < 4 * ph.n; ++q) ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1) + 1 + q] = t;
  })

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      uint32_t used = 0, epar = 0;
      int cnt = 0;
      for (int p = 0; p < ph.n; ++p) {
        const int f = ph.f[p], gram = f & 1, split = (f >> 1) & 1, par = (f >> 2) & 1;
        if (p > 0)
          while (ld_acquire_cta_shared(&phase_done) < p) __nanosleep(20);
        fence_proxy_async_global();   // order the group's generic writes before these async-proxy reads
        NSP_TRACE(if (ph.trace) ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1) + 1 + 4 * p + 0] = gtimer());
        const NsDesc* D = gram ? dg : du;
        const int tb = gram ? grp.g_begin : grp.u_begin, te = gram ? grp.g_end : grp.u_end;
        const int w = split ? 2 : 1;
        for (int t = tb; t < te; ++t) {
          const NsTile tl = tiles[t];
          const NsDesc d = D[tl.desc];
          // wide update tile (epi 4, 1-pass only): 128 x 256, B = 256 rows in two adjacent slots
          const bool wide = !gram && d.epi == 4 && !split;
          const int ws = wide ? 2 : w;
          const int m0 = (tl.local / d.tiles_n) * 128, n0 = (tl.local % d.tiles_n) * (wide ? 256 : 128);
          const int nk = (d.K + 63) / 64, a_mn = d.a_kind & 1, b_mn = d.b_kind & 1, ak = d.a_kind, bk = d.b_kind;
          const bool sym = gram && m0 == n0;   // diagonal Gram tile: B == A, loaded once
          const CUtensorMap* ma = maps + d.map_a + 2 * par;
          const CUtensorMap* mb = maps + d.map_b + 2 * par;
          for (int kb = 0; kb < nk; ++kb) {
            if (ws == 2 && cnt % kSlots == kSlots - 1) ++cnt;   // a hi/lo or wide stage takes two adjacent slots
            const int s = cnt % kSlots;
            for (int q = s; q < s + ws; ++q) {
              if ((used >> q) & 1u) {
                umma::mbar_wait(&empty_bar[q], (epar >> q) & 1u);
                epar ^= 1u << q;
              }
              used |= 1u << q;
            }
            const uint32_t sa = ring + s * kSlot;
            if (wide) {   // A 16 KB + B 256 rows (32 KB)
              umma::mbar_arrive_expect_tx(&full_bar[s], 16384u + 32768u);
              load_operand(sa, ma, &full_bar[s], kb * 64, m0, ak);
              load_operand(sa + 16384, mb, &full_bar[s], kb * 64, n0, bk);
              load_operand(sa + 32768, mb, &full_bar[s], kb * 64, n0 + 128, bk);
              cnt += 2;
              continue;
            }
            umma::mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(sym ? w * kSlot / 2 : w * kSlot));
            load_operand(sa, ma, &full_bar[s], kb * 64, m0, ak);
            if (!sym) load_operand(sa + 16384, mb, &full_bar[s], kb * 64, n0, bk);
            if (split) {
              load_operand(sa + 32768, ma + 1, &full_bar[s], kb * 64, m0, ak);
              if (!sym) load_operand(sa + 49152, mb + 1, &full_bar[s], kb * 64, n0, bk);
            }
            cnt += w;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      uint32_t fpar = 0;
      int cnt = 0, acc = 0;
      for (int p = 0; p < ph.n; ++p) {
        const int f = ph.f[p], gram = f & 1, split = (f >> 1) & 1;
        const NsDesc* D = gram ? dg : du;
        const int tb = gram ? grp.g_begin : grp.u_begin, te = gram ? grp.g_end : grp.u_end;
        const int w = split ? 2 : 1;
        for (int t = tb; t < te; ++t) {
          const NsTile tl = tiles[t];
          const NsDesc* dp = D + tl.desc;
          const int nk = (__ldg(&dp->K) + 63) / 64, a_mn = __ldg(&dp->a_kind) & 1, b_mn = __ldg(&dp->b_kind) & 1;
          const int tn = __ldg(&dp->tiles_n);
          const bool sym = gram && (tl.local / tn) == (tl.local % tn);
          const bool wide = !gram && __ldg(&dp->epi) == 4 && !split;
          const int ws = wide ? 2 : w;
          const uint32_t idesc = (wide ? umma::idesc_bf16(128, 256) : umma::idesc_bf16(128, 128)) |
                                 ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
          const int buf = acc & 1;
          if (acc >= 2) umma::mbar_wait(&tempty_bar[buf], ((acc >> 1) - 1) & 1);
          umma::tc_fence_after();
          const uint32_t dt = tmem + buf * 256;
          for (int kb = 0; kb < nk; ++kb) {
            if (ws == 2 && cnt % kSlots == kSlots - 1) ++cnt;
            const int s = cnt % kSlots;
            umma::mbar_wait(&full_bar[s], (fpar >> s) & 1u);
            fpar ^= 1u << s;
            umma::tc_fence_after();
            const uint32_t ah = ring + s * kSlot, al = ah + 32768;
            const uint32_t bh = sym ? ah : ah + 16384, bl = sym ? al : ah + 49152;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint64_t dah = op_desc(ah, q, a_mn), dbh = op_desc(bh, q, b_mn);
              umma::mma_bf16(dt, dah, dbh, idesc, (kb | q) != 0);
              if (split) {
                umma::mma_bf16(dt, dah, op_desc(bl, q, b_mn), idesc, 1);
                umma::mma_bf16(dt, op_desc(al, q, a_mn), dbh, idesc, 1);
              }
            }
            umma::mma_commit(&empty_bar[s]);
            if (ws == 2) umma::mma_commit(&empty_bar[s + 1]);
            cnt += ws;
          }
          umma::mma_commit(&tfull_bar[buf]);
          ++acc;
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    // 8 warps: warp w reads TMEM lanes 32*(w%4) (rows row0..row0+31) and the
    // 64-column half ch of the accumulator, in two 32-column chunks.  The C
    // tile of both chunks is prefetched into smem with cp.async before the
    // accumulator is ready.  Chunk: tcgen05.ld (thread = row) -> float4 rows
    // into a swizzled 32x32 smem tile -> row pass with 8 lanes per row (float4
    // C from smem, float4 FP32 stores, 8-byte BF16 stores), 4 rows per step.
    // Nothing tile-sized lives in registers (10 warps cap the kernel at 168).
    const int ew = warp - 2, row0 = (warp & 3) * 32, ch = ew >> 2;
    float* Sw = stage + ew * 3 * 1024;
    float* Sc = Sw + 1024;
    const int rsub = lane >> 3, q4 = lane & 7, c4 = q4 * 4;
    int acc = 0;
    for (int p = 0; p < ph.n; ++p) {
      const int f = ph.f[p], gram = f & 1, par = (f >> 2) & 1, write_lo = (f >> 3) & 1, write_f = (f >> 4) & 1;
      const NsDesc* D = gram ? dg : du;
      const int tb = gram ? grp.g_begin : grp.u_begin, te = gram ? grp.g_end : grp.u_end;
      for (int t = tb; t < te; ++t) {
        const NsTile tl = tiles[t];
        // this tile's descriptor -> a per-warp smem copy (one word per lane), so the
        // fields cost an LDS, not an L2 round trip, wherever they are used below
        {
          static_assert(sizeof(NsDesc) <= 32 * 4, "NsDesc must fit one word per lane");
          const uint32_t* srcw = reinterpret_cast<const uint32_t*>(D + tl.desc);
          if (lane < (int)(sizeof(NsDesc) / 4)) desc_sh[ew][lane] = __ldg(srcw + lane);
          __syncwarp();
        }
        const NsDesc* dp = reinterpret_cast<const NsDesc*>(desc_sh[ew]);
        const int tiles_n = dp->tiles_n;
        const bool upd = (dp->epi) == 1 || (dp->epi) == 4;
        const int nh = ((dp->epi) == 4 && !((f >> 1) & 1)) ? 2 : 1;   // wide update tile: two 128-column halves
        const int m0 = (tl.local / tiles_n) * 128 + row0;
        const int64_t f_off = (dp->f_off), ldf = (dp->ldf);
        const int M = (dp->M), N = (dp->N);
        const int buf = acc & 1;
        NSP_TRACE(unsigned long long t_start = 0ull; unsigned long long t_full = 0ull;)
#ifdef ORTH_NSP_TRACE
        long long cyc[6];
#endif
#pragma unroll 1
        for (int h = 0; h < nh; ++h) {
        const int n0 = (tl.local % tiles_n) * (128 * nh) + h * 128 + ch * 64;
        if (upd) {   // C = X (fp32) rows m0.., cols n0..n0+63 -> Sc[0..1]
          const float* Cm = bufs.X[0] + f_off;
          const bool fv4 = (ldf & 3) == 0;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int e = lane + 32 * k, r = e >> 3, q = e & 7;
              const int i = m0 + r, j = n0 + c * 32 + 4 * q;
              float* dst = Sc + c * 1024 + r * 32 + 4 * (q ^ (r & 7));
              const float* src = Cm + (int64_t)i * ldf + j;
              if (fv4 && (j + 3 < N || j >= N)) {
                umma::cp_async16(umma::smem_u32(dst), i < M && j < N ? src : Cm, i < M && j < N);
              } else {   // ragged / unaligned: synchronous scalar path
#pragma unroll
                for (int u = 0; u < 4; ++u) dst[u] = (i < M && j + u < N) ? __ldcg(src + u) : 0.f;
              }
            }
            umma::cp_async_commit();
          }
        }
        NSP_TRACE(if (h == 0) t_start = ph.ttrace ? gtimer() : 0ull);
        if (h == 0) {
          umma::mbar_wait(&tfull_bar[buf], (acc >> 1) & 1);
          umma::tc_fence_after();
        }
        NSP_TRACE(if (h == 0) t_full = ph.ttrace ? gtimer() : 0ull);
#ifdef ORTH_NSP_TRACE
        if (h == 0) cyc[0] = clock64();
#endif
        NSP_TRACE(if (ph.trace && ew == 0 && lane == 0 && t == tb) ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1) + 1 + 4 * p + 1] = gtimer());
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float v[16];
            umma::tmem_ld16(tmem + buf * 256 + h * 128 + ch * 64 + c * 32 + hh * 16 + ((uint32_t)row0 << 16), v);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *reinterpret_cast<float4*>(Sw + lane * 32 + 4 * ((hh * 4 + k) ^ (lane & 7))) =
                  make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          }
          if (c == 1 && h == nh - 1) {   // accumulator drained: hand the TMEM buffer back to the MMA warp
            umma::tc_fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&tempty_bar[buf]);
          }
          if (upd) {
            if (c == 0) umma::cp_async_wait<1>();
            else umma::cp_async_wait<0>();
          }
          __syncwarp();
          NSP_TRACE(if (c == 0) cyc[1] = clock64());
          // per-chunk constants re-derived here (cheap) instead of being held in registers
          const bool wf = upd || write_f;
          const int ldb16 = upd ? (dp->ldx) : (dp->ldr);
          const int64_t b_off = upd ? (dp->bx_off) : (dp->br_off);
          __nv_bfloat16* oh = (upd ? pick(bufs.xh, par ^ 1) : bufs.rh) + b_off;
          __nv_bfloat16* ol = (upd ? pick(bufs.xl, par ^ 1) : bufs.rl) + b_off;
          float* F = (upd ? bufs.X[0] : bufs.R) + f_off;
          const bool fv4 = (ldf & 3) == 0;
          const float alpha = (dp->alpha), beta = (dp->beta), diag = (dp->diag);
          const float* Scc = Sc + c * 1024;
          // Fast path (warp-uniform): an interior 32 x 32 chunk -- every row < M, every column < N (and so
          // inside the padded BF16 row), 16-byte FP32 rows, no diagonal element -- needs none of the per-element
          // predicates below: straight-line float4 math and incrementally advanced row pointers.  (The generic
          // loop costs ~60 instructions per 4-element group; this one ~20.)
          const int jc0 = n0 + c * 32;
          const bool interior = m0 + 31 < M && jc0 + 31 < N && fv4 &&
                                (diag == 0.f || m0 + 31 < jc0 || jc0 + 31 < m0);
          if (interior) {
            float* fr = F + (int64_t)(m0 + rsub) * ldf + jc0 + c4;
            __nv_bfloat16* hr = oh + (int64_t)(m0 + rsub) * ldb16 + jc0 + c4;
            __nv_bfloat16* lr = ol + (int64_t)(m0 + rsub) * ldb16 + jc0 + c4;
            const int64_t fstep = 4 * ldf, bstep = 4 * (int64_t)ldb16;
#pragma unroll 4
            for (int it = 0; it < 8; ++it) {
              const int rr = 4 * it + rsub;
              const int sw = 4 * (q4 ^ (rr & 7));
              const float4 a = *reinterpret_cast<const float4*>(Sw + rr * 32 + sw);
              float o0, o1, o2, o3;
              if (upd) {
                const float4 cv = *reinterpret_cast<const float4*>(Scc + rr * 32 + sw);
                o0 = fmaf(alpha, a.x, beta * cv.x); o1 = fmaf(alpha, a.y, beta * cv.y);
                o2 = fmaf(alpha, a.z, beta * cv.z); o3 = fmaf(alpha, a.w, beta * cv.w);
              } else {
                o0 = alpha * a.x; o1 = alpha * a.y; o2 = alpha * a.z; o3 = alpha * a.w;
              }
              if (wf) *reinterpret_cast<float4*>(fr) = make_float4(o0, o1, o2, o3);
              const uint32_t h01 = pack_bf16(o0, o1), h23 = pack_bf16(o2, o3);
              *reinterpret_cast<uint2*>(hr) = make_uint2(h01, h23);
              if (write_lo) {
                const uint32_t l01 = pack_bf16(o0 - __uint_as_float(h01 << 16), o1 - __uint_as_float(h01 & 0xFFFF0000u));
                const uint32_t l23 = pack_bf16(o2 - __uint_as_float(h23 << 16), o3 - __uint_as_float(h23 & 0xFFFF0000u));
                *reinterpret_cast<uint2*>(lr) = make_uint2(l01, l23);
              }
              fr += fstep; hr += bstep; lr += bstep;
            }
          } else
#pragma unroll 4
          for (int it = 0; it < 8; ++it) {
            const int rr = 4 * it + rsub;
            const int i = m0 + rr, j = n0 + c * 32 + c4;
            if (i < M) {
              const int sw = 4 * (q4 ^ (rr & 7));
              const float4 a = *reinterpret_cast<const float4*>(Sw + rr * 32 + sw);
              const float4 cv = upd ? *reinterpret_cast<const float4*>(Scc + rr * 32 + sw) : make_float4(0.f, 0.f, 0.f, 0.f);
              float o0 = fmaf(alpha, a.x, beta * cv.x), o1 = fmaf(alpha, a.y, beta * cv.y);
              float o2 = fmaf(alpha, a.z, beta * cv.z), o3 = fmaf(alpha, a.w, beta * cv.w);
              const int dd = i - j;   // diagonal element inside this 4-group
              if (dd == 0) o0 += diag;
              if (dd == 1) o1 += diag;
              if (dd == 2) o2 += diag;
              if (dd == 3) o3 += diag;
              if (j + 3 >= N) {       // ragged right edge: zero beyond N (keeps BF16 padding zero)
                if (j >= N) o0 = 0.f;
                if (j + 1 >= N) o1 = 0.f;
                if (j + 2 >= N) o2 = 0.f;
                o3 = 0.f;
              }
              if (wf && j < N) {
                float* dst = F + (int64_t)i * ldf + j;
                if (fv4 && j + 3 < N) {
                  *reinterpret_cast<float4*>(dst) = make_float4(o0, o1, o2, o3);
                } else {
                  dst[0] = o0;
                  if (j + 1 < N) dst[1] = o1;
                  if (j + 2 < N) dst[2] = o2;
                  if (j + 3 < N) dst[3] = o3;
                }
              }
              if (j < ldb16) {   // ldb16 % 8 == 0, j % 4 == 0: the 4-group lies inside the padded row
                const uint32_t h01 = pack_bf16(o0, o1), h23 = pack_bf16(o2, o3);
                const int64_t bo = (int64_t)i * ldb16 + j;
                *reinterpret_cast<uint2*>(oh + bo) = make_uint2(h01, h23);
                if (write_lo) {
                  const uint32_t l01 = pack_bf16(o0 - __uint_as_float(h01 << 16), o1 - __uint_as_float(h01 & 0xFFFF0000u));
                  const uint32_t l23 = pack_bf16(o2 - __uint_as_float(h23 << 16), o3 - __uint_as_float(h23 & 0xFFFF0000u));
                  *reinterpret_cast<uint2*>(ol + bo) = make_uint2(l01, l23);
                }
              }
            }
          }
          NSP_TRACE(if (c == 0) cyc[2] = clock64());
          if (gram && m0 - row0 < n0 - ch * 64) {
            // upper-triangle Gram tile: also write its mirror R[j][i] = R[i][j] (alpha * acc; no diagonal here)
#pragma unroll 2
            for (int it = 0; it < 8; ++it) {
              const int rt = 4 * it + rsub;                           // column of the chunk = row of the mirror
              const int jg = n0 + c * 32 + rt, ig = m0 + c4;
              if (jg < N && ig < ldb16) {
                float o[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int r = c4 + k;
                  o[k] = ig + k < M ? alpha * Sw[r * 32 + 4 * ((rt >> 2) ^ (r & 7)) + (rt & 3)] : 0.f;
                }
                if (wf) {
                  float* dst = F + (int64_t)jg * ldf + ig;
                  if (fv4 && ig + 3 < M) {
                    *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
                  } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                      if (ig + k < M) dst[k] = o[k];
                  }
                }
                const uint32_t h01 = pack_bf16(o[0], o[1]), h23 = pack_bf16(o[2], o[3]);
                const int64_t bo = (int64_t)jg * ldb16 + ig;
                *reinterpret_cast<uint2*>(oh + bo) = make_uint2(h01, h23);
                if (write_lo) {
                  const uint32_t l01 = pack_bf16(o[0] - __uint_as_float(h01 << 16), o[1] - __uint_as_float(h01 & 0xFFFF0000u));
                  const uint32_t l23 = pack_bf16(o[2] - __uint_as_float(h23 << 16), o[3] - __uint_as_float(h23 & 0xFFFF0000u));
                  *reinterpret_cast<uint2*>(ol + bo) = make_uint2(l01, l23);
                }
              }
            }
          }
          __syncwarp();
          NSP_TRACE(if (c == 0) cyc[3] = clock64());
        }
        }   // halves
#ifdef ORTH_NSP_TRACE
        cyc[4] = clock64();
        if (ph.ttrace && lane == 0) {
          const unsigned long long t_end = gtimer();
          const unsigned long long slot = atomicAdd(ph.ttrace, 1ull);
          if (slot < 65536) {
            unsigned long long* r = ph.ttrace + 1 + 8 * slot;
            r[0] = ((unsigned long long)blockIdx.x << 48) | ((unsigned long long)p << 40) | ((unsigned long long)ew << 36) |
                   ((unsigned long long)tl.desc << 16) | (unsigned long long)tl.local;
            r[1] = t_start;
            r[2] = t_full;
            r[3] = t_end;
            r[4] = cyc[1] - cyc[0];   // chunk 0: TMEM ld + staging (+ C wait)
            r[5] = cyc[2] - cyc[1];   // chunk 0: row pass
            r[6] = cyc[3] - cyc[2];   // chunk 0: mirror pass
            r[7] = cyc[4] - cyc[3];   // chunk 1 (all)
          }
        }
#endif
        ++acc;
      }
      // ---- phase end: publish this CTA's writes, sync the group, release the producer
      NSP_TRACE(if (ph.trace && ew == 0 && lane == 0) ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1) + 1 + 4 * p + 2] = gtimer());
      fence_proxy_async_global();
      umma::named_bar_sync(1, 32 * kEpiWarps);
      if (ew == 0 && lane == 0) {
        if (grp.G > 1) group_sync(bars + grp.gid, (unsigned)(p + 1) * (unsigned)grp.G);
        st_release_cta_shared(&phase_done, p + 1);
        NSP_TRACE(if (ph.trace) ph.trace[(size_t)blockIdx.x * (4 * ph.n + 1) + 1 + 4 * p + 3] = gtimer());
      }
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tmem, 512);
}

// Dataflow NS (default): the same per-tile pipeline as ns_persist_kernel, but
// with no phase barriers at all.  Items (phase, matrix, tile) are claimed in
// one global order through an atomic counter; before loading a tile the
// producer waits for ITS matrix's previous phase (per-matrix monotonic
// counters: Gram(t) needs all update tiles of t-1, update(t) all Gram tiles of
// t), and the epilogue bumps the matrix's counter when the tile's writes are
// visible.  Claim order = dependency order, so with all CTAs co-resident the
// smallest unfinished item can always run (no deadlock); small matrices race
// ahead instead of waiting for the slowest tile of the whole phase.
__global__ void __launch_bounds__(kThreads, 1)
    ns_flow_kernel(const NsDesc* __restrict__ dg, const NsDesc* __restrict__ du, const NsItem* __restrict__ items,
                   int n_items, unsigned* ctr, NspBufs bufs, const CUtensorMap* __restrict__ maps,
                   const __grid_constant__ NspPhases ph) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = umma::align1024_smem(smem_raw);
  float* stage = reinterpret_cast<float*>(smem + kSlots * kSlot);
  __shared__ uint64_t full_bar[kSlots], empty_bar[kSlots], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint64_t qfull[8], qempty[8];   // item queue: producer -> MMA / epilogue, in claim order
  __shared__ int q[8];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ __align__(16) uint32_t desc_sh[kEpiWarps][32];

  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      umma::mbar_init(&full_bar[i], 1);
      umma::mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      umma::mbar_init(&tfull_bar[i], 1);
      umma::mbar_init(&tempty_bar[i], kEpiWarps);
    }
    for (int i = 0; i < 8; ++i) {
      umma::mbar_init(&qfull[i], 1);
      umma::mbar_init(&qempty[i], kEpiWarps);
    }
    umma::fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc(&tmem_base_sh, 256);
  umma::tc_fence_before();
  __syncthreads();
  umma::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t ring = umma::smem_u32(smem);
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      uint32_t used = 0, epar = 0;
      int cnt = 0;
      for (int kq = 0;; ++kq) {
        // claim the next item (global order) and publish it to the MMA / epilogue warps
        const int slot = kq & 7;
        if (kq >= 8) umma::mbar_wait(&qempty[slot], ((kq >> 3) - 1) & 1);
        const int idx = (int)atomicAdd(ctr, 1u);
        if (idx < n_items) {
          NSP_TRACE(if (ph.ttrace) { ph.ttrace[16 * idx] = gtimer(); ph.ttrace[16 * idx + 3] = blockIdx.x; });
          const NsItem it0 = items[idx];
          if (it0.wait_ctr >= 0)   // data dependency: the previous phase of this matrix is complete
            wait_geq_acquire(ctr + it0.wait_ctr, it0.wait_target, true);
          NSP_TRACE(if (ph.ttrace) ph.ttrace[16 * idx + 1] = gtimer());
        }
        // publish only after the dependency is met: the epilogue prefetches C as soon as it sees the item
        q[slot] = idx < n_items ? idx : -1;
        umma::mbar_arrive(&qfull[slot]);
        if (idx >= n_items) break;
        const NsItem item = items[idx];
        fence_proxy_async_global();   // other CTAs' generic writes before these async-proxy reads
        const int p = item.p;
        const int f = ph.f[p], gram = f & 1, split = (f >> 1) & 1, par = (f >> 2) & 1;
        const NsDesc* D = gram ? dg : du;
        const int w = split ? 2 : 1;
        {
          const NsTile tl{item.desc, item.local};
          const NsDesc d = D[tl.desc];
          const int tw = (!gram && d.epi == 2) ? 64 : 128;   // 64-wide update tiles (launch_ns_persist)
          const int m0 = (tl.local / d.tiles_n) * 128, n0 = (tl.local % d.tiles_n) * tw;
          const int nk = (d.K + 63) / 64, a_mn = d.a_kind & 1, b_mn = d.b_kind & 1, ak = d.a_kind, bk = d.b_kind;
          const bool sym = gram && m0 == n0;   // diagonal Gram tile: B == A, loaded once
          const bool b_half = tw == 64 && b_mn;   // MN-major B: only the first 64-wide box
          NSP_TRACE(unsigned long long w_empty = 0;)
          const uint32_t stage_bytes = sym ? kSlot / 2 : (b_half ? kSlot / 2 + 8192 : kSlot);
          const CUtensorMap* ma = maps + d.map_a + 2 * par;
          const CUtensorMap* mb = maps + d.map_b + 2 * par;
          for (int kb = 0; kb < nk; ++kb) {
            if (w == 2 && cnt % kSlots == kSlots - 1) ++cnt;   // a hi/lo stage takes two adjacent slots
            const int s = cnt % kSlots;
            NSP_TRACE(const unsigned long long te0 = ph.ttrace ? gtimer() : 0;)
            for (int qs = s; qs < s + w; ++qs) {
              if ((used >> qs) & 1u) {
                umma::mbar_wait(&empty_bar[qs], (epar >> qs) & 1u);
                epar ^= 1u << qs;
              }
              used |= 1u << qs;
            }
            NSP_TRACE(if (ph.ttrace) w_empty += gtimer() - te0;)
            const uint32_t sa = ring + s * kSlot;
            umma::mbar_arrive_expect_tx(&full_bar[s], (uint32_t)w * stage_bytes);
            load_operand(sa, ma, &full_bar[s], kb * 64, m0, ak);
            if (b_half) umma::tma_load_2d(sa + 16384, mb, &full_bar[s], n0, kb * 64);
            else if (!sym) load_operand(sa + 16384, mb, &full_bar[s], kb * 64, n0, bk);
            if (split) {
              load_operand(sa + 32768, ma + 1, &full_bar[s], kb * 64, m0, ak);
              if (b_half) umma::tma_load_2d(sa + 49152, mb + 1, &full_bar[s], n0, kb * 64);
              else if (!sym) load_operand(sa + 49152, mb + 1, &full_bar[s], kb * 64, n0, bk);
            }
            cnt += w;
          }
          NSP_TRACE(if (ph.ttrace) ph.ttrace[16 * idx + 15] = w_empty;)
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      uint32_t fpar = 0;
      int cnt = 0, acc = 0;
      for (int kq = 0;; ++kq) {
        const int slot = kq & 7;
        umma::mbar_wait(&qfull[slot], (kq >> 3) & 1);
        const int idx = q[slot];
        if (idx < 0) break;
        const NsItem item = items[idx];
        const int p = item.p;
        const int f = ph.f[p], gram = f & 1, split = (f >> 1) & 1;
        const NsDesc* D = gram ? dg : du;
        const int w = split ? 2 : 1;
        {
          const NsTile tl{item.desc, item.local};
          const NsDesc* dp = D + tl.desc;
          const int nk = (__ldg(&dp->K) + 63) / 64, a_mn = __ldg(&dp->a_kind) & 1, b_mn = __ldg(&dp->b_kind) & 1;
          const int tn = __ldg(&dp->tiles_n);
          const bool sym = gram && (tl.local / tn) == (tl.local % tn);
          const bool w64 = !gram && __ldg(&dp->epi) == 2;
          const uint32_t idesc = (w64 ? umma::idesc_bf16(128, 64) : umma::idesc_bf16(128, 128)) |
                                 ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
          const int buf = acc & 1;
          if (acc >= 2) umma::mbar_wait(&tempty_bar[buf], ((acc >> 1) - 1) & 1);
          umma::tc_fence_after();
          const uint32_t dt = tmem + buf * 128;
          NSP_TRACE(unsigned long long w_full = 0;)
          for (int kb = 0; kb < nk; ++kb) {
            if (w == 2 && cnt % kSlots == kSlots - 1) ++cnt;
            const int s = cnt % kSlots;
            NSP_TRACE(const unsigned long long tw0 = ph.ttrace ? gtimer() : 0;)
            umma::mbar_wait(&full_bar[s], (fpar >> s) & 1u);
            NSP_TRACE(if (ph.ttrace && kb > 0) w_full += gtimer() - tw0;)
            fpar ^= 1u << s;
            umma::tc_fence_after();
            NSP_TRACE(if (ph.ttrace && kb == 0) ph.ttrace[16 * idx + 4] = gtimer());
            const uint32_t ah = ring + s * kSlot, al = ah + 32768;
            const uint32_t bh = sym ? ah : ah + 16384, bl = sym ? al : ah + 49152;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint64_t dah = op_desc(ah, q, a_mn), dbh = op_desc(bh, q, b_mn);
              umma::mma_bf16(dt, dah, dbh, idesc, (kb | q) != 0);
              if (split) {
                umma::mma_bf16(dt, dah, op_desc(bl, q, b_mn), idesc, 1);
                umma::mma_bf16(dt, op_desc(al, q, a_mn), dbh, idesc, 1);
              }
            }
            umma::mma_commit(&empty_bar[s]);
            if (w == 2) umma::mma_commit(&empty_bar[s + 1]);
            cnt += w;
          }
          NSP_TRACE(if (ph.ttrace) ph.ttrace[16 * idx + 14] = w_full;)
          umma::mma_commit(&tfull_bar[buf]);
          ++acc;
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    // 8 warps: warp w reads TMEM lanes 32*(w%4) (rows row0..row0+31) and the
    // 64-column half ch of the accumulator, in two 32-column chunks.  The C
    // tile of both chunks is prefetched into smem with cp.async before the
    // accumulator is ready.  Chunk: tcgen05.ld (thread = row) -> float4 rows
    // into a swizzled 32x32 smem tile -> row pass with 8 lanes per row (float4
    // C from smem, float4 FP32 stores, 8-byte BF16 stores), 4 rows per step.
    // Nothing tile-sized lives in registers (10 warps cap the kernel at 168).
    const int ew = warp - 2, row0 = (warp & 3) * 32, ch = ew >> 2;
    float* Sw = stage + ew * 3 * 1024;
    float* Sc = Sw + 1024;
    const int rsub = lane >> 3, q4 = lane & 7, c4 = q4 * 4;
    int acc = 0;
    for (int kq = 0;; ++kq) {
      const int slot = kq & 7;
      umma::mbar_wait(&qfull[slot], (kq >> 3) & 1);
      const int idx = q[slot];
      if (idx < 0) break;
      const NsItem item = items[idx];
      const int p = item.p;
      const int f = ph.f[p], gram = f & 1, par = (f >> 2) & 1, write_lo = (f >> 3) & 1, write_f = (f >> 4) & 1;
      const NsDesc* D = gram ? dg : du;
      {
        const NsTile tl{item.desc, item.local};
        // this tile's descriptor -> a per-warp smem copy (one word per lane), so the
        // fields cost an LDS, not an L2 round trip, wherever they are used below
        {
          static_assert(sizeof(NsDesc) <= 32 * 4, "NsDesc must fit one word per lane");
          const uint32_t* srcw = reinterpret_cast<const uint32_t*>(D + tl.desc);
          if (lane < (int)(sizeof(NsDesc) / 4)) desc_sh[ew][lane] = __ldg(srcw + lane);
          __syncwarp();
        }
        const NsDesc* dp = reinterpret_cast<const NsDesc*>(desc_sh[ew]);
        const int tiles_n = dp->tiles_n;
        const bool upd = (dp->epi) == 1 || (dp->epi) == 2;   // 3: full (non-symmetric) Gram
        const int cw = (upd && dp->epi == 2) ? 32 : 64;   // columns per warp (64-wide update tiles: one chunk)
        const int nch = cw / 32;
        const int m0 = (tl.local / tiles_n) * 128 + row0, n0 = (tl.local % tiles_n) * (2 * cw) + ch * cw;
        const int64_t f_off = (dp->f_off), ldf = (dp->ldf);
        const int M = (dp->M), N = (dp->N);
        const int buf = acc & 1;
        if (upd) {   // C = X (fp32) rows m0.., cols n0..n0+cw-1 -> Sc[0..nch-1]
          const float* Cm = bufs.X[0] + f_off;
          const bool fv4 = (ldf & 3) == 0;
#pragma unroll 1
          for (int c = 0; c < nch; ++c) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int e = lane + 32 * k, r = e >> 3, q = e & 7;
              const int i = m0 + r, j = n0 + c * 32 + 4 * q;
              float* dst = Sc + c * 1024 + r * 32 + 4 * (q ^ (r & 7));
              const float* src = Cm + (int64_t)i * ldf + j;
              if (fv4 && (j + 3 < N || j >= N)) {
                umma::cp_async16(umma::smem_u32(dst), i < M && j < N ? src : Cm, i < M && j < N);
              } else {   // ragged / unaligned: synchronous scalar path
#pragma unroll
                for (int u = 0; u < 4; ++u) dst[u] = (i < M && j + u < N) ? __ldcg(src + u) : 0.f;
              }
            }
            umma::cp_async_commit();
          }
        }
        NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 6] = gtimer());
        umma::mbar_wait(&tfull_bar[buf], (acc >> 1) & 1);
        umma::tc_fence_after();
        NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 5] = gtimer());
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float v[16];
            umma::tmem_ld16(tmem + buf * 128 + ch * cw + c * 32 + hh * 16 + ((uint32_t)row0 << 16), v);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *reinterpret_cast<float4*>(Sw + lane * 32 + 4 * ((hh * 4 + k) ^ (lane & 7))) =
                  make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          }
          if (c == nch - 1) {   // accumulator drained: hand the TMEM buffer back to the MMA warp
            umma::tc_fence_before();
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(&tempty_bar[buf]);
          }
          NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 8 + 3 * c] = gtimer());
          if (upd) {
            if (c == 0 && nch == 2) umma::cp_async_wait<1>();
            else umma::cp_async_wait<0>();
          }
          __syncwarp();
          NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 9 + 3 * c] = gtimer());
          // per-chunk constants re-derived here (cheap) instead of being held in registers
#if defined(ORTH_NS_EXP2)
          const bool wf = false;
#elif defined(ORTH_NS_EXP)   // timing experiment only (wrong results): fp32 X written by the last phases only
          const bool wf = p >= ph.n - 2;
#else
          const bool wf = upd || write_f;
#endif
          const int ldb16 = upd ? (dp->ldx) : (dp->ldr);
          const int64_t b_off = upd ? (dp->bx_off) : (dp->br_off);
          __nv_bfloat16* oh = (upd ? pick(bufs.xh, par ^ 1) : bufs.rh) + b_off;
          __nv_bfloat16* ol = (upd ? pick(bufs.xl, par ^ 1) : bufs.rl) + b_off;
          float* F = (upd ? bufs.X[0] : bufs.R) + f_off;
          const bool fv4 = (ldf & 3) == 0;
          const float alpha = (dp->alpha), beta = (dp->beta), diag = (dp->diag);
          const float* Scc = Sc + c * 1024;
          // Fast path (warp-uniform): an interior 32 x 32 chunk -- every row < M, every column < N (and so
          // inside the padded BF16 row), 16-byte FP32 rows, no diagonal element -- needs none of the per-element
          // predicates below: straight-line float4 math and incrementally advanced row pointers.  (The generic
          // loop costs ~60 instructions per 4-element group; this one ~20.)
          const int jc0 = n0 + c * 32;
          const bool interior = m0 + 31 < M && jc0 + 31 < N && fv4 &&
                                (diag == 0.f || m0 + 31 < jc0 || jc0 + 31 < m0);
          if (interior) {
            float* fr = F + (int64_t)(m0 + rsub) * ldf + jc0 + c4;
            __nv_bfloat16* hr = oh + (int64_t)(m0 + rsub) * ldb16 + jc0 + c4;
            __nv_bfloat16* lr = ol + (int64_t)(m0 + rsub) * ldb16 + jc0 + c4;
            const int64_t fstep = 4 * ldf, bstep = 4 * (int64_t)ldb16;
#pragma unroll 4
            for (int it = 0; it < 8; ++it) {
              const int rr = 4 * it + rsub;
              const int sw = 4 * (q4 ^ (rr & 7));
              const float4 a = *reinterpret_cast<const float4*>(Sw + rr * 32 + sw);
              float o0, o1, o2, o3;
              if (upd) {
                const float4 cv = *reinterpret_cast<const float4*>(Scc + rr * 32 + sw);
                o0 = fmaf(alpha, a.x, beta * cv.x); o1 = fmaf(alpha, a.y, beta * cv.y);
                o2 = fmaf(alpha, a.z, beta * cv.z); o3 = fmaf(alpha, a.w, beta * cv.w);
              } else {
                o0 = alpha * a.x; o1 = alpha * a.y; o2 = alpha * a.z; o3 = alpha * a.w;
              }
              if (wf) *reinterpret_cast<float4*>(fr) = make_float4(o0, o1, o2, o3);
              const uint32_t h01 = pack_bf16(o0, o1), h23 = pack_bf16(o2, o3);
              *reinterpret_cast<uint2*>(hr) = make_uint2(h01, h23);
              if (write_lo) {
                const uint32_t l01 = pack_bf16(o0 - __uint_as_float(h01 << 16), o1 - __uint_as_float(h01 & 0xFFFF0000u));
                const uint32_t l23 = pack_bf16(o2 - __uint_as_float(h23 << 16), o3 - __uint_as_float(h23 & 0xFFFF0000u));
                *reinterpret_cast<uint2*>(lr) = make_uint2(l01, l23);
              }
              fr += fstep; hr += bstep; lr += bstep;
            }
          } else
#pragma unroll 4
          for (int it = 0; it < 8; ++it) {
            const int rr = 4 * it + rsub;
            const int i = m0 + rr, j = n0 + c * 32 + c4;
            if (i < M) {
              const int sw = 4 * (q4 ^ (rr & 7));
              const float4 a = *reinterpret_cast<const float4*>(Sw + rr * 32 + sw);
              const float4 cv = upd ? *reinterpret_cast<const float4*>(Scc + rr * 32 + sw) : make_float4(0.f, 0.f, 0.f, 0.f);
              float o0 = fmaf(alpha, a.x, beta * cv.x), o1 = fmaf(alpha, a.y, beta * cv.y);
              float o2 = fmaf(alpha, a.z, beta * cv.z), o3 = fmaf(alpha, a.w, beta * cv.w);
              const int dd = i - j;   // diagonal element inside this 4-group
              if (dd == 0) o0 += diag;
              if (dd == 1) o1 += diag;
              if (dd == 2) o2 += diag;
              if (dd == 3) o3 += diag;
              if (j + 3 >= N) {       // ragged right edge: zero beyond N (keeps BF16 padding zero)
                if (j >= N) o0 = 0.f;
                if (j + 1 >= N) o1 = 0.f;
                if (j + 2 >= N) o2 = 0.f;
                o3 = 0.f;
              }
              if (wf && j < N) {
                float* dst = F + (int64_t)i * ldf + j;
                if (fv4 && j + 3 < N) {
                  *reinterpret_cast<float4*>(dst) = make_float4(o0, o1, o2, o3);
                } else {
                  dst[0] = o0;
                  if (j + 1 < N) dst[1] = o1;
                  if (j + 2 < N) dst[2] = o2;
                  if (j + 3 < N) dst[3] = o3;
                }
              }
#ifdef ORTH_NS_EXP2   // timing experiment only (wrong results): no BF16 stores
              if (false) {
#else
              if (j < ldb16) {   // ldb16 % 8 == 0, j % 4 == 0: the 4-group lies inside the padded row
#endif
                const uint32_t h01 = pack_bf16(o0, o1), h23 = pack_bf16(o2, o3);
                const int64_t bo = (int64_t)i * ldb16 + j;
                *reinterpret_cast<uint2*>(oh + bo) = make_uint2(h01, h23);
                if (write_lo) {
                  const uint32_t l01 = pack_bf16(o0 - __uint_as_float(h01 << 16), o1 - __uint_as_float(h01 & 0xFFFF0000u));
                  const uint32_t l23 = pack_bf16(o2 - __uint_as_float(h23 << 16), o3 - __uint_as_float(h23 & 0xFFFF0000u));
                  *reinterpret_cast<uint2*>(ol + bo) = make_uint2(l01, l23);
                }
              }
            }
          }
          NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 10 + 3 * c] = gtimer());
          if (gram && dp->epi != 3 && m0 - row0 < n0 - ch * 64) {
            // upper-triangle Gram tile: also write its mirror R[j][i] = R[i][j] (alpha * acc; no diagonal here)
#pragma unroll 2
            for (int it = 0; it < 8; ++it) {
              const int rt = 4 * it + rsub;                           // column of the chunk = row of the mirror
              const int jg = n0 + c * 32 + rt, ig = m0 + c4;
              if (jg < N && ig < ldb16) {
                float o[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int r = c4 + k;
                  o[k] = ig + k < M ? alpha * Sw[r * 32 + 4 * ((rt >> 2) ^ (r & 7)) + (rt & 3)] : 0.f;
                }
                if (wf) {
                  float* dst = F + (int64_t)jg * ldf + ig;
                  if (fv4 && ig + 3 < M) {
                    *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
                  } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                      if (ig + k < M) dst[k] = o[k];
                  }
                }
                const uint32_t h01 = pack_bf16(o[0], o[1]), h23 = pack_bf16(o[2], o[3]);
                const int64_t bo = (int64_t)jg * ldb16 + ig;
                *reinterpret_cast<uint2*>(oh + bo) = make_uint2(h01, h23);
                if (write_lo) {
                  const uint32_t l01 = pack_bf16(o[0] - __uint_as_float(h01 << 16), o[1] - __uint_as_float(h01 & 0xFFFF0000u));
                  const uint32_t l23 = pack_bf16(o[2] - __uint_as_float(h23 << 16), o[3] - __uint_as_float(h23 & 0xFFFF0000u));
                  *reinterpret_cast<uint2*>(ol + bo) = make_uint2(l01, l23);
                }
              }
            }
          }
          __syncwarp();
        }
        ++acc;
      }
      // ---- item done: publish this tile's writes, bump the matrix's counter, free the queue slot
      NSP_TRACE(if (ph.ttrace && ew == 0 && lane == 0) ph.ttrace[16 * idx + 7] = gtimer());
      fence_proxy_async_global();
      umma::named_bar_sync(1, 32 * kEpiWarps);
      if (ew == 0 && lane == 0) {   // release (cumulative over the barrier) orders all epilogue warps' writes
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + item.done_ctr) : "memory");
        NSP_TRACE(if (ph.ttrace) ph.ttrace[16 * idx + 2] = gtimer());
      }
      if (lane == 0) umma::mbar_arrive(&qempty[slot]);
    }
  }
  umma::tc_fence_before();
  __syncthreads();
  if (warp == 1) umma::tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------- host: partition
struct MatCost {
  int idx, gt, ut, nkg, nku;
};

// estimated microseconds of one NS iteration of a matrix with G CTAs (measured
// B200 per-tile figures: ~0.35 us per 64-deep k-block under full-chip
// streaming, ~3.5 us Gram / ~4 us update epilogue for a full 128x128 tile
// (less for ragged ones), ~1.5 us per group barrier; with double-buffered
// TMEM a CTA's epilogues overlap its next mainloop)
double iter_cost(const MatCost& c, int G) {
  const double ckb = 0.35, ceg = 2.5, ceu = 3.0, cbar = 1.5, cloc = 0.3;
  const double g_tiles = std::ceil((double)c.gt / G), u_tiles = std::ceil((double)c.ut / G);
  const double g_main = c.nkg * ckb, u_main = c.nku * ckb;
  const double gram = g_tiles * std::max(g_main, ceg) + std::min(g_main, ceg);
  const double upd = u_tiles * std::max(u_main, ceu) + std::min(u_main, ceu);
  return gram + upd + (G > 1 ? 2 * cbar : 2 * cloc);
}

}  // namespace

orth_status_t build_ns_persist(Plan& p) {
  if (p.ns_gram.empty()) return ORTH_OK;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (cudaFuncSetAttribute(ns_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem) != cudaSuccess) {
    cudaGetLastError();
    return ORTH_OK;   // stays on the per-phase kernels
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ns_persist_kernel, kThreads, kSmem);
  if (!coop || occ < 1 || sms < 1) return ORTH_OK;
  const int ctas = sms;   // one CTA per SM (smem-limited), all co-resident under the cooperative launch

  std::vector<MatCost> mc;
  for (size_t i = 0; i < p.ns_gram.size(); ++i) {
    const NsDesc& g = p.ns_gram[i];
    const NsDesc& u = p.ns_upd[i];
    // Gram: upper-triangle tiles only (R symmetric; the epilogue mirrors off-diagonal tiles)
    mc.push_back({(int)i, g.tiles_n * (g.tiles_n + 1) / 2, ((u.M + 127) / 128) * u.tiles_n, (g.K + 63) / 64,
                  (u.K + 63) / 64});
  }
  // (a) one group of all matrices over all CTAs
  double ga = 0, ua = 0, gmax = 0, umax = 0;
  for (auto& c : mc) {
    ga += c.gt * std::max(c.nkg * 0.35, 2.5);
    ua += c.ut * std::max(c.nku * 0.35, 3.0);
    gmax = std::max(gmax, c.nkg * 0.35 + 2.5);
    umax = std::max(umax, c.nku * 0.35 + 3.0);
  }
  const double cost_a = std::max(ga / ctas, gmax) + std::max(ua / ctas, umax) + 3.0;
  // (b) malleable-job greedy: every matrix starts as its own group of 1 CTA (or
  // LPT bins when there are more matrices than CTAs); the group with the
  // largest per-iteration cost takes one more CTA while that lowers its cost
  std::vector<int> Gi(mc.size(), 1);
  std::vector<std::vector<int>> bin_mats;
  double cost_b = 0;
  bool ok_b = true;
  if ((int)mc.size() <= ctas) {
    int used = (int)mc.size();
    std::vector<double> cur(mc.size());
    for (size_t i = 0; i < mc.size(); ++i) cur[i] = iter_cost(mc[i], 1);
    while (used < ctas) {
      const int w = (int)(std::max_element(cur.begin(), cur.end()) - cur.begin());
      const double nxt = iter_cost(mc[w], Gi[w] + 1);
      if (nxt >= cur[w] - 1e-9) break;   // the slowest group cannot improve any more
      ++Gi[w];
      cur[w] = nxt;
      ++used;
    }
    cost_b = *std::max_element(cur.begin(), cur.end());
  } else {
    ok_b = false;   // more matrices than CTAs: only the global group
  }
  (void)bin_mats;
  // materialise groups
  struct Grp { std::vector<int> mats; int G; };
  std::vector<Grp> gs;
  const char* force = std::getenv("ORTH_NSP_PARTITION");   // diagnostics: "global" | "groups"
  const bool use_a = !ok_b || cost_a <= cost_b || (force && !std::strcmp(force, "global"));
  if (use_a && !(force && !std::strcmp(force, "groups") && ok_b)) {
    Grp g;
    for (size_t i = 0; i < mc.size(); ++i) g.mats.push_back((int)i);
    g.G = ctas;
    gs.push_back(g);
    p.nsp_est_us = cost_a;
  } else {
    for (size_t i = 0; i < mc.size(); ++i) gs.push_back({{(int)i}, Gi[i]});
    p.nsp_est_us = cost_b;
  }
  if (std::getenv("ORTH_NSP_VERBOSE")) {
    std::printf("ns_persist partition: global %.1f us/iter vs groups %.1f us/iter -> %s, %zu groups\n", cost_a,
                cost_b, gs.size() == 1 ? "global" : "groups", gs.size());
    for (auto& g : gs)
      if (g.mats.size() == 1)
        std::printf("  mat %d (%dx%d): G=%d gram tiles %d (nk %d) upd tiles %d (nk %d) cost %.1f\n", g.mats[0],
                    p.ns_upd[mc[g.mats[0]].idx].M, p.ns_upd[mc[g.mats[0]].idx].N, g.G, mc[g.mats[0]].gt,
                    mc[g.mats[0]].nkg, mc[g.mats[0]].ut, mc[g.mats[0]].nku, iter_cost(mc[g.mats[0]], g.G));
  }
  // per-CTA tile lists: LPT inside each group (tile cost: k-blocks + epilogue;
  // diagonal Gram tiles load one operand, off-diagonal ones also write the mirror)
  auto gram_cost = [&](int m, int l) {
    const int tn = p.ns_gram[mc[m].idx].tiles_n;
    const bool diag = l / tn == l % tn;
    return mc[m].nkg * 0.3 * (diag ? 0.5 : 1.0) + (diag ? 0.8 : 1.6);
  };
  auto upd_cost = [&](int m) { return mc[m].nku * 0.3 + 2.0; };
  // wide update tiles (128 x 256, epi = 4) for this phase-synchronous kernel: a K=16 tcgen05.mma costs
  // the same ~128 cycles for N = 128 and N = 256, and the big sweeps are operand-bandwidth bound, so a
  // 256-wide tile does twice the work per instruction and per A byte.  BF16 mode only (its updates are
  // 1-pass); ORTH_NS_NARROW=1 keeps 128-wide tiles (A/B).
  static const bool narrow = std::getenv("ORTH_NS_NARROW") != nullptr;
  p.ns_upd_wide = p.ns_upd;
  if (!narrow && p.opts.compute == ORTH_BF16)
    for (auto& d : p.ns_upd_wide)
      if (d.N >= 256) {
        d.epi = 4;
        d.tiles_n = (d.N + 255) / 256;
      }
  if (p.d_ns_upd_wide) cudaFree(p.d_ns_upd_wide);
  p.d_ns_upd_wide = nullptr;
  if (cudaMalloc(&p.d_ns_upd_wide, std::max<size_t>(p.ns_upd_wide.size(), 1) * sizeof(NsDesc)) != cudaSuccess ||
      cudaMemcpy(p.d_ns_upd_wide, p.ns_upd_wide.data(), p.ns_upd_wide.size() * sizeof(NsDesc),
                 cudaMemcpyHostToDevice) != cudaSuccess) {
    set_error("NS wide descriptors: %s", cudaGetErrorString(cudaGetLastError()));
    return ORTH_ERR_OUT_OF_MEMORY;
  }
  std::vector<NsTile> tg, tu;
  std::vector<NsGroup> ctas_v;
  int cta = 0;
  for (size_t gi = 0; gi < gs.size(); ++gi) {
    const int G = gs[gi].G;
    struct Item { double c; NsTile t; };
    std::vector<Item> gi_items, ui_items;
    for (int m : gs[gi].mats) {
      const int tn = p.ns_gram[mc[m].idx].tiles_n;
      for (int l = 0; l < tn * tn; ++l)
        if (l / tn <= l % tn) gi_items.push_back({gram_cost(m, l), {mc[m].idx, l}});
      {
        const NsDesc& uw = p.ns_upd_wide[mc[m].idx];
        const bool wide = uw.epi == 4;
        const int utw = ((uw.M + 127) / 128) * uw.tiles_n;
        for (int l = 0; l < utw; ++l) ui_items.push_back({upd_cost(m) * (wide ? 1.7 : 1.0), {mc[m].idx, l}});
      }
    }
    auto lpt = [&](std::vector<Item>& items) {
      std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.c > b.c; });
      std::vector<std::vector<NsTile>> bins(G);
      std::vector<double> load(G, 0.0);
      for (auto& it : items) {
        const int b = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[b] += it.c;
        bins[b].push_back(it.t);
      }
      return bins;
    };
    auto gb = lpt(gi_items), ub = lpt(ui_items);
    for (int c = 0; c < G; ++c) {
      NsGroup e{};
      e.gid = (int32_t)gi;
      e.G = G;
      e.g_begin = (int)tg.size();
      tg.insert(tg.end(), gb[c].begin(), gb[c].end());
      e.g_end = (int)tg.size();
      e.u_begin = (int)tu.size();
      tu.insert(tu.end(), ub[c].begin(), ub[c].end());
      e.u_end = (int)tu.size();
      ctas_v.push_back(e);
    }
    cta += G;
  }
  // a single NsTile array: gram tiles then update tiles (update ranges shifted)
  const int off_u = (int)tg.size();
  for (auto& e : ctas_v) { e.u_begin += off_u; e.u_end += off_u; }
  tg.insert(tg.end(), tu.begin(), tu.end());
  const size_t b_tiles = tg.size() * sizeof(NsTile), b_ctas = ctas_v.size() * sizeof(NsGroup);
  // barrier words: the phase-synchronous kernel's group barriers, or the dataflow kernel's counters
  const size_t n_words = std::max(gs.size(), 1 + 2 * p.ns_gram.size());
  const size_t b_bars = n_words * sizeof(unsigned);
  const size_t total_b = b_tiles + b_ctas + b_bars + 64;
  char* mem = nullptr;
  cudaError_t e = cudaMalloc(&mem, total_b);
  if (e != cudaSuccess) {
    set_error("NS persistent tables: %s", cudaGetErrorString(e));
    return ORTH_ERR_OUT_OF_MEMORY;
  }
  p.nsp_mem = mem;
  p.nsp_tiles = reinterpret_cast<NsTile*>(mem);
  p.nsp_groups = reinterpret_cast<NsGroup*>(mem + b_tiles);
  p.nsp_bars = reinterpret_cast<unsigned*>(mem + ((b_tiles + b_ctas + 15) & ~size_t(15)));
  e = cudaMemcpy(p.nsp_tiles, tg.data(), b_tiles, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p.nsp_groups, ctas_v.data(), b_ctas, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(p.nsp_bars, 0, b_bars);
  if (e != cudaSuccess) {
    set_error("NS persistent tables upload: %s", cudaGetErrorString(e));
    return ORTH_ERR_CUDA;
  }
  p.nsp_groups_n = (int)gs.size();
  p.nsp_zero_n = (int)n_words;
  p.nsp_ctas = cta;
  return ORTH_OK;
}

// dataflow items for a phase list: phase-major; inside a phase the matrices with
// the longest tiles first (dynamic claiming then balances the tail)
static int build_flow_items(Plan& p, const uint8_t* flags, int nphases) {
  if (p.nsf_nphases == nphases && p.nsf_flags.size() == (size_t)nphases &&
      std::memcmp(p.nsf_flags.data(), flags, (size_t)nphases) == 0)
    return 0;
  const int nm = (int)p.ns_gram.size();
  // 64-wide update tiles: half the epilogue (the latency-critical part of a phase; measured ~4 us per
  // 128x128 tile), twice the CTAs per update phase; ORTH_NS_W128=1 keeps 128-wide tiles (A/B)
  static const bool w128 = std::getenv("ORTH_NS_W128") != nullptr;
  if (p.ns_upd64.empty()) {
    p.ns_upd64 = p.ns_upd;
    // only for the large matrices (>= 32 update tiles of 128 x 128: the long chains); for the many small
    // ones the extra items cost throughput (cfg3: 0.51 -> 0.64 ms with every matrix split)
    static const int min_tiles = std::getenv("ORTH_NS_W64_MIN") ? std::atoi(std::getenv("ORTH_NS_W64_MIN")) : 32;
    if (!w128)
      for (auto& d : p.ns_upd64)
        if (((d.M + 127) / 128) * d.tiles_n >= min_tiles) {
          d.epi = 2;
          d.tiles_n = (d.N + 63) / 64;
        }
    if (cudaMalloc(&p.d_ns_upd64, std::max<size_t>(p.ns_upd64.size(), 1) * sizeof(NsDesc)) != cudaSuccess ||
        cudaMemcpy(p.d_ns_upd64, p.ns_upd64.data(), p.ns_upd64.size() * sizeof(NsDesc), cudaMemcpyHostToDevice) !=
            cudaSuccess)
      return (int)cudaGetLastError();
  }
  // Full (non-symmetric) Gram for the widest matrices: every tile computed, no mirror pass in the
  // epilogue (the mirror made a Gram tile's epilogue ~4.8 us on the critical 24-phase chain); +tn(tn-1)/2
  // tiles of MMA work for those few matrices only.  ORTH_NS_SYMGRAM=1 keeps the symmetric Gram (A/B).
  static const bool symgram = std::getenv("ORTH_NS_SYMGRAM") != nullptr;
  if (p.ns_gram_flow.empty()) {
    p.ns_gram_flow = p.ns_gram;
    static const int nmin = std::getenv("ORTH_NS_FULLGRAM_MIN") ? std::atoi(std::getenv("ORTH_NS_FULLGRAM_MIN")) : 512;
    if (!symgram)
      for (auto& d : p.ns_gram_flow)
        if (d.N >= nmin) d.epi = 3;
    if (cudaMalloc(&p.d_ns_gram_flow, std::max<size_t>(p.ns_gram_flow.size(), 1) * sizeof(NsDesc)) != cudaSuccess ||
        cudaMemcpy(p.d_ns_gram_flow, p.ns_gram_flow.data(), p.ns_gram_flow.size() * sizeof(NsDesc),
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return (int)cudaGetLastError();
  }
  std::vector<int> GT(nm), UT(nm), order(nm);
  for (int i = 0; i < nm; ++i) {
    const int tn = p.ns_gram[i].tiles_n;
    GT[i] = p.ns_gram_flow[i].epi == 3 ? tn * tn : tn * (tn + 1) / 2;
    UT[i] = ((p.ns_upd64[i].M + 127) / 128) * p.ns_upd64[i].tiles_n;
    order[i] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return p.ns_gram[a].K > p.ns_gram[b].K; });
  std::vector<NsItem> items;
  for (int ph = 0; ph < nphases; ++ph) {
    const bool gram = flags[ph] & 1;
    const int t = ph / 2;   // iteration (the residual Gram is phase 2T: t = T)
    for (int i : order) {
      const int tn = gram ? p.ns_gram[i].tiles_n : p.ns_upd64[i].tiles_n;
      const int ntile = gram ? tn * tn : UT[i];
      for (int l = 0; l < ntile; ++l) {
        if (gram && p.ns_gram_flow[i].epi != 3 && l / tn > l % tn) continue;   // upper-triangle Gram tiles only
        NsItem it{};
        it.p = ph; it.desc = i; it.local = l;
        if (gram) {   // Gram(t) reads X_t: all update tiles of iteration t - 1 done
          it.wait_ctr = t > 0 ? 2 + 2 * i : -1;
          it.wait_target = (uint32_t)(t * UT[i]);
          it.done_ctr = 1 + 2 * i;
        } else {      // update(t) reads R_t: all Gram tiles of iteration t done
          it.wait_ctr = 1 + 2 * i;
          it.wait_target = (uint32_t)((t + 1) * GT[i]);
          it.done_ctr = 2 + 2 * i;
        }
        items.push_back(it);
      }
    }
  }
  if (p.nsf_items) cudaFree(p.nsf_items);
  p.nsf_items = nullptr;
  cudaError_t e = cudaMalloc(&p.nsf_items, std::max<size_t>(items.size(), 1) * sizeof(NsItem));
  if (e == cudaSuccess && !items.empty())
    e = cudaMemcpy(p.nsf_items, items.data(), items.size() * sizeof(NsItem), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return (int)e;
  p.nsf_n_items = (int)items.size();
  p.nsf_nphases = nphases;
  p.nsf_flags.assign(flags, flags + nphases);
  return 0;
}

// diagnostics (ORTH_NSP_TRACE builds, ORTH_NS_TRACE=1): per item {claimed, dependency met, done, cta}
// -> per phase of the three largest matrices: span and where the time went; CTA busy fraction
static void flow_trace_report(const Plan& p, const uint8_t* flags, int nphases, const unsigned long long* ttrace,
                              cudaStream_t stream) {
  cudaStreamSynchronize(stream);
  const int n = p.nsf_n_items;
  std::vector<unsigned long long> r((size_t)16 * n);
  cudaMemcpy(r.data(), ttrace, r.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<NsItem> items(n);
  cudaMemcpy(items.data(), p.nsf_items, (size_t)n * sizeof(NsItem), cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, t1 = 0;
  double busy = 0, waiting = 0;
  for (int i = 0; i < n; ++i) {
    t0 = std::min(t0, r[16 * i]);
    t1 = std::max(t1, r[16 * i + 2]);
    busy += (double)(r[16 * i + 2] - r[16 * i + 1]);
    waiting += (double)(r[16 * i + 1] - r[16 * i]);
  }
  std::printf("ns_flow: %d items, %d CTAs, span %.1f us; sum(item dep-met->done) %.1f us = %.0f%% of CTA-time, "
              "sum(claim->dep-met) %.1f us\n", n, p.nsp_ctas, (t1 - t0) * 1e-3, busy * 1e-3,
              100.0 * busy / ((double)(t1 - t0) * p.nsp_ctas), waiting * 1e-3);
  std::vector<int> order((size_t)p.ns_gram.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return (double)p.ns_upd[a].M * p.ns_upd[a].N * p.ns_gram[a].N > (double)p.ns_upd[b].M * p.ns_upd[b].N * p.ns_gram[b].N;
  });
  {   // per matrix: when its last phase finished (sorted by size)
    std::map<std::pair<int, int>, std::pair<double, int>> fin;   // (M, N) -> (max done, count)
    std::vector<unsigned long long> last(order.size(), 0);
    for (int i = 0; i < n; ++i) last[items[i].desc] = std::max(last[items[i].desc], r[16 * i + 2]);
    for (size_t m = 0; m < order.size(); ++m) {
      auto& f = fin[{p.ns_upd[m].M, p.ns_upd[m].N}];
      f.first = std::max(f.first, (last[m] - t0) * 1e-3);
      f.second++;
    }
    for (auto& kv : fin)
      std::printf(" matrices %4dx%-4d x%-3d done by %.1f us\n", kv.first.first, kv.first.second, kv.second.second,
                  kv.second.first);
  }
  for (int mi = 0; mi < 3 && mi < (int)order.size(); ++mi) {
    const int m = order[mi];
    std::printf(" matrix %d (upd %dx%d, gram N=%d K=%d):\n", m, p.ns_upd[m].M, p.ns_upd[m].N, p.ns_gram[m].N,
                p.ns_gram[m].K);
    for (int ph = 0; ph < nphases; ++ph) {
      unsigned long long dmin = ~0ull, dmax = 0, emax = 0, cmin = ~0ull;
      double dur = 0, d_load = 0, d_mma = 0, d_epiq = 0, d_epi = 0, d_pub = 0, sub[6] = {0, 0, 0, 0, 0, 0};
      double d_fw = 0, d_ew = 0;
      int cnt = 0;
      for (int i = 0; i < n; ++i)
        if (items[i].p == ph && items[i].desc == m) {
          const unsigned long long* q = &r[16 * i];
          cmin = std::min(cmin, q[0]);
          dmin = std::min(dmin, q[1]);
          dmax = std::max(dmax, q[1]);
          emax = std::max(emax, q[2]);
          dur += (double)(q[2] - q[1]);
          d_load += (double)q[4] - (double)q[1];   // dependency met -> first k-block in smem
          d_mma += (double)q[5] - (double)q[4];    // -> accumulator complete
          d_epiq += (double)q[6] - (double)q[1];   // dependency met -> epilogue reaches this item
          d_epi += (double)q[7] - (double)q[5];    // accumulator -> last store issued (warp 0)
          d_pub += (double)q[2] - (double)q[7];    // -> fences, barrier, counter bump
          for (int z = 0; z < 6; ++z) sub[z] += (double)q[8 + z] - (double)(z == 0 ? q[5] : q[7 + z]);
          d_fw += (double)q[14];
          d_ew += (double)q[15];
          ++cnt;
        }
      if (!cnt) continue;
      std::printf("  ph%2d %s x%d%s: claimed %.1f dep %.1f..%.1f done %.1f us (mean tile %.2f us: load %.2f mma %.2f "
                  "epi %.2f pub %.2f; epi free after %.2f)\n", ph,
                  (flags[ph] & 1) ? "gram" : "upd ", cnt, (flags[ph] & 2) ? " 3p" : "   ", (cmin - t0) * 1e-3,
                  (dmin - t0) * 1e-3, (dmax - t0) * 1e-3, (emax - t0) * 1e-3, dur / cnt * 1e-3, d_load / cnt * 1e-3,
                  d_mma / cnt * 1e-3, d_epi / cnt * 1e-3, d_pub / cnt * 1e-3, d_epiq / cnt * 1e-3);
      std::printf("        MMA thread waiting for full stages %.2f us, producer waiting for empty stages %.2f us\n",
                  d_fw / cnt * 1e-3, d_ew / cnt * 1e-3);
      std::printf("        epi chunks: drain %.2f cwait %.2f rows %.2f | drain %.2f cwait %.2f rows %.2f us\n",
                  sub[0] / cnt * 1e-3, sub[1] / cnt * 1e-3, sub[2] / cnt * 1e-3, sub[3] / cnt * 1e-3, sub[4] / cnt * 1e-3,
                  sub[5] / cnt * 1e-3);
    }
  }
}

int launch_ns_persist(Plan& p, float* const bufs[BUF_COUNT], const uint8_t* flags, int nphases, void* stream) {
  NspBufs b;
  b.X[0] = bufs[BUF_X];
  b.X[1] = bufs[BUF_Y];
  b.R = bufs[BUF_G];
  auto bx = reinterpret_cast<__nv_bfloat16*>(p.d_bx);
  const int64_t nx = p.bx_numel > 64 ? p.bx_numel : 64;
  for (int k = 0; k < 2; ++k) {
    b.xh[k] = bx + (0 + k) * nx;
    b.xl[k] = bx + (2 + k) * nx;
  }
  auto br = reinterpret_cast<__nv_bfloat16*>(p.d_br);
  b.rh = br;
  b.rl = br + (p.br_numel > 64 ? p.br_numel : 64);
  NspPhases ph;
  std::memset(&ph, 0, sizeof(ph));
  ph.n = nphases;
  std::memcpy(ph.f, flags, (size_t)nphases);
#ifdef ORTH_NSP_TRACE
  static const bool tracing = std::getenv("ORTH_NS_TRACE") != nullptr;
#else
  constexpr bool tracing = false;
#endif
  static unsigned long long* trace = nullptr;
  static unsigned long long* ttrace = nullptr;
  if (tracing) {
    if (!trace) cudaMalloc(&trace, (size_t)p.nsp_ctas * (4 * kNspMaxPhases + 1) * 8);
    if (!ttrace) cudaMalloc(&ttrace, (1 + 8 * 65536) * 8);
    cudaMemsetAsync(ttrace, 0, 8, (cudaStream_t)stream);
    ph.trace = trace;
    ph.ttrace = ttrace;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.nsp_ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  p.launches++;
  // dataflow for latency-bound batches (cfg2 / cfg3: a few hundred tiles per phase; measured 0.63 -> 0.57 ms
  // on cfg3), phase-synchronous for big uniform sweeps (cfg5 n = 2048: 34.3 ms sync vs 40.5 ms dataflow)
  static const char* mode_env = std::getenv("ORTH_NS_MODE");   // "flow" | "sync" (A/B)
  // decided on the whole network's tile count, not this rank's share: the two schedules differ in the
  // Gram of N >= 512 matrices (full tiles vs symmetric + mirror, whose 3-pass cross terms accumulate in
  // the opposite order), so a per-rank choice would make sharded results differ in the last bits
  const bool small = p.ns_upd_tiles_all <= 4 * (int64_t)p.nsp_ctas;
  const bool flow = mode_env ? std::strcmp(mode_env, "sync") != 0 : small;
  if (flow) {
    if (int e = build_flow_items(p, flags, nphases)) return e;
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(ns_flow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
      attr_set = true;
    }
    const int ef = (int)cudaLaunchKernelEx(&cfg, ns_flow_kernel, (const NsDesc*)p.d_ns_gram_flow, (const NsDesc*)p.d_ns_upd64,
                                           (const NsItem*)p.nsf_items, p.nsf_n_items, p.nsp_bars, b,
                                           reinterpret_cast<const CUtensorMap*>(p.d_ns_maps), ph);
    if (tracing && ef == 0) flow_trace_report(p, flags, nphases, ttrace, (cudaStream_t)stream);
    return ef;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, ns_persist_kernel, (const NsDesc*)p.d_ns_gram,
                                           (const NsDesc*)p.d_ns_upd_wide, (const NsTile*)p.nsp_tiles,
                                           (const NsGroup*)p.nsp_groups, p.nsp_bars,
                                           b, reinterpret_cast<const CUtensorMap*>(p.d_ns_maps), ph);
  if (tracing && e == cudaSuccess) {   // diagnostics only: serialises the stream
    cudaStreamSynchronize((cudaStream_t)stream);
    {
      unsigned long long nrec = 0;
      cudaMemcpy(&nrec, ttrace, 8, cudaMemcpyDeviceToHost);
      nrec = std::min<unsigned long long>(nrec, 65536);
      std::vector<unsigned long long> r(8 * nrec);
      cudaMemcpy(r.data(), ttrace + 1, r.size() * 8, cudaMemcpyDeviceToHost);
      // per (phase type, M, N, K): count, mean wait-for-accumulator, mean epilogue (warp 0 of the epilogue only)
      struct Acc { int n = 0; double wait = 0, epi = 0, epimax = 0, c[4] = {0, 0, 0, 0}; };
      std::map<std::tuple<int, int, int, int, int>, Acc> agg;
      for (unsigned long long k = 0; k < nrec; ++k) {
        const unsigned long long* q = &r[8 * k];
        const int ph_ = (int)((q[0] >> 40) & 0xFF), ew = (int)((q[0] >> 36) & 0xF), desc = (int)((q[0] >> 16) & 0xFFFFF);
        const int local = (int)(q[0] & 0xFFFF);
        if (ew != 0 || ph_ > 3) continue;
        const bool gram = flags[ph_] & 1;
        const NsDesc& d = gram ? p.ns_gram[desc] : p.ns_upd[desc];
        const int diag = gram && (local / d.tiles_n == local % d.tiles_n);
        Acc& a = agg[std::make_tuple(ph_, d.M, d.N, d.K, diag)];
        a.n++;
        a.wait += (q[2] - q[1]) * 1e-3;
        a.epi += (q[3] - q[2]) * 1e-3;
        a.epimax = std::max(a.epimax, (q[3] - q[2]) * 1e-3);
        for (int z = 0; z < 4; ++z) a.c[z] += (double)q[4 + z];
      }
      for (auto& kv : agg)
        std::printf("  tile ph%d M=%4d N=%4d K=%4d diag=%d: n=%3d wait %.2f epi %.2f (max %.2f) us | cyc ld0 %.0f row0 %.0f mir0 %.0f ch1 %.0f\n",
                    std::get<0>(kv.first), std::get<1>(kv.first), std::get<2>(kv.first), std::get<3>(kv.first),
                    std::get<4>(kv.first), kv.second.n, kv.second.wait / kv.second.n, kv.second.epi / kv.second.n,
                    kv.second.epimax, kv.second.c[0] / kv.second.n, kv.second.c[1] / kv.second.n,
                    kv.second.c[2] / kv.second.n, kv.second.c[3] / kv.second.n);
    }
    const int W = 4 * nphases + 1;
    std::vector<unsigned long long> h((size_t)p.nsp_ctas * W);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < p.nsp_ctas; ++c) {
      t0 = std::min(t0, h[(size_t)c * W]);
      t1 = std::max(t1, h[(size_t)c * W + W - 1]);
    }
    std::printf("ns_persist: %d CTAs, %d groups, %d phases, span %.1f us (model %.1f us/iter)\n", p.nsp_ctas,
                p.nsp_groups_n, nphases, (t1 - t0) * 1e-3, p.nsp_est_us);
    // per phase, averaged over CTAs: producer start -> epi first full -> epi done -> after sync (relative to previous sync)
    for (int q = 0; q < nphases && q < 6; ++q) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, m3 = 0, m1 = 0, m2 = 0;
      for (int c = 0; c < p.nsp_ctas; ++c) {
        const unsigned long long* r = &h[(size_t)c * W];
        const double prev = (double)(q == 0 ? r[0] : r[1 + 4 * (q - 1) + 3]);
        a0 += r[1 + 4 * q] - prev; a1 += r[2 + 4 * q] - prev; a2 += r[3 + 4 * q] - prev; a3 += r[4 + 4 * q] - prev;
        m3 = std::max(m3, (double)(r[4 + 4 * q] - prev));
        m1 = std::max(m1, (double)(r[2 + 4 * q] - prev));
        m2 = std::max(m2, (double)(r[3 + 4 * q] - prev));
      }
      const double n = p.nsp_ctas * 1e3;
      std::printf("  phase %d: prod_start %.2f first_full %.2f (max %.2f) epi_done %.2f (max %.2f) synced %.2f (max %.2f) us\n",
                  q, a0 / n, a1 / n, m1 * 1e-3, a2 / n, m2 * 1e-3, a3 / n, m3 * 1e-3);
    }
  }
  return (int)e;
}

}  // namespace orth
