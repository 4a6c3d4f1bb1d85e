// Host planner of the C ABI (include/orth.h): validation, unit derivation
// (SURVEY §8(a) a1), packed layouts, construction sharding, GEMM/tile
// descriptors of every phase, one-shot workspace allocation, queries.
//
// The derivation follows P:323-338 (AOC = RKO (*) K_BCOP, k >= s) with the
// readings R5-R8 of DESIGN.md: s == 1 -> BCOP at width max(ci, co), k' = k;
// k == s > 1 -> RKO only; k > s > 1 -> k' = k - s + 1,
// c_mid = max(ci, floor(co / s^2)), BCOP at width c_mid.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>

#include "orth_internal.h"

namespace orth {

static thread_local char g_err[512] = "";
thread_local int g_conv_variant = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }

static orth_status_t validate_opts(const orth_opts_t& o) {
  if (o.ns_iters < 1) { set_error("ns_iters must be >= 1 (got %d)", o.ns_iters); return ORTH_ERR_INVALID_ARGUMENT; }
  if (!(o.beta > 0.0f && o.beta <= 0.5f)) { set_error("beta must be in (0, 1/2] (P:311), got %g", o.beta); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.prescale != ORTH_PRESCALE_POWER && o.prescale != ORTH_PRESCALE_FROBENIUS) { set_error("bad prescale %d", o.prescale); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.prescale == ORTH_PRESCALE_POWER && o.power_iters < 1) { set_error("power_iters must be >= 1"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.compute != ORTH_F32 && o.compute != ORTH_BF16 && o.compute != ORTH_BF16X3) { set_error("bad compute mode %d", o.compute); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.polish_iters < 0 || o.polish_iters > o.ns_iters) { set_error("polish_iters must be in [0, ns_iters]"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) { set_error("bad rank/world %d/%d", o.rank, o.world); return ORTH_ERR_INVALID_ARGUMENT; }
  if (o.max_batch < 0) { set_error("max_batch must be >= 0"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (!(o.ns_tol == o.ns_tol)) { set_error("ns_tol is NaN"); return ORTH_ERR_INVALID_ARGUMENT; }
  return ORTH_OK;
}

static orth_status_t validate_layer(const orth_layer_desc_t& L, int idx) {
  if (L.kind < 0 || L.kind > 5) { set_error("layer %d: bad kind %d", idx, L.kind); return ORTH_ERR_INVALID_ARGUMENT; }
  if (L.c_in < 1 || L.c_out < 1 || L.k_h < 1 || L.k_w < 1 || L.stride_h < 1 || L.stride_w < 1 || L.dil_h < 1 ||
      L.dil_w < 1 || L.groups < 1) {
    set_error("layer %d: every dimension must be >= 1 (S:31)", idx);
    return ORTH_ERR_INVALID_ARGUMENT;
  }
  if (L.c_in % L.groups || L.c_out % L.groups) {
    set_error("layer %d: groups %d must divide c_in %d and c_out %d (S:38)", idx, L.groups, L.c_in, L.c_out);
    return ORTH_ERR_INVALID_ARGUMENT;
  }
  if (L.grid_h < 0 || L.grid_w < 0) { set_error("layer %d: grid_h/grid_w must be >= 0", idx); return ORTH_ERR_INVALID_ARGUMENT; }
  if (L.padding_mode != ORTH_PAD_ZEROS && L.padding_mode != ORTH_PAD_CIRCULAR) {
    set_error("layer %d: bad padding_mode %d", idx, L.padding_mode);
    return ORTH_ERR_INVALID_ARGUMENT;
  }
  const bool all_def = L.pad_t == -1 && L.pad_b == -1 && L.pad_l == -1 && L.pad_r == -1;
  const bool all_set = L.pad_t >= 0 && L.pad_b >= 0 && L.pad_l >= 0 && L.pad_r >= 0;
  if (!all_def && !all_set) { set_error("layer %d: pads must be all -1 (same rule) or all >= 0", idx); return ORTH_ERR_INVALID_ARGUMENT; }
  if (L.kind == ORTH_DENSE) {
    if (L.k_h != 1 || L.k_w != 1 || L.stride_h != 1 || L.stride_w != 1 || L.dil_h != 1 || L.dil_w != 1 || L.groups != 1) {
      set_error("layer %d: dense layers need k = s = d = g = 1", idx);
      return ORTH_ERR_INVALID_ARGUMENT;
    }
    return ORTH_OK;
  }
  if (L.k_h != L.k_w || L.stride_h != L.stride_w || L.dil_h != L.dil_w) {
    set_error("layer %d: only square kernel/stride/dilation are supported", idx);
    return ORTH_ERR_UNSUPPORTED_CONFIG;
  }
  if (L.kind == ORTH_SLL || L.kind == ORTH_SLL_BLOCK) {   // f4: plain, circular, g = d = 1
    if (L.groups != 1 || L.dil_h != 1) { set_error("layer %d: SLL layers / blocks need g = d = 1", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    if (L.padding_mode != ORTH_PAD_CIRCULAR) { set_error("layer %d: the SLL block is exact for circular padding only (R30)", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    if (L.pad_t != -1) { set_error("layer %d: SLL layers / blocks use the 'same' pads (pads must be -1)", idx); return ORTH_ERR_INVALID_ARGUMENT; }
    if (L.kind == ORTH_SLL && L.stride_h != 1) { set_error("layer %d: an SLL kernel has stride 1", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    return ORTH_OK;
  }
  if (L.kind == ORTH_SOC) {   // f3: square channel map, odd kernel, stride 1 (R27)
    const int n = L.soc_terms == 0 ? 6 : L.soc_terms;
    if (L.c_in != L.c_out) { set_error("layer %d: SOC needs c_in == c_out (channel change: R27, not built)", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    if (L.k_h % 2 == 0) { set_error("layer %d: SOC needs an odd kernel (centred padding keeps skew-adjointness)", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    if (L.stride_h != 1) { set_error("layer %d: SOC stride > 1 (RKO composition, R27) is not built", idx); return ORTH_ERR_UNSUPPORTED_CONFIG; }
    if (n < 1 || n > 16 || n * (L.k_h - 1) + 1 > 63) { set_error("layer %d: soc_terms %d out of range [1, 16] (k_eff <= 63)", idx, n); return ORTH_ERR_INVALID_ARGUMENT; }
    if (L.pad_t != -1) { set_error("layer %d: SOC uses the centred 'same' padding (pads must be -1)", idx); return ORTH_ERR_INVALID_ARGUMENT; }
    return ORTH_OK;
  }
  if (L.k_h < L.stride_h) {
    set_error("layer %d: k = %d < s = %d has no orthogonal AOC kernel (P:330)", idx, L.k_h, L.stride_h);
    return ORTH_ERR_UNSUPPORTED_CONFIG;
  }
  if (gcd_i(L.stride_h, L.dil_h) != 1) {
    set_error("layer %d: gcd(s=%d, d=%d) != 1 loses orthogonality (reading R10)", idx, L.stride_h, L.dil_h);
    return ORTH_ERR_UNSUPPORTED_CONFIG;
  }
  return ORTH_OK;
}

static orth_status_t derive(Plan& P, const orth_layer_desc_t* layers, int n_layers) {
  P.layers.clear();
  P.mats.clear();
  const int T = P.opts.ns_iters;
  for (int l = 0; l < n_layers; ++l) {
    LayerInfo L{};
    L.desc = layers[l];
    const auto& D = layers[l];
    L.k = D.k_h; L.s = D.stride_h; L.d = D.dil_h; L.g = D.groups;
    if (D.kind == ORTH_CONV_TRANSPOSE2D) { L.ci_f = D.c_out; L.co_f = D.c_in; }  // R13
    else { L.ci_f = D.c_in; L.co_f = D.c_out; }
    L.ci = L.ci_f / L.g; L.co = L.co_f / L.g;
    if (D.pad_t == -1) {
      const int e = L.d * (L.k - 1);
      L.pt = L.pl = e / 2; L.pb = L.pr = e - e / 2;     // R11
    } else { L.pt = D.pad_t; L.pb = D.pad_b; L.pl = D.pad_l; L.pr = D.pad_r; }
    std::vector<std::pair<int, std::pair<int64_t, int64_t>>> ms;  // role, (m, n)
    if (D.kind == ORTH_SLL) {
      L.cons = CONS_SLL;
      ms.push_back({ROLE_K, {L.co, (int64_t)L.ci * L.k * L.k}});
    } else if (D.kind == ORTH_SLL_BLOCK) {   // merged kernels of three earlier layers (validated)
      L.cons = CONS_SLL_BLOCK;
      L.blk_id = 0;
      for (const auto& Q : P.layers) L.blk_id += Q.cons == CONS_SLL_BLOCK ? 1 : 0;
      L.blk_pre = D.blk_pre; L.blk_sll = D.blk_sll; L.blk_post = D.blk_post;
      const LayerInfo &Pre = P.layers[D.blk_pre], &S = P.layers[D.blk_sll], &Po = P.layers[D.blk_post];
      L.blk_cs = S.co;
      const int kA = Po.k + Pre.k - 1, kB = Po.k + S.k - 1;
      L.kC = S.k + Pre.k - 1;
      L.pC = S.pt + Pre.pt;
      const int pA = Po.pt + Pre.pt, pB = Po.pt + (S.k - 1 - S.pt);
      L.pM = std::max(pA, pB);
      L.kM = std::max(L.pM - pA + kA, L.pM - pB + kB);
      L.k = L.kM;
      L.pt = L.pl = L.pM; L.pb = L.pr = L.kM - 1 - L.pM;
    } else if (D.kind == ORTH_SOC) {
      L.cons = CONS_SOC;
      L.k_free = D.k_h;
      L.soc_terms = D.soc_terms == 0 ? 6 : D.soc_terms;
      L.k = L.soc_terms * (L.k_free - 1) + 1;   // the applied kernel: k_eff
      const int e = L.d * (L.k - 1);
      L.pt = L.pl = e / 2; L.pb = L.pr = e - e / 2;
      ms.push_back({ROLE_K, {L.co, (int64_t)L.ci * L.k_free * L.k_free}});
    } else if (D.kind == ORTH_DENSE) {
      L.cons = CONS_DENSE;
      ms.push_back({ROLE_W, {L.co, L.ci}});
    } else if (L.s == 1) {
      L.cons = CONS_BCOP; L.kp = L.k; L.c_b = std::max(L.ci, L.co);
    } else if (L.k == L.s) {
      L.cons = CONS_RKO; L.c_mid = L.ci;
    } else {
      L.cons = CONS_AOC; L.kp = L.k - L.s + 1;
      L.c_mid = std::max(L.ci, L.co / (L.s * L.s)); L.c_b = L.c_mid;
    }
    if (L.cons == CONS_BCOP || L.cons == CONS_AOC) {
      ms.push_back({ROLE_Q, {L.c_b, L.c_b}});
      for (int j = 0; j < 2 * (L.kp - 1); ++j) ms.push_back({ROLE_U, {L.c_b, L.c_b / 2}});
    }
    if (L.cons == CONS_RKO || L.cons == CONS_AOC) ms.push_back({ROLE_R, {L.co, (int64_t)L.c_mid * L.s * L.s}});
    L.first_mat = (int)P.mats.size();
    L.mats_per_group = (int)ms.size();
    L.kernel_numel = (D.kind == ORTH_DENSE) ? (int64_t)L.co * L.ci : (int64_t)L.co_f * L.ci * L.k * L.k;
    if (D.kind == ORTH_SLL_BLOCK) {   // [C (c_s, c, kC, kC) | M (c_out, c + c_s, kM, kM)], M 128 B aligned
      L.m_off = pad_up((int64_t)L.blk_cs * L.ci * L.kC * L.kC, 64);
      L.kernel_numel = L.m_off + (int64_t)L.co * (L.ci + L.blk_cs) * L.kM * L.kM;
    }
    double fl = 0.0;
    for (int gi = 0; gi < L.g; ++gi)
      for (auto& e : ms) {
        MatInfo M{};
        M.layer = l; M.group = gi; M.role = e.first; M.m = e.second.first; M.n = e.second.second;
        P.mats.push_back(M);
        const double a = (double)std::max(M.m, M.n), b = (double)std::min(M.m, M.n);
        if (M.role != ROLE_K) fl += 4.0 * a * b * b * T;
      }
    L.ns_flops = fl;
    // composition flops (structured chain, a4/a5; used only for load balance)
    double cf = 0.0;
    if (L.kp > 1) {
      const double c = L.c_b;
      cf += 2.0 * (L.kp - 1) * 2.0 * c * c * (c / 2);  // projectors
      for (int j = 1; j < L.kp; ++j) cf += 2.0 * c * c * c * ((j + 1) * j + (j + 1) * (j + 1));
    }
    if (L.cons == CONS_AOC) cf += 2.0 * L.co * L.c_mid * L.ci * L.s * L.s * L.kp * L.kp;
    if (L.cons == CONS_SOC) {   // S^(*)j = S^(*)(j-1) (*) S: (kj-1 taps) x k^2 products of c x c, j = 2..max(n, 2)
      const double c = L.co;
      for (int j = 2; j <= std::max(L.soc_terms, 2); ++j) {
        const double kj1 = (j - 1) * (L.k_free - 1) + 1;
        cf += kj1 * kj1 * L.k_free * L.k_free * 2.0 * c * c * c;
      }
    }
    L.comp_flops = cf * L.g;
    P.layers.push_back(L);
  }
  return ORTH_OK;
}

// LPT greedy by cost over (layer, group) units (R22): the largest
// unit (NS + composition flops of one group) to the least-loaded rank; ties
// keep the (layer, group) order, so every rank derives the same assignment.
static void assign_owners(Plan& P) {
  const int R = P.opts.world;
  P.units.clear();
  for (int l = 0; l < (int)P.layers.size(); ++l) {
    LayerInfo& L = P.layers[l];
    L.first_unit = (int)P.units.size();
    for (int g = 0; g < L.g; ++g) {
      UnitInfo u{};
      u.layer = l; u.group = g; u.owner = 0;
      u.numel = L.kernel_numel / L.g;
      P.units.push_back(u);
    }
  }
  std::vector<int> order(P.units.size());
  std::iota(order.begin(), order.end(), 0);
  auto cost = [&](int u) {
    const LayerInfo& L = P.layers[P.units[u].layer];
    return (L.ns_flops + L.comp_flops) / L.g;
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
  std::vector<double> load(R, 0.0);
  for (int u : order) {
    int best = 0;
    for (int r = 1; r < R; ++r) if (load[r] < load[best]) best = r;
    P.units[u].owner = best;
    load[best] += cost(u) + 1.0;
  }
  for (auto& L : P.layers)   // an SLL block is merged on one rank: its three layers follow its owner
    if (L.cons == CONS_SLL_BLOCK)
      for (int r : {L.blk_pre, L.blk_sll, L.blk_post}) {
        const LayerInfo& M = P.layers[r];
        for (int g = 0; g < M.g; ++g) P.units[M.first_unit + g].owner = P.units[L.first_unit].owner;
      }
  for (auto& L : P.layers) L.owner = P.units[L.first_unit].owner;
}

static void layout(Plan& P) {
  int64_t off = 0, coff = 0, goff = 0;
  P.ns_flops = 0.0;
  P.bx_numel = 0;
  P.br_numel = 0;
  for (auto& M : P.mats) {
    M.off = off; off += pad_up(M.m * M.n, kPadF32);
    M.cache_off = coff; coff += pad_up(M.n, kPadF32);
    const int64_t s = std::min(M.m, M.n);
    M.gram_off = goff; goff += pad_up(s * s, kPadF32);
    M.bx_off = P.bx_numel; P.bx_numel += pad_up(pad_up(M.m, 8) * pad_up(M.n, 8), kPadBF16);
    M.br_off = P.br_numel; P.br_numel += pad_up(pad_up(s, 8) * pad_up(s, 8), kPadBF16);
    M.owned = P.units[P.layers[M.layer].first_unit + M.group].owner == P.opts.rank;
    if (M.owned && M.role != ROLE_K) {
      const double a = (double)std::max(M.m, M.n), b = (double)s;
      P.ns_flops += 4.0 * a * b * b * P.opts.ns_iters;
    }
  }
  P.params_numel = std::max<int64_t>(off, kPadF32);
  P.cache_numel = std::max<int64_t>(coff, kPadF32);
  P.gram_numel = std::max<int64_t>(goff, kPadF32);
  // final layout: layers back to back (128 B aligned), a layer's groups contiguous along dim 0
  int64_t f32 = 0, b16 = 0;
  for (auto& L : P.layers) {
    L.kf32_off = f32; f32 += pad_up(L.kernel_numel, kPadF32);
    L.kbf16_off = b16; b16 += pad_up(L.kernel_numel, kPadBF16);
  }
  P.kf32_numel = std::max<int64_t>(f32, kPadF32);
  P.kbf16_numel = std::max<int64_t>(b16, kPadBF16);
  // gather layout (a8): rank-major equal segments, each rank's units in (layer, group) order, every unit
  // 128 B aligned; world == 1 writes the final layout directly
  const int R = P.opts.world;
  std::vector<int64_t> s32(R, 0), s16(R, 0);
  for (auto& u : P.units) {
    const LayerInfo& L = P.layers[u.layer];
    u.fin_f32 = L.kf32_off + (int64_t)u.group * u.numel;
    u.fin_bf16 = L.kbf16_off + (int64_t)u.group * u.numel;
    u.gat_f32 = s32[u.owner]; s32[u.owner] += pad_up(u.numel, kPadF32);
    u.gat_bf16 = s16[u.owner]; s16[u.owner] += pad_up(u.numel, kPadBF16);
  }
  P.seg_f32 = std::max<int64_t>(*std::max_element(s32.begin(), s32.end()), kPadF32);
  P.seg_bf16 = std::max<int64_t>(*std::max_element(s16.begin(), s16.end()), kPadBF16);
  for (auto& u : P.units) { u.gat_f32 += u.owner * P.seg_f32; u.gat_bf16 += u.owner * P.seg_bf16; }
  P.gat_f32_numel = R > 1 ? P.seg_f32 * R : P.kf32_numel;
  P.gat_bf16_numel = R > 1 ? P.seg_bf16 * R : P.kbf16_numel;
}

static void finish_phase(GemmPhase& ph) {
  int32_t t = 0, tt = 0;
  for (auto& d : ph.descs) {
    const int tm = (d.M + 63) / 64, tn = (d.N + 63) / 64;
    d.tile_begin = t;
    d.tiles_n = tn;
    t += tm * tn;
    const int um = (d.M + 127) / 128, un = (d.N + 127) / 128;
    d.tc_tile_begin = tt;
    d.tc_tiles_n = un;
    tt += um * un;
  }
  ph.total_tiles = t;
  ph.tc_total_tiles = tt;
}

static GemmDesc mk(int M, int N, int K) {
  GemmDesc d{};
  d.M = M; d.N = N; d.K = K;
  d.a_buf = d.b_buf = d.c_buf = d.d_buf = BUF_NONE;
  d.c_off = -1;
  d.alpha = 1.0f; d.beta = 0.0f;
  return d;
}

static void add_seg(GemmPhase& ph, GemmDesc& d, int64_t a_off, int64_t a2_off, int64_t b_off) {
  if (d.seg_count == 0) d.seg_begin = (int32_t)ph.segs.size();
  ph.segs.push_back(GemmSeg{a_off, a2_off, b_off});
  d.seg_count++;
}

// NS phases: gram G = X^T X (m >= n) or X X^T, then X' = (1+b) X - b X G or (1+b) X - b G X.
static void build_ns(Plan& P) {
  const float b = P.opts.beta;
  P.owned_mats.clear();
  for (int i = 0; i < (int)P.mats.size(); ++i)
    if (P.mats[i].owned && P.mats[i].m > 0 && P.mats[i].n > 0 && P.mats[i].role != ROLE_K) P.owned_mats.push_back(i);
  for (int par = 0; par < 2; ++par) {
    const int xin = par == 0 ? BUF_X : BUF_Y, xout = par == 0 ? BUF_Y : BUF_X;
    GemmPhase& g = P.gram[par];
    GemmPhase& u = P.update[par];
    g.descs.clear(); g.segs.clear(); u.descs.clear(); u.segs.clear();
    for (int i : P.owned_mats) {
      const MatInfo& M = P.mats[i];
      const int m = (int)M.m, n = (int)M.n;
      if (m >= n) {
        GemmDesc d = mk(n, n, m);
        d.a_buf = xin; d.b_buf = xin; d.d_buf = BUF_G;
        d.sa_m = 1; d.sa_k = n; d.sb_k = n; d.sb_n = 1;
        d.d_off = M.gram_off; d.ldd = n;
        add_seg(g, d, M.off, -1, M.off);
        g.descs.push_back(d);
        GemmDesc e = mk(m, n, n);
        e.a_buf = xin; e.b_buf = BUF_G; e.c_buf = xin; e.d_buf = xout;
        e.sa_m = n; e.sa_k = 1; e.sb_k = n; e.sb_n = 1;
        e.c_off = M.off; e.ldc = n; e.d_off = M.off; e.ldd = n;
        e.alpha = -b; e.beta = 1.0f + b;
        add_seg(u, e, M.off, -1, M.gram_off);
        u.descs.push_back(e);
      } else {
        GemmDesc d = mk(m, m, n);
        d.a_buf = xin; d.b_buf = xin; d.d_buf = BUF_G;
        d.sa_m = n; d.sa_k = 1; d.sb_k = 1; d.sb_n = n;
        d.d_off = M.gram_off; d.ldd = m;
        add_seg(g, d, M.off, -1, M.off);
        g.descs.push_back(d);
        GemmDesc e = mk(m, n, m);
        e.a_buf = BUF_G; e.b_buf = xin; e.c_buf = xin; e.d_buf = xout;
        e.sa_m = m; e.sa_k = 1; e.sb_k = n; e.sb_n = 1;
        e.c_off = M.off; e.ldc = n; e.d_off = M.off; e.ldd = n;
        e.alpha = -b; e.beta = 1.0f + b;
        add_seg(u, e, M.gram_off, -1, M.off);
        u.descs.push_back(e);
      }
    }
    finish_phase(g);
    finish_phase(u);
    // residual form (tensor-core path): R = I - Gram, X' = X + b * (X R | R X)
    GemmPhase& gr = P.gram_r[par];
    GemmPhase& ur = P.update_r[par];
    gr = g;
    ur = u;
    for (auto& d : gr.descs) { d.alpha = -1.0f; d.diag = 1.0f; }
    for (auto& e : ur.descs) { e.alpha = b; e.beta = 1.0f; }
  }
  // tensor-core NS on BF16 copies: Gram R = I - X^T X (tall: A = B = columns of X,
  // kind 1 = MN-major loads) or I - X X^T (wide: A = B = X rows); update
  // X' = X + b X R (tall: A = X, B = R) or X + b R X (wide: A = R, B = columns
  // of X).  R is symmetric, so its rows serve as B.
  P.ns_gram.clear();
  P.ns_upd.clear();
  int32_t tg = 0, tu = 0;
  for (int i : P.owned_mats) {
    const MatInfo& M = P.mats[i];
    const int m = (int)M.m, n = (int)M.n, s = std::min(m, n);
    NsDesc base{};
    base.bx_off = M.bx_off; base.br_off = M.br_off;
    base.ldx = (int32_t)pad_up(n, 8); base.ldxt = (int32_t)pad_up(m, 8); base.ldr = (int32_t)pad_up(s, 8);
    NsDesc g = base;
    g.M = s; g.N = s; g.K = std::max(m, n);
    g.a_kind = g.b_kind = (m >= n) ? 1 : 0;
    g.a_off = g.b_off = M.bx_off;
    g.lda = g.ldb = base.ldx;   // tall: columns of X, loaded MN-major from the row-major copy
    g.epi = 0; g.f_off = M.gram_off; g.ldf = s;
    g.alpha = -1.0f; g.beta = 0.0f; g.diag = 1.0f;
    g.tile_begin = tg; g.tiles_n = (s + 127) / 128;
    tg += ((s + 127) / 128) * g.tiles_n;
    P.ns_gram.push_back(g);
    NsDesc u = base;
    u.M = m; u.N = n; u.K = s;
    if (m >= n) { u.a_kind = 0; u.a_off = M.bx_off; u.lda = base.ldx; u.b_kind = 2; u.b_off = M.br_off; u.ldb = base.ldr; }
    else { u.a_kind = 2; u.a_off = M.br_off; u.lda = base.ldr; u.b_kind = 1; u.b_off = M.bx_off; u.ldb = base.ldx; }
    u.epi = 1; u.f_off = M.off; u.ldf = n;
    u.alpha = b; u.beta = 1.0f; u.diag = 0.0f;
    u.tile_begin = tu; u.tiles_n = (n + 127) / 128;
    tu += ((m + 127) / 128) * u.tiles_n;
    P.ns_upd.push_back(u);
  }
  P.ns_gram_tiles = tg;
  P.ns_upd_tiles = tu;
  // the same count over EVERY matrix of the network (all ranks' units): the NS schedule choice
  // (ns_persist.cu: dataflow vs phase-synchronous) depends only on it, so a sharded rank runs the
  // same per-matrix arithmetic as a single-rank plan and its results are bitwise identical (R22)
  int64_t tu_all = 0;
  for (const auto& M : P.mats)
    if (M.m > 0 && M.n > 0) tu_all += ((M.m + 127) / 128) * ((M.n + 127) / 128);
  P.ns_upd_tiles_all = tu_all;
  // pre-scaling work items.  Row items (t = W v, and the scale kernels): ~8K
  // elements each, <= 64 per matrix.  Column items (w = W^T u): >= 32 columns,
  // ~8K elements each, <= 64 per matrix.  Every cross-item sum is taken in
  // item order (deterministic).
  P.power_items.clear();
  P.col_items.clear();
  P.mat_items.clear();
  P.res_items.clear();
  int chunk = 0, cchunk = 0;
  int64_t t_off = 0;
  for (int i : P.owned_mats) {
    const MatInfo& M = P.mats[i];
    const int64_t rows_fit = std::max<int64_t>(1, 8192 / M.n);
    int64_t nc = std::min<int64_t>(64, (M.m + rows_fit - 1) / rows_fit);
    nc = std::max<int64_t>(1, std::min<int64_t>(nc, M.m));
    const int64_t rpc = (M.m + nc - 1) / nc;
    // column items of 16 columns when m is large: a 512 x 16 block (row pitch 20) still fits the
    // kernel's shared-memory stage, a 512 x 32 one did not and fell back to strided L2 loads
    // (measured: column passes 10-14 us vs 6 us for the row passes)
    int64_t cpc = std::max<int64_t>(16, (8192 / std::max<int64_t>(M.m, 1)) / 16 * 16);
    cpc = std::max<int64_t>(cpc, pad_up((M.n + 63) / 64, 16));
    MatItem mi{};
    mi.mat = i; mi.m = (int32_t)M.m; mi.n = (int32_t)M.n; mi.chunk0 = chunk; mi.col0 = cchunk;
    mi.off = M.off; mi.cache_off = M.cache_off; mi.gram_off = M.gram_off; mi.t_off = t_off;
    const int midx = (int)P.mat_items.size();
    for (int64_t r0 = 0; r0 < M.m; r0 += rpc) {
      PowerItem it{};
      it.mat = i; it.r0 = (int32_t)r0; it.r1 = (int32_t)std::min<int64_t>(M.m, r0 + rpc); it.chunk = chunk++;
      it.n = (int32_t)M.n; it.m = (int32_t)M.m; it.midx = midx;
      it.off = M.off; it.cache_off = M.cache_off; it.bx_off = M.bx_off; it.t_off = t_off;
      P.power_items.push_back(it);
    }
    for (int64_t c0 = 0; c0 < M.n; c0 += cpc) {
      ColItem ci{};
      ci.mat = i; ci.c0 = (int32_t)c0; ci.c1 = (int32_t)std::min<int64_t>(M.n, c0 + cpc); ci.chunk = cchunk++;
      ci.n = (int32_t)M.n; ci.m = (int32_t)M.m; ci.midx = midx;
      ci.off = M.off; ci.cache_off = M.cache_off; ci.t_off = t_off;
      P.col_items.push_back(ci);
    }
    mi.nchunks = chunk - mi.chunk0;
    mi.ncols = cchunk - mi.col0;
    {   // residual reduction items: ~16K elements of the s x s Gram each (fixed split: deterministic sums)
      const int64_t sq = std::min(M.m, M.n) * std::min(M.m, M.n);
      const int64_t per = 16384;
      mi.res0 = (int32_t)P.res_items.size();
      for (int64_t e0 = 0; e0 < sq; e0 += per) P.res_items.push_back(ResItem{midx, 0, e0, std::min(sq, e0 + per)});
      mi.nres = (int32_t)P.res_items.size() - mi.res0;
    }
    P.mat_items.push_back(mi);
    t_off += M.m;
  }
  P.n_chunks = chunk;
  P.t_numel = t_off;
  P.partial_stride = 0;
  P.partial_numel = std::max<int64_t>(pad_up(t_off, kPadF32) + pad_up(chunk, kPadF32) + pad_up(cchunk, kPadF32),
                                      kPadF32);
}

// Composition phases (a4/a5).  Workspace (BUF_W): projectors, per-unit chain
// ping/pong, per-unit AOC result.  Inputs come from the ortho buffer (BUF_X).
static void build_compose(Plan& P) {
  int64_t w = 0;
  std::vector<int64_t> proj_off(P.mats.size(), -1);
  P.proj = GemmPhase{};
  P.chain.clear();
  P.aoc = GemmPhase{};
  P.emit.clear();
  for (int i = 0; i < (int)P.mats.size(); ++i) {
    const MatInfo& M = P.mats[i];
    if (!M.owned || M.role != ROLE_U) continue;
    proj_off[i] = w;
    w += pad_up(M.m * M.m, kPadF32);
    if (M.n == 0) continue;   // rank-0 projector: P = 0 (zero-filled at compose time)
    GemmDesc d = mk((int)M.m, (int)M.m, (int)M.n);
    d.a_buf = BUF_X; d.b_buf = BUF_X; d.d_buf = BUF_W;
    d.sa_m = M.n; d.sa_k = 1; d.sb_k = 1; d.sb_n = M.n;
    d.d_off = proj_off[i]; d.ldd = M.m;
    add_seg(P.proj, d, M.off, -1, M.off);
    P.proj.descs.push_back(d);
  }
  P.comp_proj_off = 0;
  int max_sub = 0;
  using Unit = CompUnit;
  std::vector<Unit>& units = P.comp_units;
  units.clear();
  for (int l = 0; l < (int)P.layers.size(); ++l) {
    LayerInfo& L = P.layers[l];
    for (int gi = 0; gi < L.g; ++gi) {
      if (P.units[L.first_unit + gi].owner != P.opts.rank) continue;
      Unit u{l, gi, -1, -1, -1, 0, 0};
      if ((L.cons == CONS_BCOP || L.cons == CONS_AOC) && L.kp > 1) {
        u.c = L.c_b;
        u.rows = (L.cons == CONS_BCOP) ? std::min(L.co, L.c_b) : L.c_b;   // row subset (only [:co] is kept)
        const int64_t sz = pad_up((int64_t)u.rows * u.c * L.kp * L.kp, kPadF32);
        u.ping = w; w += sz;
        u.pong = w; w += sz;
        max_sub = std::max(max_sub, 2 * (L.kp - 1));
      }
      if (L.cons == CONS_AOC) { u.fin = w; w += pad_up((int64_t)L.co * L.ci * L.k * L.k, kPadF32); }
      units.push_back(u);
    }
  }
  P.chain.assign(max_sub, GemmPhase{});
  for (auto& u : units) {
    const LayerInfo& L = P.layers[u.layer];
    if (u.ping < 0) continue;
    const int base = L.first_mat + u.group * L.mats_per_group;
    const MatInfo& Q = P.mats[base];
    const int r = u.rows, c = u.c;
    const int64_t tap = (int64_t)r * c;
    int kh = 1, kw = 1;
    int in_buf = BUF_X;
    int64_t in_off = Q.off;
    for (int t = 0; t < 2 * (L.kp - 1); ++t) {
      const bool vert = (t % 2) == 0;
      const int uidx = base + 1 + t;                 // U_{t+1}: P_{2j-1} vertical, P_{2j} horizontal
      const int64_t poff = proj_off[uidx];
      const int oh = vert ? kh + 1 : kh, ow = vert ? kw : kw + 1;
      const int64_t out_off = (t % 2 == 0) ? u.ping : u.pong;
      GemmPhase& ph = P.chain[t];
      for (int p = 0; p < oh; ++p)
        for (int q = 0; q < ow; ++q) {
          // D[p,q] = (K[cur] - K[prev]) P + K[prev]; prev = tap shifted by one along the step axis
          const int cp = p, cq = q;
          const int pp = vert ? p - 1 : p, pq = vert ? q : q - 1;
          const bool has_cur = vert ? (p < kh) : (q < kw);
          const bool has_prev = vert ? (p >= 1) : (q >= 1);
          const int64_t cur = in_off + (int64_t)(cp * kw + cq) * tap;
          const int64_t prev = in_off + (int64_t)(pp * kw + pq) * tap;
          GemmDesc d = mk(r, c, c);
          d.a_buf = in_buf; d.b_buf = BUF_W; d.d_buf = BUF_W;
          d.sa_m = c; d.sa_k = 1; d.sb_k = c; d.sb_n = 1;
          d.d_off = out_off + (int64_t)(p * ow + q) * tap; d.ldd = c;
          if (has_cur && has_prev) {
            add_seg(ph, d, cur, prev, poff);
            d.c_buf = in_buf; d.c_off = prev; d.ldc = c; d.beta = 1.0f;
          } else if (has_cur) {
            add_seg(ph, d, cur, -1, poff);
          } else {  // last row/col: K[prev] (I - P)
            add_seg(ph, d, prev, -1, poff);
            d.alpha = -1.0f;
            d.c_buf = in_buf; d.c_off = prev; d.ldc = c; d.beta = 1.0f;
          }
          ph.descs.push_back(d);
        }
      kh = oh; kw = ow;
      in_buf = BUF_W;
      in_off = out_off;
    }
  }
  // AOC: K[p,q] = sum_{a,b} R_{ab} Kb[p-a, q-b]   (R_{ab}[o, j] = R[o, j s^2 + a s + b], R7)
  for (auto& u : units) {
    const LayerInfo& L = P.layers[u.layer];
    if (L.cons != CONS_AOC) continue;
    const int base = L.first_mat + u.group * L.mats_per_group;
    const MatInfo& R = P.mats[base + L.mats_per_group - 1];
    const int s = L.s, kp = L.kp, k = L.k, c = u.c;
    const int64_t tap = (int64_t)u.rows * c;
    for (int p = 0; p < k; ++p)
      for (int q = 0; q < k; ++q) {
        GemmDesc d = mk(L.co, L.ci, L.c_mid);
        d.a_buf = BUF_X; d.b_buf = BUF_W; d.d_buf = BUF_W;
        d.sa_m = (int64_t)L.c_mid * s * s; d.sa_k = (int64_t)s * s; d.sb_k = c; d.sb_n = 1;
        d.d_off = u.fin + (int64_t)(p * k + q) * L.co * L.ci; d.ldd = L.ci;
        for (int a = 0; a < s; ++a)
          for (int b = 0; b < s; ++b) {
            const int ta = p - a, tb = q - b;
            if (ta < 0 || tb < 0 || ta >= kp || tb >= kp) continue;
            add_seg(P.aoc, d, R.off + a * s + b, -1, u.pong + (int64_t)(ta * kp + tb) * tap);
          }
        P.aoc.descs.push_back(d);
      }
  }
  for (auto* ph : {&P.proj, &P.aoc}) finish_phase(*ph);
  for (auto& ph : P.chain) finish_phase(ph);
  // f3 SOC units: S (skew part, k^2 taps), its powers S^(*)j (((j(k-1)+1)^2 taps), j = 2..max(n, 2)) and the
  // explicit exponential E (kn^2 taps), all tap-major c x c in the composition workspace
  P.soc.clear();
  P.soc_copy.clear();
  std::vector<int64_t> soc_e(units.size(), -1);
  int max_terms = 0;
  for (size_t ui = 0; ui < units.size(); ++ui) {
    const auto& u = units[ui];
    const LayerInfo& L = P.layers[u.layer];
    if (L.cons != CONS_SOC) continue;
    const MatInfo& Km = P.mats[L.first_mat + u.group];
    SocItem it{};
    it.c = L.co; it.k = L.k_free; it.kn = L.k; it.terms = L.soc_terms;
    it.alpha_slot = (int)P.soc.size();
    it.src_off = Km.off;
    P.soc_copy.push_back(Km.off);
    P.soc_copy.push_back(Km.m * Km.n);
    const int64_t c2 = (int64_t)it.c * it.c;
    for (int j = 1; j <= std::max(it.terms, 2); ++j) {
      const int64_t kj = (int64_t)j * (it.k - 1) + 1;
      it.u_off[j] = w;
      w += pad_up(kj * kj * c2, kPadF32);
    }
    it.e_off = w;
    w += pad_up((int64_t)it.kn * it.kn * c2, kPadF32);
    soc_e[ui] = it.e_off;
    max_terms = std::max(max_terms, std::max(it.terms, 2));
    P.soc.push_back(it);
  }
  P.soc_pow.assign(std::max(0, max_terms - 1), GemmPhase{});
  for (const auto& it : P.soc) {
    const int64_t c2 = (int64_t)it.c * it.c;
    for (int j = 2; j <= std::max(it.terms, 2); ++j) {
      GemmPhase& ph = P.soc_pow[j - 2];
      const int kj = j * (it.k - 1) + 1, kp = (j - 1) * (it.k - 1) + 1;
      for (int p1 = 0; p1 < kj; ++p1)
        for (int p2 = 0; p2 < kj; ++p2) {
          GemmDesc d = mk(it.c, it.c, it.c);   // U_j[p] = sum_{a + b = p} U_{j-1}[a] S[b]
          d.a_buf = BUF_W; d.b_buf = BUF_W; d.d_buf = BUF_W;
          d.sa_m = it.c; d.sa_k = 1; d.sb_k = it.c; d.sb_n = 1;
          d.d_off = it.u_off[j] + (int64_t)(p1 * kj + p2) * c2; d.ldd = it.c;
          for (int b1 = 0; b1 < it.k; ++b1)
            for (int b2 = 0; b2 < it.k; ++b2) {
              const int a1 = p1 - b1, a2 = p2 - b2;
              if (a1 < 0 || a2 < 0 || a1 >= kp || a2 >= kp) continue;
              add_seg(ph, d, it.u_off[j - 1] + (int64_t)(a1 * kp + a2) * c2, -1,
                      it.u_off[1] + (int64_t)(b1 * it.k + b2) * c2);
            }
          ph.descs.push_back(d);
        }
    }
  }
  for (auto& ph : P.soc_pow) finish_phase(ph);
  // f4 SLL units: V[Delta] = sum_t W_t^T W_{t+Delta} read in place from ortho (W: (co, ci, k, k)), the
  // per-input-channel scale, the rescaled tap-major kernel (R28)
  P.sll.clear();
  P.sll_v = GemmPhase{};
  std::vector<int64_t> sll_kt(units.size(), -1);
  for (size_t ui = 0; ui < units.size(); ++ui) {
    const auto& u = units[ui];
    const LayerInfo& L = P.layers[u.layer];
    if (L.cons != CONS_SLL) continue;
    SllItem it{};
    it.ci = L.ci; it.co = L.co; it.k = L.k;
    it.src_off = P.mats[L.first_mat].off;
    P.soc_copy.push_back(it.src_off);                       // role K: passed through params -> ortho
    P.soc_copy.push_back(P.mats[L.first_mat].m * P.mats[L.first_mat].n);
    const int k2 = 2 * L.k - 1, kk = L.k * L.k;
    const int64_t c2 = (int64_t)L.ci * L.ci;
    it.v_off = w; w += pad_up((int64_t)k2 * k2 * c2, kPadF32);
    it.s_off = w; w += pad_up(L.ci, kPadF32);
    it.kt_off = w; w += pad_up((int64_t)kk * L.co * L.ci, kPadF32);
    sll_kt[ui] = it.kt_off;
    for (int d1 = -(L.k - 1); d1 < L.k; ++d1)
      for (int d2 = -(L.k - 1); d2 < L.k; ++d2) {
        GemmDesc d = mk(L.ci, L.ci, L.co);
        d.a_buf = BUF_X; d.b_buf = BUF_X; d.d_buf = BUF_W;
        d.sa_m = kk; d.sa_k = (int64_t)L.ci * kk; d.sb_k = (int64_t)L.ci * kk; d.sb_n = kk;
        d.d_off = it.v_off + (int64_t)((d1 + L.k - 1) * k2 + (d2 + L.k - 1)) * c2; d.ldd = L.ci;
        for (int a1 = 0; a1 < L.k; ++a1)
          for (int a2 = 0; a2 < L.k; ++a2) {
            const int b1 = a1 + d1, b2 = a2 + d2;
            if (b1 < 0 || b2 < 0 || b1 >= L.k || b2 >= L.k) continue;
            add_seg(P.sll_v, d, it.src_off + a1 * L.k + a2, -1, it.src_off + b1 * L.k + b2);
          }
        if (d.seg_count == 0) {   // no overlapping taps cannot happen for |Delta| < k, kept for safety
          add_seg(P.sll_v, d, it.src_off, -1, it.src_off);
          d.alpha = 0.f;
        }
        P.sll_v.descs.push_back(d);
      }
    P.sll.push_back(it);
  }
  finish_phase(P.sll_v);
  // f4 SLL x AOC blocks: C, A, B from the emitted FP32 kernels of the three layers (BUF_Y = kernels_f32, at
  // the offsets the first emit wrote), M = [A | -2 B] (R29), second emit into the block's kernel region
  P.blk.clear();
  P.blk_mm = GemmPhase{};
  P.emit2.clear();
  auto kofs = [&](int layer) {
    const UnitInfo& U = P.units[P.layers[layer].first_unit];
    return P.opts.world > 1 ? U.gat_f32 : U.fin_f32;
  };
  for (auto& u : units) {
    const LayerInfo& L = P.layers[u.layer];
    if (L.cons != CONS_SLL_BLOCK) continue;
    const LayerInfo &Pre = P.layers[L.blk_pre], &S = P.layers[L.blk_sll], &Po = P.layers[L.blk_post];
    const int c = L.ci, cs = L.blk_cs, co = L.co, kp = Pre.k, ks = S.k, kq = Po.k;
    const int64_t pre = kofs(L.blk_pre), sl = kofs(L.blk_sll), post = kofs(L.blk_post);
    BlkItem b{};
    b.c = c; b.cs = cs; b.co = co;
    b.kA = kq + kp - 1; b.kB = kq + ks - 1; b.kM = L.kM;
    b.oa = L.pM - (Po.pt + Pre.pt);
    b.ob = L.pM - (Po.pt + (ks - 1 - S.pt));
    b.c_off = w; w += pad_up((int64_t)L.kC * L.kC * cs * c, kPadF32);
    b.a_off = w; w += pad_up((int64_t)b.kA * b.kA * co * c, kPadF32);
    b.b_off = w; w += pad_up((int64_t)b.kB * b.kB * co * cs, kPadF32);
    b.m_off = w; w += pad_up((int64_t)b.kM * b.kM * co * (c + cs), kPadF32);
    // X[p] = sum_{a + b = p} F[a] G[b] over PyTorch-layout factors: F tap a (rows x inner) at fo + (r * inner + i) kf^2 + a
    auto prod = [&](int rows, int inner, int cols, int64_t fo, int kf, int64_t go, int kg, bool g_adj, int64_t out) {
      const int kx = kf + kg - 1;
      for (int p1 = 0; p1 < kx; ++p1)
        for (int p2 = 0; p2 < kx; ++p2) {
          GemmDesc d = mk(rows, cols, inner);
          d.a_buf = BUF_Y; d.b_buf = BUF_Y; d.d_buf = BUF_W;
          d.sa_m = (int64_t)inner * kf * kf; d.sa_k = (int64_t)kf * kf;
          if (!g_adj) { d.sb_k = (int64_t)cols * kg * kg; d.sb_n = (int64_t)kg * kg; }   // G[i][j] at (i cols + j) kg^2
          else { d.sb_k = (int64_t)kg * kg; d.sb_n = (int64_t)inner * kg * kg; }          // G = K^T flipped: K[j][i]
          d.d_off = out + (int64_t)(p1 * kx + p2) * rows * cols; d.ldd = cols;
          for (int a1 = 0; a1 < kf; ++a1)
            for (int a2 = 0; a2 < kf; ++a2) {
              const int b1 = p1 - a1, b2 = p2 - a2;
              if (b1 < 0 || b2 < 0 || b1 >= kg || b2 >= kg) continue;
              const int gt = g_adj ? (kg * kg - 1 - (b1 * kg + b2)) : (b1 * kg + b2);
              add_seg(P.blk_mm, d, fo + a1 * kf + a2, -1, go + gt);
            }
          P.blk_mm.descs.push_back(d);
        }
    };
    prod(cs, c, c, sl, ks, pre, kp, false, b.c_off);     // C = K (*) K_pre
    prod(co, c, c, post, kq, pre, kp, false, b.a_off);   // A = K_post (*) K_pre
    prod(co, c, cs, post, kq, sl, ks, true, b.b_off);    // B = K_post (*) K^T
    P.blk.push_back(b);
    const UnitInfo& U = P.units[L.first_unit];
    EmitItem ec{}, em{};
    ec.layer = em.layer = u.layer;
    ec.co = cs; ec.ci = c; ec.k = L.kC; ec.s = 1; ec.ci_f_per_g = c;
    ec.src_buf = BUF_W; ec.src_off = b.c_off; ec.tap_stride = (int64_t)cs * c; ec.ld = c;
    ec.mode = (int64_t)L.kC * L.kC * c * 4 > 96 * 1024 ? 2 : 0;
    ec.f32_off = P.opts.world > 1 ? U.gat_f32 : U.fin_f32;
    ec.bf16_off = P.opts.world > 1 ? U.gat_bf16 : U.fin_bf16;
    em.co = co; em.ci = c + cs; em.k = L.kM; em.s = L.s; em.ci_f_per_g = c + cs;
    em.src_buf = BUF_W; em.src_off = b.m_off; em.tap_stride = (int64_t)co * (c + cs); em.ld = c + cs;
    em.mode = (int64_t)L.kM * L.kM * (c + cs) * 4 > 96 * 1024 ? 2 : 0;
    em.f32_off = ec.f32_off + L.m_off;
    em.bf16_off = ec.bf16_off + L.m_off;
    P.emit2.push_back(ec);
    P.emit2.push_back(em);
  }
  finish_phase(P.blk_mm);
  // emit items
  for (size_t ui = 0; ui < units.size(); ++ui) {
    const auto& u = units[ui];
    const LayerInfo& L = P.layers[u.layer];
    const int base = L.first_mat + u.group * L.mats_per_group;
    EmitItem e{};
    e.layer = u.layer; e.group = u.group;
    e.co = L.co; e.ci = L.ci; e.k = (L.cons == CONS_DENSE) ? 1 : L.k; e.s = L.s; e.ci_f_per_g = L.ci;
    if (L.cons == CONS_SLL_BLOCK) continue;    // written by the second emit (emit2)
    const UnitInfo& U = P.units[L.first_unit + u.group];
    e.f32_off = P.opts.world > 1 ? U.gat_f32 : U.fin_f32;     // world > 1: this rank's gather segment
    e.bf16_off = P.opts.world > 1 ? U.gat_bf16 : U.fin_bf16;
    switch (L.cons) {
      case CONS_DENSE:
        e.src_buf = BUF_X; e.src_off = P.mats[base].off; e.mode = 0; e.tap_stride = 0; e.ld = L.ci; break;
      case CONS_RKO:
        e.src_buf = BUF_X; e.src_off = P.mats[base].off; e.mode = 1; e.tap_stride = 0; e.ld = 0; break;
      case CONS_AOC:
        e.src_buf = BUF_W; e.src_off = u.fin; e.mode = 0; e.tap_stride = (int64_t)L.co * L.ci; e.ld = L.ci; break;
      case CONS_SLL:   // the AOL-rescaled kernel, tap-major
        e.src_buf = BUF_W; e.src_off = sll_kt[ui]; e.tap_stride = (int64_t)L.co * L.ci; e.ld = L.ci;
        e.mode = (int64_t)L.k * L.k * L.ci * 4 > 96 * 1024 ? 2 : 0;
        break;
      case CONS_SOC:   // E, tap-major; large k_eff^2 c rows are written without the shared-memory stage
        e.src_buf = BUF_W; e.src_off = soc_e[ui]; e.tap_stride = (int64_t)L.co * L.ci; e.ld = L.ci;
        e.mode = (int64_t)L.k * L.k * L.ci * 4 > 96 * 1024 ? 2 : 0;
        break;
      default:  // BCOP
        if (L.kp == 1) { e.src_buf = BUF_X; e.src_off = P.mats[base].off; e.mode = 0; e.tap_stride = 0; e.ld = L.c_b; }
        else { e.src_buf = BUF_W; e.src_off = u.pong; e.mode = 0; e.tap_stride = (int64_t)u.rows * u.c; e.ld = u.c; }
    }
    P.emit.push_back(e);
  }
  P.comp_numel = std::max<int64_t>(w, kPadF32);
  P.proj_off = proj_off;
}


// ---------------------------------------------------------------------------------------------------
// f1: VJP phases (opts.vjp != 0).  Buffers of every VJP GEMM: BUF_X = ortho (compose VJP), BUF_Y = the VJP
// arena, BUF_G = d_ortho (compose VJP output), BUF_W = comp (projectors).  The NS VJP reads G_T from a copy
// of d_ortho in the arena, so all its operands share BUF_Y.
// ---------------------------------------------------------------------------------------------------
static void build_vjp(Plan& P) {
  const float b = P.opts.beta;
  const int T = P.opts.ns_iters;
  int64_t w = 0;
  auto take = [&](int64_t n) { int64_t o = w; w += pad_up(std::max<int64_t>(n, 1), kPadF32); return o; };
  // ---- NS: X_t slots, two G slots, R / S (short-side squares)
  const int64_t PN = P.params_numel;
  P.vj_x_off = take((int64_t)T * PN);
  P.vj_g_off[0] = take(PN);
  P.vj_g_off[1] = take(PN);
  P.vj_r_off = take(P.gram_numel);
  P.vj_s_off = take(P.gram_numel);
  P.vj_fwd.assign(2 * T, GemmPhase{});
  P.vj_bwd.assign(2 * T, GemmPhase{});
  auto gram_desc = [&](const MatInfo& M, int64_t x, int64_t r) {   // R = I - X^T X | I - X X^T
    const int m = (int)M.m, n = (int)M.n;
    const bool tall = m >= n;
    const int sh = tall ? n : m;
    GemmDesc d = mk(sh, sh, tall ? m : n);
    d.a_buf = d.b_buf = d.d_buf = BUF_Y;
    if (tall) { d.sa_m = 1; d.sa_k = n; d.sb_k = n; d.sb_n = 1; }
    else { d.sa_m = n; d.sa_k = 1; d.sb_k = 1; d.sb_n = n; }
    d.d_off = r; d.ldd = sh;
    d.alpha = -1.0f; d.diag = 1.0f;
    return d;
  };
  for (int t = 0; t < T; ++t) {
    GemmPhase& g = P.vj_fwd[2 * t];
    GemmPhase& u = P.vj_fwd[2 * t + 1];
    const int64_t xt = P.vj_x_off + (int64_t)t * PN;
    for (int i : P.owned_mats) {
      const MatInfo& M = P.mats[i];
      const int m = (int)M.m, n = (int)M.n;
      const bool tall = m >= n;
      const int sh = tall ? n : m;
      GemmDesc d = gram_desc(M, xt + M.off, P.vj_r_off + M.gram_off);
      add_seg(g, d, xt + M.off, -1, xt + M.off);
      g.descs.push_back(d);
      if (t + 1 < T) {   // X_{t+1} = X_t + b (X_t R | R X_t) into slot t + 1 (X_T itself is not needed)
        GemmDesc e = mk(m, n, sh);
        e.a_buf = e.b_buf = e.c_buf = e.d_buf = BUF_Y;
        e.sa_m = tall ? n : sh; e.sa_k = 1; e.sb_k = n; e.sb_n = 1;
        if (tall) add_seg(u, e, xt + M.off, -1, P.vj_r_off + M.gram_off);
        else add_seg(u, e, P.vj_r_off + M.gram_off, -1, xt + M.off);
        e.c_off = xt + M.off; e.ldc = n; e.d_off = xt + PN + M.off; e.ldd = n;
        e.alpha = b; e.beta = 1.0f;
        u.descs.push_back(e);
      }
    }
    finish_phase(g);
    finish_phase(u);
  }
  // backward: iteration j handles t = T-1-j; G_in = slot[(j+1)&1] (slot 1 holds the copy of G_T), G_out =
  // slot[j&1].  Tall: S' = -(X^T G + G^T X), G' = G + b (G R + X S').  Wide: S' = -(G X^T + X G^T),
  // G' = G + b (R G + S' X).  (The adjoint of X' = X + b X (I - X^T X).)
  for (int j = 0; j < T; ++j) {
    const int t = T - 1 - j;
    const int64_t xt = P.vj_x_off + (int64_t)t * PN;
    const int64_t gin = P.vj_g_off[(j + 1) & 1], gout = P.vj_g_off[j & 1];
    GemmPhase& a = P.vj_bwd[2 * j];
    GemmPhase& c = P.vj_bwd[2 * j + 1];
    for (int i : P.owned_mats) {
      const MatInfo& M = P.mats[i];
      const int m = (int)M.m, n = (int)M.n;
      const bool tall = m >= n;
      const int sh = tall ? n : m;
      GemmDesc d = gram_desc(M, xt + M.off, P.vj_r_off + M.gram_off);
      add_seg(a, d, xt + M.off, -1, xt + M.off);
      a.descs.push_back(d);
      GemmDesc sd = mk(sh, sh, tall ? m : n);
      sd.a_buf = sd.b_buf = sd.d_buf = BUF_Y;
      if (tall) {   // X^T G + G^T X
        sd.sa_m = 1; sd.sa_k = n; sd.sb_k = n; sd.sb_n = 1;
        add_seg(a, sd, xt + M.off, -1, gin + M.off);
        add_seg(a, sd, gin + M.off, -1, xt + M.off);
      } else {      // G X^T + X G^T
        sd.sa_m = n; sd.sa_k = 1; sd.sb_k = 1; sd.sb_n = n;
        add_seg(a, sd, gin + M.off, -1, xt + M.off);
        add_seg(a, sd, xt + M.off, -1, gin + M.off);
      }
      sd.d_off = P.vj_s_off + M.gram_off; sd.ldd = sh; sd.alpha = -1.0f;
      a.descs.push_back(sd);
      GemmDesc e = mk(m, n, sh);
      e.a_buf = e.b_buf = e.c_buf = e.d_buf = BUF_Y;
      e.c_off = gin + M.off; e.ldc = n; e.beta = 1.0f;
      e.d_off = gout + M.off; e.ldd = n; e.alpha = b;
      e.sa_m = tall ? n : sh; e.sa_k = 1; e.sb_k = n; e.sb_n = 1;
      if (tall) {
        add_seg(c, e, gin + M.off, -1, P.vj_r_off + M.gram_off);   // G R
        add_seg(c, e, xt + M.off, -1, P.vj_s_off + M.gram_off);    // X S'
      } else {
        add_seg(c, e, P.vj_r_off + M.gram_off, -1, gin + M.off);   // R G
        add_seg(c, e, P.vj_s_off + M.gram_off, -1, xt + M.off);    // S' X
      }
      c.descs.push_back(e);
    }
    finish_phase(a);
    finish_phase(c);
  }
  P.vj_g_final = T > 0 ? ((T - 1) & 1) : 1;
  // ---- composition VJP (owned BCOP / AOC / RKO / dense units)
  P.cv_fwd.clear(); P.cv_bwd_a.clear(); P.cv_bwd_b.clear(); P.cv_bwd_c.clear();
  P.cv_dr = GemmPhase{}; P.cv_dkb = GemmPhase{};
  P.cv_items.clear(); P.cv_scatter.clear(); P.cv_qcopy.clear();
  P.vjp_supported = true;
  P.cv_zero_off = w;   // everything taken from here on is zeroed at the start of orth_compose_vjp
  int64_t max_tap = 64;
  for (auto& u : P.comp_units) max_tap = std::max<int64_t>(max_tap, (int64_t)u.rows * u.c);
  const int64_t zero_off = take(max_tap);   // a zero tap for missing chain neighbours
  int max_steps = 0;
  struct UnitV { int64_t step_off[64]; int64_t dstep_off[64]; int nsteps; int64_t dfin_off, drab_off, q_off; };
  std::vector<UnitV> uv(P.comp_units.size());
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    const LayerInfo& L = P.layers[u.layer];
    UnitV& V = uv[ui];
    V.nsteps = 0; V.dfin_off = V.drab_off = V.q_off = -1;
    if (L.cons == CONS_SOC || L.cons == CONS_SLL || L.cons == CONS_SLL_BLOCK) { P.vjp_supported = false; continue; }
    if (u.ping >= 0) {
      V.nsteps = 2 * (L.kp - 1);
      V.q_off = take((int64_t)u.rows * u.c);
      int kh = 1, kw = 1;
      for (int t = 0; t < V.nsteps; ++t) {
        const bool vert = (t % 2) == 0;
        const int oh = vert ? kh + 1 : kh, ow = vert ? kw : kw + 1;
        V.step_off[t] = take((int64_t)oh * ow * u.rows * u.c);
        V.dstep_off[t] = take((int64_t)oh * ow * u.rows * u.c);
        kh = oh; kw = ow;
      }
      max_steps = std::max(max_steps, V.nsteps);
    }
    if (L.cons == CONS_AOC) {
      V.dfin_off = take((int64_t)L.k * L.k * L.co * L.ci);
      V.drab_off = take((int64_t)L.s * L.s * L.co * L.c_mid);
    }
  }
  P.cv_fwd.assign(max_steps, GemmPhase{});
  P.cv_bwd_a.assign(max_steps, GemmPhase{});
  P.cv_bwd_b.assign(max_steps, GemmPhase{});
  P.cv_bwd_c.assign(max_steps, GemmPhase{});
  for (size_t ui = 0; ui < P.comp_units.size(); ++ui) {
    const CompUnit& u = P.comp_units[ui];
    const LayerInfo& L = P.layers[u.layer];
    const UnitV& V = uv[ui];
    if (L.cons == CONS_SOC || L.cons == CONS_SLL || L.cons == CONS_SLL_BLOCK) continue;
    const int base = L.first_mat + u.group * L.mats_per_group;
    const UnitInfo& U = P.units[L.first_unit + u.group];
    const int r = u.rows, c = u.c;
    const int64_t tap = (int64_t)r * c;
    VjpItem it{};
    it.co = L.co; it.ci = L.ci; it.kk = (L.cons == CONS_DENSE) ? 1 : L.k * L.k;
    it.src_off = U.fin_f32;   // dK arrives in the final layout (all-reduced across ranks)
    it.zero_off = -1; it.zero_n = 0;
    if (L.cons == CONS_DENSE || L.cons == CONS_RKO) {
      it.mode = 2;
      it.dst_off = P.mats[base + L.mats_per_group - 1].off;
      it.rows = L.co; it.c = L.ci;
      P.cv_items.push_back(it);
      continue;
    }
    if (L.cons == CONS_BCOP && L.kp == 1) {
      it.mode = 3; it.dst_off = P.mats[base].off; it.rows = L.c_b; it.c = L.c_b;
      P.cv_items.push_back(it);
      continue;
    }
    // chain unit (BCOP k' > 1, or AOC): zero dQ, then the last step's gradient (BCOP) or dFin (AOC)
    it.zero_off = P.mats[base].off; it.zero_n = (int64_t)c * c;
    it.rows = r; it.c = c;
    if (L.cons == CONS_AOC) { it.mode = 1; it.dst_off = V.dfin_off; }
    else { it.mode = 0; it.dst_off = V.dstep_off[V.nsteps - 1]; }
    P.cv_items.push_back(it);
    P.cv_qcopy.push_back(P.mats[base].off);   // Q rows [0, r) -> the arena (the backward reads it from BUF_Y)
    P.cv_qcopy.push_back(V.q_off);
    P.cv_qcopy.push_back(tap);
    // forward chain into per-step buffers (same arithmetic as build_compose's chain)
    auto step_geo = [](int t, int& kh, int& kw) { kh = 1; kw = 1; for (int x = 0; x < t; ++x) { if (x % 2 == 0) kh++; else kw++; } };
    for (int t = 0; t < V.nsteps; ++t) {
      const bool vert = (t % 2) == 0;
      int kh, kw;
      step_geo(t, kh, kw);
      const int64_t poff = P.proj_off[base + 1 + t];
      const int oh = vert ? kh + 1 : kh, ow = vert ? kw : kw + 1;
      const int64_t in_off = t == 0 ? V.q_off : V.step_off[t - 1];
      for (int p = 0; p < oh; ++p)
        for (int q = 0; q < ow; ++q) {
          const int pp = vert ? p - 1 : p, pq = vert ? q : q - 1;
          const bool has_cur = vert ? (p < kh) : (q < kw);
          const bool has_prev = vert ? (p >= 1) : (q >= 1);
          const int64_t cur = in_off + (int64_t)(p * kw + q) * tap;
          const int64_t prev = in_off + (int64_t)(pp * kw + pq) * tap;
          GemmDesc d = mk(r, c, c);
          d.a_buf = BUF_Y; d.b_buf = BUF_W; d.d_buf = BUF_Y;
          d.sa_m = c; d.sa_k = 1; d.sb_k = c; d.sb_n = 1;
          d.d_off = V.step_off[t] + (int64_t)(p * ow + q) * tap; d.ldd = c;
          if (has_cur && has_prev) {
            add_seg(P.cv_fwd[t], d, cur, prev, poff);
            d.c_buf = BUF_Y; d.c_off = prev; d.ldc = c; d.beta = 1.0f;
          } else if (has_cur) {
            add_seg(P.cv_fwd[t], d, cur, -1, poff);
          } else {
            add_seg(P.cv_fwd[t], d, prev, -1, poff);
            d.alpha = -1.0f;
            d.c_buf = BUF_Y; d.c_off = prev; d.ldc = c; d.beta = 1.0f;
          }
          P.cv_fwd[t].descs.push_back(d);
        }
    }
    // AOC backward: dR_ab = sum_p dFin[p] Kb[p - ab]^T (first ci columns), dKb[q] = sum_ab R_ab^T dFin[q + ab]
    if (L.cons == CONS_AOC) {
      const MatInfo& R = P.mats[base + L.mats_per_group - 1];
      const int s = L.s, kp = L.kp, k = L.k, cm = L.c_mid;
      const int64_t kb_off = V.step_off[V.nsteps - 1];
      for (int a = 0; a < s; ++a)
        for (int bb = 0; bb < s; ++bb) {
          GemmDesc d = mk(L.co, cm, L.ci);
          d.a_buf = BUF_Y; d.b_buf = BUF_Y; d.d_buf = BUF_Y;
          d.sa_m = L.ci; d.sa_k = 1; d.sb_k = 1; d.sb_n = c;
          d.d_off = V.drab_off + (int64_t)(a * s + bb) * L.co * cm; d.ldd = cm;
          for (int p = 0; p < k; ++p)
            for (int q = 0; q < k; ++q) {
              const int ta = p - a, tb = q - bb;
              if (ta < 0 || tb < 0 || ta >= kp || tb >= kp) continue;
              add_seg(P.cv_dr, d, V.dfin_off + (int64_t)(p * k + q) * L.co * L.ci, -1,
                      kb_off + (int64_t)(ta * kp + tb) * tap);
            }
          P.cv_dr.descs.push_back(d);
        }
      ScatterItem sc{L.co, cm, s * s, 0, V.drab_off, R.off};
      P.cv_scatter.push_back(sc);
      for (int ta = 0; ta < kp; ++ta)
        for (int tb = 0; tb < kp; ++tb) {
          GemmDesc d = mk(cm, L.ci, L.co);   // dKb[q][j][i] for i < ci (the rest of the row stays 0)
          d.a_buf = BUF_X; d.b_buf = BUF_Y; d.d_buf = BUF_Y;
          d.sa_m = s * s; d.sa_k = (int64_t)cm * s * s; d.sb_k = L.ci; d.sb_n = 1;
          d.d_off = V.dstep_off[V.nsteps - 1] + (int64_t)(ta * kp + tb) * tap; d.ldd = c;
          for (int a = 0; a < s; ++a)
            for (int bb = 0; bb < s; ++bb)
              add_seg(P.cv_dkb, d, R.off + a * s + bb, -1,
                      V.dfin_off + (int64_t)((ta + a) * k + (tb + bb)) * L.co * L.ci);
          P.cv_dkb.descs.push_back(d);
        }
    }
    // chain backward, aligned from each unit's last step: iteration j handles step t = nsteps - 1 - j
    for (int j = 0; j < V.nsteps; ++j) {
      const int t = V.nsteps - 1 - j;
      const bool vert = (t % 2) == 0;
      int kh, kw;
      step_geo(t, kh, kw);
      const int oh = vert ? kh + 1 : kh, ow = vert ? kw : kw + 1;
      const int uidx = base + 1 + t;
      const int64_t poff = P.proj_off[uidx];
      const int64_t in_off = t == 0 ? V.q_off : V.step_off[t - 1];
      const int64_t dout = V.dstep_off[t];
      const int64_t dP_off = take((int64_t)c * c);
      // dP = sum_y (K_in[cur(y)] - K_in[prev(y)])^T dS[y]   (a missing neighbour is the zero tap)
      GemmDesc dp = mk(c, c, r);
      dp.a_buf = BUF_Y; dp.b_buf = BUF_Y; dp.d_buf = BUF_Y;
      dp.sa_m = 1; dp.sa_k = c; dp.sb_k = c; dp.sb_n = 1;
      dp.d_off = dP_off; dp.ldd = c;
      for (int p = 0; p < oh; ++p)
        for (int q = 0; q < ow; ++q) {
          const int pp = vert ? p - 1 : p, pq = vert ? q : q - 1;
          const bool has_cur = vert ? (p < kh) : (q < kw);
          const bool has_prev = vert ? (p >= 1) : (q >= 1);
          const int64_t cur = has_cur ? in_off + (int64_t)(p * kw + q) * tap : zero_off;
          const int64_t prev = has_prev ? in_off + (int64_t)(pp * kw + pq) * tap : -1;
          add_seg(P.cv_bwd_a[j], dp, cur, prev, dout + (int64_t)(p * ow + q) * tap);
        }
      P.cv_bwd_a[j].descs.push_back(dp);
      // dK_in[x] = (dS[x] - dS[x + step]) P + dS[x + step]   (every input tap has both neighbours)
      for (int p = 0; p < kh; ++p)
        for (int q = 0; q < kw; ++q) {
          const int np = vert ? p + 1 : p, nq = vert ? q : q + 1;
          const int64_t d0 = dout + (int64_t)(p * ow + q) * tap, d1 = dout + (int64_t)(np * ow + nq) * tap;
          GemmDesc d = mk(r, c, c);
          d.a_buf = BUF_Y; d.b_buf = BUF_W;
          d.sa_m = c; d.sa_k = 1; d.sb_k = c; d.sb_n = 1;
          d.c_buf = BUF_Y; d.c_off = d1; d.ldc = c; d.beta = 1.0f;
          if (t == 0) { d.d_buf = BUF_G; d.d_off = P.mats[base].off; }   // dQ rows [0, r)
          else { d.d_buf = BUF_Y; d.d_off = V.dstep_off[t - 1] + (int64_t)(p * kw + q) * tap; }
          d.ldd = c;
          add_seg(P.cv_bwd_a[j], d, d0, d1, poff);
          P.cv_bwd_a[j].descs.push_back(d);
        }
      // dU = (dP + dP^T) U: dP U (phase b), then + dP^T U through C (phase c)
      const MatInfo& Um = P.mats[uidx];
      if (Um.n > 0) {
        GemmDesc du = mk((int)Um.m, (int)Um.n, c);
        du.a_buf = BUF_Y; du.b_buf = BUF_X; du.d_buf = BUF_G;
        du.sa_m = c; du.sa_k = 1; du.sb_k = Um.n; du.sb_n = 1;
        du.d_off = Um.off; du.ldd = Um.n;
        add_seg(P.cv_bwd_b[j], du, dP_off, -1, Um.off);
        P.cv_bwd_b[j].descs.push_back(du);
        GemmDesc dt = mk((int)Um.m, (int)Um.n, c);
        dt.a_buf = BUF_Y; dt.b_buf = BUF_X; dt.d_buf = BUF_G;
        dt.sa_m = 1; dt.sa_k = c; dt.sb_k = Um.n; dt.sb_n = 1;
        dt.d_off = Um.off; dt.ldd = Um.n;
        dt.c_buf = BUF_G; dt.c_off = Um.off; dt.ldc = Um.n; dt.beta = 1.0f;
        add_seg(P.cv_bwd_c[j], dt, dP_off, -1, Um.off);
        P.cv_bwd_c[j].descs.push_back(dt);
      }
    }
  }
  P.cv_zero_n = w - P.cv_zero_off;
  finish_phase(P.cv_dr);
  finish_phase(P.cv_dkb);
  for (auto& ph : P.cv_fwd) finish_phase(ph);
  for (auto& ph : P.cv_bwd_a) finish_phase(ph);
  for (auto& ph : P.cv_bwd_b) finish_phase(ph);
  for (auto& ph : P.cv_bwd_c) finish_phase(ph);
  P.vjp_numel = std::max<int64_t>(w, kPadF32);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Per-layer conv scratch, sized now from the declared grid and max_batch so that no call allocates
// later; one private slice per layer so calls on different layers may overlap on
// different streams: [split-K flags (zeroed) | padded copy / split-K partials | BF16 weight scratch].
static void size_conv(Plan& P) {
  for (auto& L : P.layers) {
    L.pad_bytes = 0;
    L.n_flags = 0;
    if (L.cons == CONS_DENSE || P.opts.max_batch <= 0 || L.desc.grid_h <= 0 || L.desc.grid_w <= 0) continue;
    L.pad_bytes = conv_scratch_need(L, P.opts.max_batch, L.desc.grid_h, L.desc.grid_w, &L.n_flags);
  }
}

static orth_status_t allocate_conv(Plan& P) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  struct Slice { size_t flags, pad, wt, blk_h, blk_z; };
  std::vector<Slice> sl(P.layers.size());
  std::vector<std::pair<size_t, size_t>> flag_ranges;
  for (size_t l = 0; l < P.layers.size(); ++l) {
    LayerInfo& L = P.layers[l];
    sl[l] = Slice{0, 0, 0, 0, 0};
    if (L.cons == CONS_DENSE) continue;
    if (L.pad_bytes > 0) {
      const size_t fb = (size_t)std::max<int64_t>(L.n_flags, 1) * sizeof(unsigned);
      sl[l].flags = take(fb);
      flag_ranges.push_back({sl[l].flags, fb});
      sl[l].pad = take((size_t)L.pad_bytes);
    }
    // W^T of the adjoint, group-packed copies (<= 8x each, conv_tc.cu) when the layer packs groups
    const bool packs = L.g > 1 && (L.ci < 64 || L.co < 64);
    sl[l].wt = take((size_t)(packs ? 16 : 1) * L.kernel_numel * 2);
    if (L.cons == CONS_SLL_BLOCK) {   // h (c_s) and [x | h] (c + c_s) of the declared grid and batch, FP32-sized
      L.blk_scratch_bytes = (P.opts.max_batch > 0 && L.desc.grid_h > 0 && L.desc.grid_w > 0)
                                ? (int64_t)P.opts.max_batch * L.desc.grid_h * L.desc.grid_w * 4 : 0;
      sl[l].blk_h = take((size_t)L.blk_scratch_bytes * L.blk_cs + 16);
      sl[l].blk_z = take((size_t)L.blk_scratch_bytes * (L.ci + L.blk_cs) + 16);
    }
  }
  P.conv_mem_bytes = (int64_t)off;
  if (off == 0) return ORTH_OK;
  if (cudaMalloc(&P.d_conv_mem, off) != cudaSuccess) {
    cudaGetLastError();
    P.d_conv_mem = nullptr;
    set_error("conv scratch cudaMalloc(%zu bytes) failed (grid_h/grid_w x max_batch too large?)", off);
    return ORTH_ERR_OUT_OF_MEMORY;
  }
  char* base = (char*)P.d_conv_mem;
  for (auto& fr : flag_ranges)
    if (cudaMemset(base + fr.first, 0, fr.second) != cudaSuccess) {
      set_error("conv scratch memset failed");
      return ORTH_ERR_CUDA;
    }
  for (size_t l = 0; l < P.layers.size(); ++l) {
    LayerInfo& L = P.layers[l];
    if (L.cons == CONS_DENSE) continue;
    L.wt_scratch = base + sl[l].wt;
    if (L.cons == CONS_SLL_BLOCK) {
      L.blk_h = base + sl[l].blk_h;
      L.blk_z = base + sl[l].blk_z;
    }
    if (L.pad_bytes > 0) {
      L.pad_scratch = base + sl[l].pad;
      L.conv_flags = reinterpret_cast<unsigned*>(base + sl[l].flags);
    }
  }
  // conv views of every SLL block: C (c -> c_s, stride 1, top pad pC) and M (c + c_s -> c_out, stride s,
  // top pad pM), circular, sharing the block's weight scratch (no split-K / padded-copy scratch)
  P.blk_conv.clear();
  for (auto& L : P.layers) {
    if (L.cons != CONS_SLL_BLOCK) continue;
    LayerInfo c{}, m{};
    c.desc = L.desc; c.desc.kind = ORTH_CONV2D;
    c.cons = CONS_BCOP; c.g = 1; c.d = 1; c.s = 1;
    c.ci_f = c.ci = L.ci; c.co_f = c.co = L.blk_cs; c.k = L.kC;
    c.pt = c.pl = L.pC; c.pb = c.pr = L.kC - 1 - L.pC;
    c.kernel_numel = (int64_t)c.co * c.ci * c.k * c.k;
    c.wt_scratch = L.wt_scratch;
    m = c;
    m.s = L.s; m.ci_f = m.ci = L.ci + L.blk_cs; m.co_f = m.co = L.co; m.k = L.kM;
    m.pt = m.pl = L.pM; m.pb = m.pr = L.kM - 1 - L.pM;
    m.kernel_numel = (int64_t)m.co * m.ci * m.k * m.k;
    P.blk_conv.push_back(c);
    P.blk_conv.push_back(m);
  }
  return ORTH_OK;
}

static orth_status_t allocate(Plan& P) {
  if (cudaSetDevice(P.device) != cudaSuccess) {
    set_error("cudaSetDevice(%d) failed: %s", P.device, cudaGetErrorString(cudaGetLastError()));
    return ORTH_ERR_CUDA;
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + std::max<size_t>(bytes, 1), 256); return o; };
  const size_t o_scr = take(P.params_numel * 4), o_gram = take(P.gram_numel * 4), o_v = take(P.cache_numel * 4);
  const size_t o_sig = take(std::max<size_t>(P.mats.size(), 1) * 4), o_part = take(P.partial_numel * 4);
  const size_t o_comp = take(P.comp_numel * 4), o_stat = take(64);
  const size_t o_pi = take(std::max<size_t>(P.power_items.size(), 1) * sizeof(PowerItem));
  const size_t o_own = take(std::max<size_t>(P.mat_items.size(), 1) * sizeof(MatItem));
  const size_t o_ri = take(std::max<size_t>(P.res_items.size(), 1) * sizeof(ResItem));
  const size_t o_rp = take(std::max<size_t>(P.res_items.size(), 1) * sizeof(float));
  const size_t o_col = take(std::max<size_t>(P.col_items.size(), 1) * sizeof(ColItem));
  const size_t o_emit = take(std::max<size_t>(P.emit.size(), 1) * sizeof(EmitItem));
  const size_t o_nsg = take(std::max<size_t>(P.ns_gram.size(), 1) * sizeof(NsDesc));
  const size_t o_nsu = take(std::max<size_t>(P.ns_upd.size(), 1) * sizeof(NsDesc));
  const size_t o_bx = take((size_t)4 * std::max<int64_t>(P.bx_numel, 64) * 2);
  const size_t o_units = take(std::max<size_t>(P.units.size(), 1) * sizeof(UnitInfo));
  const size_t o_res = take(std::max<size_t>(P.mats.size(), 1) * 4);
  const size_t o_br = take((size_t)2 * std::max<int64_t>(P.br_numel, 64) * 2);
  std::vector<GemmPhase*> phases = {&P.gram[0], &P.gram[1], &P.update[0], &P.update[1], &P.gram_r[0],
                                    &P.gram_r[1], &P.update_r[0], &P.update_r[1], &P.proj, &P.aoc};
  for (auto& ph : P.chain) phases.push_back(&ph);
  for (auto& ph : P.soc_pow) phases.push_back(&ph);
  phases.push_back(&P.sll_v);
  phases.push_back(&P.blk_mm);
  for (auto& ph : P.vj_fwd) phases.push_back(&ph);
  for (auto& ph : P.vj_bwd) phases.push_back(&ph);
  for (auto& ph : P.cv_fwd) phases.push_back(&ph);
  for (auto& ph : P.cv_bwd_a) phases.push_back(&ph);
  for (auto& ph : P.cv_bwd_b) phases.push_back(&ph);
  for (auto& ph : P.cv_bwd_c) phases.push_back(&ph);
  phases.push_back(&P.cv_dr);
  phases.push_back(&P.cv_dkb);
  const size_t o_cvi = take(std::max<size_t>(P.cv_items.size(), 1) * sizeof(VjpItem));
  const size_t o_cvs = take(std::max<size_t>(P.cv_scatter.size(), 1) * sizeof(ScatterItem));
  const size_t o_sll = take(std::max<size_t>(P.sll.size(), 1) * sizeof(SllItem));
  const size_t o_blk = take(std::max<size_t>(P.blk.size(), 1) * sizeof(BlkItem));
  const size_t o_em2 = take(std::max<size_t>(P.emit2.size(), 1) * sizeof(EmitItem));
  const size_t o_soc = take(std::max<size_t>(P.soc.size(), 1) * sizeof(SocItem));
  const size_t o_sal = take(std::max<size_t>(P.soc.size(), 1) * sizeof(float));
  std::vector<std::pair<size_t, size_t>> ph_off;
  for (auto* ph : phases)
    ph_off.push_back({take(std::max<size_t>(ph->descs.size(), 1) * sizeof(GemmDesc)),
                      take(std::max<size_t>(ph->segs.size(), 1) * sizeof(GemmSeg))});
  P.arena_bytes = off;
  if (cudaMalloc(&P.d_arena, off) != cudaSuccess) {
    cudaGetLastError();
    set_error("workspace cudaMalloc(%zu bytes) failed", off);
    return ORTH_ERR_OUT_OF_MEMORY;
  }
  char* base = (char*)P.d_arena;
  P.d_scratch = (float*)(base + o_scr);
  P.d_gram = (float*)(base + o_gram);
  P.d_vbuf = (float*)(base + o_v);
  P.d_sigma = (float*)(base + o_sig);
  P.d_partial = (float*)(base + o_part);
  P.d_comp = (float*)(base + o_comp);
  P.d_status = (int32_t*)(base + o_stat);
  P.d_power_items = (PowerItem*)(base + o_pi);
  P.d_mat_items = (MatItem*)(base + o_own);
  P.d_res_items = (ResItem*)(base + o_ri);
  P.d_res_part = (float*)(base + o_rp);
  P.d_col_items = (ColItem*)(base + o_col);
  P.d_emit = (EmitItem*)(base + o_emit);
  P.d_ns_gram = (NsDesc*)(base + o_nsg);
  P.d_ns_upd = (NsDesc*)(base + o_nsu);
  P.d_bx = (uint16_t*)(base + o_bx);
  P.d_units = (UnitInfo*)(base + o_units);
  P.d_soc = (SocItem*)(base + o_soc);
  P.d_sll = (SllItem*)(base + o_sll);
  P.d_cv_items = (VjpItem*)(base + o_cvi);
  P.d_cv_scatter = (ScatterItem*)(base + o_cvs);
  P.d_blk = (BlkItem*)(base + o_blk);
  P.d_emit2 = (EmitItem*)(base + o_em2);
  P.d_soc_alpha = (float*)(base + o_sal);
  P.d_ns_res = (float*)(base + o_res);
  P.d_br = (uint16_t*)(base + o_br);
  cudaError_t e = cudaMemset(P.d_arena, 0, off);   // also zero-pads the BF16 operand copies
  if (!P.ns_gram.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_ns_gram, P.ns_gram.data(), P.ns_gram.size() * sizeof(NsDesc), cudaMemcpyHostToDevice);
  if (!P.ns_upd.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_ns_upd, P.ns_upd.data(), P.ns_upd.size() * sizeof(NsDesc), cudaMemcpyHostToDevice);
  if (!P.power_items.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_power_items, P.power_items.data(), P.power_items.size() * sizeof(PowerItem), cudaMemcpyHostToDevice);
  if (!P.res_items.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_res_items, P.res_items.data(), P.res_items.size() * sizeof(ResItem), cudaMemcpyHostToDevice);
  if (!P.mat_items.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_mat_items, P.mat_items.data(), P.mat_items.size() * sizeof(MatItem), cudaMemcpyHostToDevice);
  if (!P.col_items.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_col_items, P.col_items.data(), P.col_items.size() * sizeof(ColItem), cudaMemcpyHostToDevice);
  if (!P.cv_items.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_cv_items, P.cv_items.data(), P.cv_items.size() * sizeof(VjpItem), cudaMemcpyHostToDevice);
  if (!P.cv_scatter.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_cv_scatter, P.cv_scatter.data(), P.cv_scatter.size() * sizeof(ScatterItem),
                   cudaMemcpyHostToDevice);
  if (!P.sll.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_sll, P.sll.data(), P.sll.size() * sizeof(SllItem), cudaMemcpyHostToDevice);
  if (!P.blk.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_blk, P.blk.data(), P.blk.size() * sizeof(BlkItem), cudaMemcpyHostToDevice);
  if (!P.emit2.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_emit2, P.emit2.data(), P.emit2.size() * sizeof(EmitItem), cudaMemcpyHostToDevice);
  if (!P.soc.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_soc, P.soc.data(), P.soc.size() * sizeof(SocItem), cudaMemcpyHostToDevice);
  if (!P.units.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_units, P.units.data(), P.units.size() * sizeof(UnitInfo), cudaMemcpyHostToDevice);
  if (!P.emit.empty() && e == cudaSuccess)
    e = cudaMemcpy(P.d_emit, P.emit.data(), P.emit.size() * sizeof(EmitItem), cudaMemcpyHostToDevice);
  for (size_t i = 0; i < phases.size() && e == cudaSuccess; ++i) {
    GemmPhase* ph = phases[i];
    ph->d_descs = (GemmDesc*)(base + ph_off[i].first);
    ph->d_segs = (GemmSeg*)(base + ph_off[i].second);
    if (!ph->descs.empty())
      e = cudaMemcpy(ph->d_descs, ph->descs.data(), ph->descs.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice);
    if (!ph->segs.empty() && e == cudaSuccess)
      e = cudaMemcpy(ph->d_segs, ph->segs.data(), ph->segs.size() * sizeof(GemmSeg), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    set_error("plan upload failed: %s", cudaGetErrorString(e));
    cudaFree(P.d_arena);
    P.d_arena = nullptr;
    return ORTH_ERR_CUDA;
  }
  if (P.opts.vjp && P.vjp_numel > 0) {   // f1 backward workspace (separate allocation, only on request)
    if (cudaMalloc(&P.d_vjp, (size_t)P.vjp_numel * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      P.d_vjp = nullptr;
      set_error("VJP workspace cudaMalloc(%lld floats) failed", (long long)P.vjp_numel);
      return ORTH_ERR_OUT_OF_MEMORY;
    }
    cudaMemset(P.d_vjp, 0, (size_t)P.vjp_numel * sizeof(float));
  }
  return allocate_conv(P);
}

}  // namespace orth

using namespace orth;

extern "C" {

void orth_opts_default(orth_opts_t* o) {
  if (!o) return;
  o->ns_iters = 12;
  o->beta = 0.5f;
  o->prescale = ORTH_PRESCALE_POWER;
  o->power_iters = 3;
  o->compute = ORTH_F32;
  o->polish_iters = 2;
  o->rank = 0;
  o->world = 1;
  o->ns_tol = 1e-3f;
  o->max_batch = 0;
  o->vjp = 0;
}

orth_status_t orth_validate_desc(const orth_layer_desc_t* layers, int32_t n_layers, const orth_opts_t* opts) {
  if (!layers || n_layers < 1) { set_error("layers is NULL or n_layers < 1"); return ORTH_ERR_INVALID_ARGUMENT; }
  orth_opts_t o;
  orth_opts_default(&o);
  if (opts) o = *opts;
  orth_status_t st = validate_opts(o);
  if (st != ORTH_OK) return st;
  for (int i = 0; i < n_layers; ++i) {
    st = validate_layer(layers[i], i);
    if (st != ORTH_OK) return st;
  }
  for (int i = 0; i < n_layers; ++i) {   // SLL blocks: the three referenced layers (R29)
    const orth_layer_desc_t& B = layers[i];
    if (B.kind != ORTH_SLL_BLOCK) continue;
    const int r[3] = {B.blk_pre, B.blk_sll, B.blk_post};
    for (int j = 0; j < 3; ++j)
      if (r[j] < 0 || r[j] >= i) { set_error("block %d: referenced layer %d must be an earlier layer", i, r[j]); return ORTH_ERR_INVALID_ARGUMENT; }
    const orth_layer_desc_t &Pre = layers[B.blk_pre], &S = layers[B.blk_sll], &Po = layers[B.blk_post];
    const bool ok = Pre.kind == ORTH_CONV2D && Pre.c_in == B.c_in && Pre.c_out == B.c_in && Pre.stride_h == 1 &&
                    S.kind == ORTH_SLL && S.c_in == B.c_in &&
                    Po.kind == ORTH_CONV2D && Po.c_in == B.c_in && Po.c_out == B.c_out && Po.stride_h == B.stride_h &&
                    Pre.groups == 1 && Po.groups == 1 && Pre.dil_h == 1 && Po.dil_h == 1 && Pre.pad_t == -1 &&
                    Po.pad_t == -1 && Pre.padding_mode == ORTH_PAD_CIRCULAR && Po.padding_mode == ORTH_PAD_CIRCULAR;
    if (!ok) {
      set_error("block %d: needs pre = conv c->c (s 1), sll = SLL c->c_s, post = conv c->c_out (stride s), g = d = 1, "
                "circular, 'same' pads", i);
      return ORTH_ERR_INVALID_ARGUMENT;
    }
  }
  return ORTH_OK;
}

orth_status_t orth_plan_create(const orth_layer_desc_t* layers, int32_t n_layers, const orth_opts_t* opts,
                               int32_t device, orth_plan_t* plan) {
  if (!plan) { set_error("plan out-pointer is NULL"); return ORTH_ERR_INVALID_ARGUMENT; }
  *plan = nullptr;
  orth_status_t st = orth_validate_desc(layers, n_layers, opts);
  if (st != ORTH_OK) return st;
  if (device < -1) { set_error("device must be >= -1"); return ORTH_ERR_INVALID_ARGUMENT; }
  auto* h = new orth_plan();
  Plan& P = h->p;
  orth_opts_default(&P.opts);
  if (opts) P.opts = *opts;
  P.device = device;
  derive(P, layers, n_layers);
  assign_owners(P);
  layout(P);
  build_ns(P);
  build_compose(P);
  if (P.opts.vjp) build_vjp(P);
  size_conv(P);
  if (device >= 0) {
    st = allocate(P);
    if (st == ORTH_OK && P.opts.compute != ORTH_F32) st = build_compose_tc(P);
    if (st == ORTH_OK && P.opts.compute != ORTH_F32) st = build_ns_tma(P);
    if (st == ORTH_OK && P.opts.compute != ORTH_F32) st = build_ns_persist(P);
    if (st != ORTH_OK) {
      free_compose_tc(P);
      if (P.d_ns_maps) cudaFree(P.d_ns_maps);
      if (P.nsp_mem) cudaFree(P.nsp_mem);
      if (P.d_arena) cudaFree(P.d_arena);
      if (P.d_conv_mem) cudaFree(P.d_conv_mem);
      if (P.d_vjp) cudaFree(P.d_vjp);
      delete h;
      return st;
    }
  }
  *plan = h;
  return ORTH_OK;
}

orth_status_t orth_plan_destroy(orth_plan_t plan) {
  if (!plan) return ORTH_OK;
  free_compose_tc(plan->p);
  if (plan->p.d_ns_maps) cudaFree(plan->p.d_ns_maps);
  if (plan->p.nsp_mem) cudaFree(plan->p.nsp_mem);
  if (plan->p.nsf_items) cudaFree(plan->p.nsf_items);
  if (plan->p.d_arena) cudaFree(plan->p.d_arena);
  if (plan->p.d_conv_mem) cudaFree(plan->p.d_conv_mem);
  if (plan->p.d_vjp) cudaFree(plan->p.d_vjp);
  orth_plan_trace_free(plan->p);
  if (plan->p.d_ns_upd64) cudaFree(plan->p.d_ns_upd64);
  if (plan->p.d_ns_gram_flow) cudaFree(plan->p.d_ns_gram_flow);
  if (plan->p.d_ns_upd_wide) cudaFree(plan->p.d_ns_upd_wide);
  delete plan;
  return ORTH_OK;
}

orth_status_t orth_plan_query(orth_plan_t plan, int32_t what, int32_t index, int64_t* out) {
  if (!plan || !out) { set_error("NULL plan or out"); return ORTH_ERR_INVALID_ARGUMENT; }
  const Plan& P = plan->p;
  const bool lq = what >= 20 && what < 40, mq = what >= 40 && what < 60, uq = what >= 60;
  if (lq && (index < 0 || index >= (int)P.layers.size())) { set_error("layer index %d out of range", index); return ORTH_ERR_INVALID_ARGUMENT; }
  if (mq && (index < 0 || index >= (int)P.mats.size())) { set_error("matrix index %d out of range", index); return ORTH_ERR_INVALID_ARGUMENT; }
  if (uq && (index < 0 || index >= (int)P.units.size())) { set_error("unit index %d out of range", index); return ORTH_ERR_INVALID_ARGUMENT; }
  switch (what) {
    case ORTH_Q_N_LAYERS: *out = (int64_t)P.layers.size(); break;
    case ORTH_Q_N_MATRICES: *out = (int64_t)P.mats.size(); break;
    case ORTH_Q_PARAMS_NUMEL: *out = P.params_numel; break;
    case ORTH_Q_CACHE_NUMEL: *out = P.cache_numel; break;
    case ORTH_Q_KERNELS_F32_NUMEL: *out = P.kf32_numel; break;
    case ORTH_Q_KERNELS_BF16_NUMEL: *out = P.kbf16_numel; break;
    case ORTH_Q_WORKSPACE_BYTES: *out = (int64_t)P.arena_bytes; break;
    case ORTH_Q_NS_FLOPS: *out = (int64_t)P.ns_flops; break;
    case ORTH_Q_KERNEL_SEGMENT_F32: *out = P.seg_f32; break;
    case ORTH_Q_KERNEL_SEGMENT_BF16: *out = P.seg_bf16; break;
    case ORTH_Q_N_UNITS: *out = (int64_t)P.units.size(); break;
    case ORTH_Q_GATHER_F32_NUMEL: *out = P.gat_f32_numel; break;
    case ORTH_Q_GATHER_BF16_NUMEL: *out = P.gat_bf16_numel; break;
    case ORTH_Q_CONV_SCRATCH_BYTES: *out = P.conv_mem_bytes; break;
    case ORTH_Q_LAYER_SCRATCH_BYTES: *out = P.layers[index].pad_bytes; break;
    case ORTH_Q_LAYER_NS_FLOPS: *out = (int64_t)P.layers[index].ns_flops; break;
    case ORTH_Q_LAYER_COMP_FLOPS: *out = (int64_t)P.layers[index].comp_flops; break;
    case ORTH_Q_LAYER_K_EFF: *out = P.layers[index].k; break;
    case ORTH_Q_LAYER_BLOCK_KC: *out = P.layers[index].kC; break;
    case ORTH_Q_LAYER_BLOCK_M_OFF: *out = P.layers[index].m_off; break;
    case ORTH_Q_LAYER_BLOCK_PADS: *out = (int64_t)P.layers[index].pC | ((int64_t)P.layers[index].pM << 16); break;
    case ORTH_Q_COMP_FLOPS: {
      double f = 0.0;
      for (auto& u : P.units)
        if (u.owner == P.opts.rank) f += P.layers[u.layer].comp_flops / P.layers[u.layer].g;
      *out = (int64_t)f;
      break;
    }
    case ORTH_Q_UNIT_LAYER: *out = P.units[index].layer; break;
    case ORTH_Q_UNIT_GROUP: *out = P.units[index].group; break;
    case ORTH_Q_UNIT_OWNER: *out = P.units[index].owner; break;
    case ORTH_Q_UNIT_NUMEL: *out = P.units[index].numel; break;
    case ORTH_Q_UNIT_GATHER_OFF_F32: *out = P.units[index].gat_f32; break;
    case ORTH_Q_UNIT_GATHER_OFF_BF16: *out = P.units[index].gat_bf16; break;
    case ORTH_Q_UNIT_KERNEL_OFF_F32: *out = P.units[index].fin_f32; break;
    case ORTH_Q_UNIT_KERNEL_OFF_BF16: *out = P.units[index].fin_bf16; break;
    case ORTH_Q_LAYER_FIRST_MATRIX: *out = P.layers[index].first_mat; break;
    case ORTH_Q_LAYER_MATS_PER_GROUP: *out = P.layers[index].mats_per_group; break;
    case ORTH_Q_LAYER_KERNEL_OFF_F32: *out = P.layers[index].kf32_off; break;
    case ORTH_Q_LAYER_KERNEL_OFF_BF16: *out = P.layers[index].kbf16_off; break;
    case ORTH_Q_LAYER_KERNEL_NUMEL: *out = P.layers[index].kernel_numel; break;
    case ORTH_Q_LAYER_OWNER: *out = P.layers[index].owner; break;
    case ORTH_Q_LAYER_C_MID: *out = P.layers[index].c_mid; break;
    case ORTH_Q_LAYER_C_B: *out = P.layers[index].c_b; break;
    case ORTH_Q_LAYER_KP: *out = P.layers[index].kp; break;
    case ORTH_Q_MATRIX_ROWS: *out = P.mats[index].m; break;
    case ORTH_Q_MATRIX_COLS: *out = P.mats[index].n; break;
    case ORTH_Q_MATRIX_OFFSET: *out = P.mats[index].off; break;
    case ORTH_Q_MATRIX_CACHE_OFFSET: *out = P.mats[index].cache_off; break;
    case ORTH_Q_MATRIX_LAYER: *out = P.mats[index].layer; break;
    case ORTH_Q_MATRIX_GROUP: *out = P.mats[index].group; break;
    case ORTH_Q_MATRIX_ROLE: *out = P.mats[index].role; break;
    default: set_error("unknown query %d", what); return ORTH_ERR_INVALID_ARGUMENT;
  }
  return ORTH_OK;
}

int64_t orth_plan_launch_count(orth_plan_t plan) { return plan ? plan->p.launches : 0; }

const char* orth_status_string(orth_status_t s) {
  switch (s) {
    case ORTH_OK: return "ORTH_OK";
    case ORTH_ERR_INVALID_ARGUMENT: return "ORTH_ERR_INVALID_ARGUMENT";
    case ORTH_ERR_UNSUPPORTED_CONFIG: return "ORTH_ERR_UNSUPPORTED_CONFIG";
    case ORTH_ERR_SHAPE_MISMATCH: return "ORTH_ERR_SHAPE_MISMATCH";
    case ORTH_ERR_ZERO_NORM: return "ORTH_ERR_ZERO_NORM";
    case ORTH_ERR_NOT_CONVERGED: return "ORTH_ERR_NOT_CONVERGED";
    case ORTH_ERR_CUDA: return "ORTH_ERR_CUDA";
    case ORTH_ERR_OUT_OF_MEMORY: return "ORTH_ERR_OUT_OF_MEMORY";
    case ORTH_ERR_NO_DEVICE: return "ORTH_ERR_NO_DEVICE";
  }
  return "ORTH_ERR_UNKNOWN";
}

const char* orth_last_error(void) { return orth::g_err; }

const char* orth_build_info(void) {
#ifdef ORTH_EXPERIMENTAL
  return "sm_100a experimental=1";
#else
  return "sm_100a experimental=0";
#endif
}

}  // extern "C"
