// Internal plan structures shared by the host planner (plan.cpp) and the CUDA
// translation units.  Not part of the ABI (include/orth.h is).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/orth.h"

struct CUtensorMap_st;   // cuda.h (TMA descriptors), forward-declared for the launcher prototypes

namespace orth {

enum Role : int32_t { ROLE_Q = 0, ROLE_U = 1, ROLE_R = 2, ROLE_W = 3, ROLE_K = 4 };
enum Construct : int32_t { CONS_BCOP = 0, CONS_RKO = 1, CONS_AOC = 2, CONS_DENSE = 3, CONS_SOC = 4, CONS_SLL = 5,
                           CONS_SLL_BLOCK = 6 };
enum BufId : int32_t { BUF_NONE = -1, BUF_X = 0, BUF_Y = 1, BUF_G = 2, BUF_W = 3, BUF_COUNT = 4 };

constexpr int kPadF32 = 32;    // 128 B alignment of every packed float object
constexpr int kPadBF16 = 64;   // 128 B alignment of every packed bf16 object

inline int64_t pad_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct MatInfo {
  int32_t layer, group, role;
  int64_t m, n;
  int64_t off;        // float offset in params / ortho / scratch
  int64_t cache_off;  // float offset in power cache / v workspace
  int64_t gram_off;   // float offset of its short-side Gram in the G workspace
  int64_t bx_off;     // bf16 offset in the X / X^T copies (tensor-core NS)
  int64_t br_off;     // bf16 offset in the R copies
  int32_t owned;      // 1 if this rank orthogonalises it (its unit's owner)
};

struct LayerInfo {
  orth_layer_desc_t desc;
  int32_t cons;                 // Construct
  int32_t ci_f, co_f;           // forward-conv channels (swapped for transposed, R13)
  int32_t ci, co;               // per group
  int32_t k, s, d, g;
  int32_t pt, pb, pl, pr;
  int32_t kp, c_b, c_mid;
  int32_t k_free, soc_terms;    // ORTH_SOC: free kernel size and series order (k = k_eff for the conv)
  // ORTH_SLL_BLOCK: referenced layers, merged kernel sizes / top pads, offset of M in the kernel region,
  // index of its two conv views in Plan::blk_conv (2 * blk_id: C, 2 * blk_id + 1: M), scratch for h and [x | h]
  int32_t blk_pre = -1, blk_sll = -1, blk_post = -1, blk_id = -1, blk_cs = 0;
  int32_t kC = 0, kM = 0, pC = 0, pM = 0;
  int64_t m_off = 0;
  void* blk_h = nullptr;
  void* blk_z = nullptr;
  int64_t blk_scratch_bytes = 0;
  int32_t first_mat, mats_per_group;
  int32_t owner;                // owner of group 0 (ORTH_Q_LAYER_OWNER)
  int32_t first_unit;           // units [first_unit, first_unit + g) of Plan::units
  int64_t kf32_off, kbf16_off, kernel_numel;   // final layout (contiguous layer)
  // this layer's private conv scratch, sized at create from (grid_h, grid_w, max_batch):
  void* pad_scratch = nullptr;  // padded input copy, or split-K partial tiles of the gather conv
  int64_t pad_bytes = 0;
  int64_t n_flags = 0;
  unsigned* conv_flags = nullptr;   // split-K tile flags (zeroed at create; each launch leaves them zero)
  void* wt_scratch = nullptr;   // BF16 transposed / group-packed weights of one call
  double ns_flops, comp_flops;
};

// One construction unit (layer, group) -- the sharding unit.
struct UnitInfo {
  int32_t layer, group, owner, pad_;
  int64_t numel;                  // kernel elements of the unit
  int64_t gat_f32, gat_bf16;      // gather layout (rank-major equal segments)
  int64_t fin_f32, fin_bf16;      // final layout
};

// D[M x N] (+)= alpha * sum_seg opA(seg)[M x K] * opB(seg)[K x N] + beta * C.
// Element (i,k) of A at bufs[a_buf][a_off + i*sa_m + k*sa_k] (minus the same
// element of A2 when a2_off >= 0).  Offsets are relative to base pointers the
// kernel receives, so descriptors are built once at plan creation.
struct GemmSeg {
  int64_t a_off, a2_off, b_off;
};
struct GemmDesc {
  int32_t M, N, K;
  int32_t a_buf, b_buf, c_buf, d_buf;
  int64_t sa_m, sa_k, sb_k, sb_n;
  int64_t c_off, ldc, d_off, ldd;
  float alpha, beta;
  float diag;           // added on the diagonal of D (residual-form Gram R = I - X^T X)
  int32_t seg_begin, seg_count;
  int32_t tile_begin;   // first global tile of this problem (SIMT 64x64 tiles)
  int32_t tiles_n;      // tiles along N
  int32_t tc_tile_begin;  // same for the tensor-core kernel (128 x 128 tiles)
  int32_t tc_tiles_n;
};

struct GemmPhase {        // one launch: a batch of independent problems
  std::vector<GemmDesc> descs;
  std::vector<GemmSeg> segs;
  int32_t total_tiles = 0;
  int32_t tc_total_tiles = 0;
  // device copies (inside the plan's descriptor arena)
  GemmDesc* d_descs = nullptr;
  GemmSeg* d_segs = nullptr;
};

// Tensor-core NS problem (ns_tc.cu).  Operands are BF16 copies of X, X^T and
// R = I - Gram kept in plan workspace (row stride padded to 8 elements, so
// every row is 16-byte aligned and zero-padded), written by the previous
// phase's epilogue.  kinds: 0 = X (m x n), 1 = X^T (n x m), 2 = R (s x s).
struct NsDesc {
  int32_t M, N, K;
  int32_t a_kind, b_kind;   // 0: rows of X, 1: columns of X (MN-major), 2: rows of R
  int32_t epi;              // 0: Gram epilogue (bf16 R, fp32 R on request), 1: update epilogue (X' fp32 + bf16 X')
  int64_t a_off, lda, b_off, ldb;
  int64_t f_off, ldf;       // fp32 offset/ld of D (and C for the update)
  int64_t bx_off;           // offset of this matrix in the bf16 X buffers
  int64_t br_off;           // offset of this matrix in the bf16 R buffers
  int32_t ldx, ldxt, ldr;   // padded bf16 leading dims: pad8(n), pad8(m), pad8(s)
  float alpha, beta, diag;
  int32_t tile_begin, tiles_n;
  int32_t map_a, map_b;     // TMA tensor maps: maps[map_x + 2 * parity + lo]
};

// persistent NS (ns_persist.cu): one tile of a phase, and a group of CTAs
// that owns a set of matrices for all 2T phases
struct NsTile {
  int32_t desc, local;      // matrix index (ns_gram / ns_upd), tile index inside the matrix
};
struct NsGroup {           // per CTA: its barrier group and its own tile ranges (LPT-assigned on the host)
  int32_t gid, G;           // group index (barrier counter), CTAs in the group
  int32_t g_begin, g_end;   // Gram tiles [g_begin, g_end) of the tile array
  int32_t u_begin, u_end;   // update tiles
};
constexpr int kNspMaxPhases = 132;   // 2T + 1 for T <= 65
struct NsItem {           // dataflow NS: one (phase, matrix, tile) work item, in claim order
  int32_t p, desc, local;   // phase index (flags), matrix (ns_gram / ns_upd index), tile in the matrix
  int32_t wait_ctr;         // counter that must reach wait_target before the tile's operands are read (-1: none)
  uint32_t wait_target;
  int32_t done_ctr;         // counter bumped when the tile's outputs are visible
  int32_t pad_[2];
};

struct PowerItem {        // row block of the pre-scaling / scale kernels: rows [r0, r1) of matrix `mat`
  int32_t mat, r0, r1, chunk;   // chunk: global row-item slot (|t|^2 partial)
  int32_t n, m, midx, pad_;     // midx: index into mat_items
  int64_t off, cache_off, bx_off, t_off;   // t_off: the matrix's rows in the t buffer
};

struct ColItem {          // column block of the power kernel: w[c0:c1] = (W^T u)[c0:c1]
  int32_t mat, c0, c1, chunk;   // chunk: global column-item slot (|w|^2 partial)
  int32_t n, m, midx, pad_;
  int64_t off, cache_off, t_off;
};

struct MatItem {          // one owned, non-empty matrix (power finalize / residual kernels)
  int32_t mat, m, n, chunk0, nchunks, col0, ncols, res0;   // row items [chunk0, +nchunks), column items [col0, +ncols)
  int32_t nres, pad_[3];    // residual items [res0, res0 + nres)
  int64_t off, cache_off, gram_off, t_off;
};

struct ResItem {          // one slice [e0, e1) of a matrix's s x s Gram / R (residual reduction, stage 1)
  int32_t midx, pad_;
  int64_t e0, e1;
};

struct EmitItem {         // one (layer, group): copy the unit kernel into both layouts
  int32_t layer, group;
  int32_t src_buf;          // BUF_* base of the source
  int64_t src_off;
  int32_t mode;             // 0 tap-major (tap stride, ld), 1 RKO reshape
  int64_t tap_stride, ld;
  int32_t co, ci, k, s;
  int64_t f32_off, bf16_off; // of the group's first output channel
  int32_t ci_f_per_g;        // == ci
};

// One BCOP/AOC construction unit (layer, group) of the composition workspace.
struct CompUnit {
  int layer, group;
  int64_t ping, pong, fin;   // float offsets in the comp workspace (-1: none)
  int rows, c;               // chain tap = rows x c (row subset when only [:co] is kept)
};

// f3: one SOC unit (layer, group) of the explicit-exponential construction (soc.cu).  Offsets are floats
// in the composition workspace (tap-major c x c matrices), except src_off (ortho / params).
constexpr int kSocMaxTerms = 16;
struct SocItem {
  int32_t c, k, kn, terms;        // width, free kernel size, k_eff, series order
  int32_t alpha_slot, pad_[3];
  int64_t src_off;                // free kernel (PyTorch layout (c, c, k, k)) in ortho
  int64_t e_off;                  // E (kn^2 taps)
  int64_t u_off[kSocMaxTerms + 1];   // u_off[1] = S (skew part), u_off[j] = S^(*)j, j >= 2 (u_off[2] always)
};

// f4 (sll.cu): AOL rescale of one SLL unit; offsets in the composition workspace except src_off (ortho)
struct SllItem {
  int32_t ci, co, k, pad_;
  int64_t src_off;      // free kernel W (co, ci, k, k) in ortho
  int64_t v_off;        // V[Delta] = sum_t W_t^T W_{t+Delta}: (2k-1)^2 taps of ci x ci
  int64_t s_off;        // per-input-channel scale d_i^{-1/2} (ci floats)
  int64_t kt_off;       // rescaled kernel, tap-major k^2 x co x ci
};
// f4: one SLL x AOC block: M = [A | -2 B] from the A / B products (comp workspace)
struct BlkItem {
  int32_t c, cs, co, kA, kB, kM, oa, ob;
  int64_t a_off, b_off, m_off, c_off;   // A, B, M, C (tap-major) in comp
};

// f1 (vjp.cu): per-unit gradient moves of the composition VJP
struct VjpItem {
  int32_t mode;           // 0 chain unit: dS_last[t][o][i] = (i < ci) dK[o][i][t] (rows x c); 1 AOC: dFin[t][o][i];
                          // 2 copy (RKO / dense: d_ortho slab = dK slab); 3 BCOP k' = 1: dQ[:co, :ci] = dK
  int32_t co, ci, kk, rows, c, pad_[2];
  int64_t src_off;        // dK (final FP32 layout) of the unit
  int64_t dst_off;        // mode 0/1: VJP arena; mode 2/3: d_ortho
  int64_t zero_off, zero_n;   // d_ortho region zeroed first (dQ of chain units), -1 none
};
struct ScatterItem {      // AOC dR: dR[o][j s^2 + t] = dRab[t][o][j]
  int32_t co, cm, ss, pad_;
  int64_t src_off, dst_off;   // arena, d_ortho
};

struct TcComposePlan;   // tensor-core composition (compose_tc.cu)
}  // namespace orth
struct orth_trace_state;   // abi.cu (orth_plan_trace)
namespace orth {

struct Plan {
  std::vector<LayerInfo> layers;
  std::vector<UnitInfo> units;
  UnitInfo* d_units = nullptr;       // device copy (orth_kernels_assemble)
  int64_t gat_f32_numel = 0, gat_bf16_numel = 0;
  std::vector<CompUnit> comp_units;
  std::vector<int64_t> proj_off;     // per matrix: float offset of P = U U^T in comp (U only)
  TcComposePlan* tcc = nullptr;
  std::vector<MatInfo> mats;
  orth_opts_t opts;
  int32_t device = -1;

  int64_t params_numel = 0, cache_numel = 0, gram_numel = 0;
  int64_t kf32_numel = 0, kbf16_numel = 0, seg_f32 = 0, seg_bf16 = 0;
  int64_t comp_numel = 0;          // chain / projector / final workspace floats
  int64_t partial_numel = 0;
  int32_t n_chunks = 0;
  double ns_flops = 0.0;

  // NS phases (built once): gram and update per parity of the X buffer
  GemmPhase gram[2], update[2];     // [0]: X in BUF_X -> out BUF_Y ; [1]: X in BUF_Y -> out BUF_X
  // residual form for the tensor-core path: R = I - Gram(X); X' = X + beta * (X R | R X)
  GemmPhase gram_r[2], update_r[2];
  // tensor-core NS on BF16 operand copies (ns_tc.cu)
  std::vector<NsDesc> ns_gram, ns_upd;
  int32_t ns_gram_tiles = 0, ns_upd_tiles = 0;
  int64_t ns_upd_tiles_all = 0;     // over all ranks' matrices (schedule choice, bitwise-stable sharding)
  NsDesc* d_ns_gram = nullptr;
  NsDesc* d_ns_upd = nullptr;
  std::vector<NsDesc> ns_upd64;     // dataflow NS: the update descriptors with 64-wide tiles (epi = 2)
  NsDesc* d_ns_upd64 = nullptr;
  std::vector<NsDesc> ns_upd_wide;  // phase-synchronous NS: update descriptors (epi = 4: 128 x 256 tiles)
  NsDesc* d_ns_upd_wide = nullptr;
  std::vector<NsDesc> ns_gram_flow; // dataflow NS: Gram descriptors (epi = 3: full, non-symmetric)
  NsDesc* d_ns_gram_flow = nullptr;
  int64_t bx_numel = 0, br_numel = 0;
  uint16_t* d_bx = nullptr;         // 4 x bx_numel: Xh[2], Xl[2] (row-major, rows padded to 8)
  uint16_t* d_br = nullptr;         // 2 x br_numel: Rh, Rl
  void* d_ns_maps = nullptr;        // CUtensorMap array of the NS operands (separate allocation)
  int* d_ns_tile_gram = nullptr;    // tile -> problem tables (inside the d_ns_maps allocation)
  int* d_ns_tile_upd = nullptr;
  // persistent NS (all phases in one cooperative launch); nsp_ctas == 0: unavailable
  void* nsp_mem = nullptr;
  NsTile* nsp_tiles = nullptr;
  NsGroup* nsp_groups = nullptr;
  unsigned* nsp_bars = nullptr;
  int32_t nsp_ctas = 0, nsp_groups_n = 0;
  double nsp_est_us = 0.0;
  // dataflow NS items for the last phase list used (rebuilt when the list changes)
  NsItem* nsf_items = nullptr;
  int32_t nsf_n_items = 0, nsf_nphases = -1;
  std::vector<uint8_t> nsf_flags;
  int32_t nsp_zero_n = 0;           // words of nsp_bars the scale kernel zeroes before every launch
  // (group barriers of the phase-synchronous kernel, or the dataflow kernel's
  //  [claim][gram done, update done] x matrices counters)
  std::vector<PowerItem> power_items;
  std::vector<ColItem> col_items;
  ColItem* d_col_items = nullptr;
  int64_t t_numel = 0;              // sum of rows: the power kernel's t = W v buffer
  std::vector<int32_t> owned_mats;  // indices of owned, non-empty matrices
  std::vector<MatItem> mat_items;   // same order as owned_mats
  std::vector<ResItem> res_items;
  ResItem* d_res_items = nullptr;
  float* d_res_part = nullptr;      // one partial sum of squares per residual item

  // composition phases
  GemmPhase proj;                   // P_j = U_j U_j^T
  std::vector<GemmPhase> chain;     // 2(k'-1) substeps, batched over units
  GemmPhase aoc;                    // RKO (*) BCOP
  std::vector<EmitItem> emit;
  std::vector<SocItem> soc;         // f3 units owned by this rank
  std::vector<GemmPhase> soc_pow;   // soc_pow[j - 2]: S^(*)j = S^(*)(j-1) (*) S, batched over units
  std::vector<int64_t> soc_copy;    // (offset, numel) pairs of owned SOC free kernels (params -> ortho)
  SocItem* d_soc = nullptr;
  float* d_soc_alpha = nullptr;
  std::vector<SllItem> sll;         // f4
  GemmPhase sll_v;                  // V of every SLL unit
  std::vector<BlkItem> blk;
  GemmPhase blk_mm;                 // C, A, B of every block (read the emitted FP32 kernels: BUF_Y)
  std::vector<LayerInfo> blk_conv;  // conv views of every block: [C, M] per block
  std::vector<EmitItem> emit2;      // the blocks' C and M (after the first emit)
  // f1 VJP (opts.vjp != 0): arena, NS iterate storage, composition VJP phases
  float* d_vjp = nullptr;
  int64_t vjp_numel = 0;
  int64_t vj_x_off = 0, vj_g_off[2] = {0, 0}, vj_r_off = 0, vj_s_off = 0;
  std::vector<GemmPhase> vj_fwd;    // per t: [2t] R_t = I - Gram(X_t), [2t+1] X_{t+1} = X_t + b (X_t R_t | R_t X_t)
  std::vector<GemmPhase> vj_bwd;    // per t (reverse): [2j] {R_t, S'_t}, [2j+1] G_t from G_{t+1}
  int32_t vj_g_final = 0;           // 0/1: which G slot holds G_0 (-1: d_ortho itself when T == 0)
  std::vector<GemmPhase> cv_fwd;    // chain steps into per-step buffers
  GemmPhase cv_dr, cv_dkb;          // AOC: dR_ab, dKb
  std::vector<GemmPhase> cv_bwd_a, cv_bwd_b, cv_bwd_c;   // per backward iteration: {dP, dK_in}, {dP U}, {+dP^T U}
  std::vector<int64_t> cv_qcopy;    // (ortho off, arena off, floats) triples: Q rows copied into the arena
  int64_t cv_zero_off = 0, cv_zero_n = 0;
  std::vector<VjpItem> cv_items;
  std::vector<ScatterItem> cv_scatter;
  VjpItem* d_cv_items = nullptr;
  ScatterItem* d_cv_scatter = nullptr;
  bool vjp_supported = true;        // false if an owned unit is SOC / SLL / block (no VJP)
  SllItem* d_sll = nullptr;
  BlkItem* d_blk = nullptr;
  EmitItem* d_emit2 = nullptr;
  int64_t comp_proj_off = 0, comp_ping_off = 0, comp_pong_off = 0, comp_final_off = 0;

  // device allocations
  void* d_arena = nullptr;          // one cudaMalloc for everything
  size_t arena_bytes = 0;
  float* d_scratch = nullptr;       // NS ping-pong partner (params_numel)
  float* d_gram = nullptr;
  float* d_vbuf = nullptr;
  float* d_sigma = nullptr;
  float* d_partial = nullptr;       // power kernel: [t (t_numel) | |t|^2 per row item | |w|^2 per column item]
  float* d_comp = nullptr;
  int32_t* d_status = nullptr;
  PowerItem* d_power_items = nullptr;
  MatItem* d_mat_items = nullptr;
  EmitItem* d_emit = nullptr;
  int64_t partial_stride = 0;
  int64_t launches = 0;
  void* d_conv_mem = nullptr;       // every layer's conv scratch (one allocation at create)
  int64_t conv_mem_bytes = 0;
  float* d_ns_res = nullptr;        // per-matrix residual of the last iteration's Gram (convergence check)
  orth_trace_state* trace = nullptr;
};

void set_error(const char* fmt, ...);

// Which conv kernel the last conv launcher on this thread used (orth_conv_variant_t of orth.h); the ABI
// copies it into the trace record of the call.
extern thread_local int g_conv_variant;

// kernel launchers (CUDA translation units); return 0 or a cudaError_t value
int launch_gemm_f32(const GemmPhase& ph, float* const bufs[BUF_COUNT], void* stream);
// tensor-core batched GEMM: BF16 operands converted from FP32 on load, FP32
// accumulation in TMEM; npass = 1 (bf16) or 3 (hi*hi + hi*lo + lo*hi split)
int launch_gemm_tc(const GemmPhase& ph, float* const bufs[BUF_COUNT], int npass, void* stream);
int launch_residual_r(Plan& p, float* residual_out, void* stream);
// tensor-core NS phase on the BF16 copies.  par: parity of the current X
// (0: BUF_X, 1: BUF_Y).  gram: Gram (else update).  npass 1|3.  write_lo:
// the epilogue also writes the lo halves of its BF16 outputs.
int launch_ns_tc(Plan& p, float* const bufs[BUF_COUNT], int par, bool gram, int npass, bool write_lo, bool write_f,
                 void* stream);
// tensor-core stem (ci = 3, k = 3 | 4, co in {32, 64, 128}); -1 = not applicable
int launch_conv_fwd_stem(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                         int H, int W, int Ho, int Wo, void* stream);
// shared by the TMA-window conv kernels (conv_pad.cu): SM count, 4-D SWIZZLE_128B activation map
// (C, W, H, N) with box 64 ch x bw px x bh rows x 1 image (cached per pointer/shape)
int conv_sm_count();
bool conv_act_tmap(::CUtensorMap_st* out, const void* x, int C, int W, int H, int N, int bw, int bh);
// stride-1 forward conv, >= 128 output channels per group: images stacked into one padded-row
// window stream, tcgen05 M = 128 channels x N = 256 window pixels (conv_stack.cu); -1 = not applicable
int launch_conv_fwd_stack(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                          int H, int W, int Ho, int Wo, void* stream, int flip = 0);
// padded copy of a layer input into the plan's conv scratch (conv_stack.cu); -1 = does not fit
int launch_pad_input(const LayerInfo& L, const void* x, int N, int H, int W, int Hp, int P, void* stream);
// stride-1 forward conv as an implicit GEMM whose A tiles are single 4-D TMA boxes of the padded input
// (conv_tma.cu): M = 128 output pixels (NI images x TH rows x Wo), N = BN channels; -1 = not applicable
int launch_conv_fwd_tma(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                        int H, int W, int Ho, int Wo, void* stream, int flip = 0);
// forward conv over TMA-loaded padded row windows (stride 1, rows <= 128 px); -1 = not applicable.
// flip = 1 reads weight tap t from row k^2-1-t (a stride-1 adjoint in its forward-conv form).
int launch_conv_fwd_reuse(const LayerInfo& L, const void* kernel, const float* bias, const void* x, void* y, int N,
                          int H, int W, int Ho, int Wo, void* stream, int flip = 0);
// persistent NS: build the CTA-group partition (after build_ns_tma); launch all
// phases (flags per phase: bit0 gram, bit1 3-pass, bit2 X parity, bit3 write lo,
// bit4 write fp32 R)
orth_status_t build_ns_persist(Plan& p);
int launch_ns_persist(Plan& p, float* const bufs[BUF_COUNT], const uint8_t* flags, int nphases, void* stream);
// X0 = W / sigma (fp32) plus its row-major BF16 copies (hi, and lo if write_lo)
int launch_scale_bf16(Plan& p, const float* W, float* X0, int par, bool write_lo, void* stream);
// tensor-core composition: built after the workspace exists; freed with the plan
orth_status_t build_compose_tc(Plan& p);
orth_status_t build_ns_tma(Plan& p);   // tensor maps of the NS operand copies; freed in destroy
void free_compose_tc(Plan& p);
int launch_compose_tc(Plan& p, const float* ortho, void* stream);   // fills comp (fp32) like the SIMT chain
int launch_scale(Plan& p, const float* W, float* X0, void* stream);
// all power iterations (or the Frobenius pass) in one cooperative launch
int launch_power_fused(Plan& p, const float* W, const float* v_in, int use_const_v, int frob, int iters,
                       float* cache_out, void* stream);
// the fused power kernel's grid-barrier counter (a word of the status block; re-armed by the scale kernels)
inline unsigned* power_bar(Plan& p) { return reinterpret_cast<unsigned*>(p.d_status + 8); }
int launch_residual(Plan& p, float* residual_out, void* stream);
// convergence check: r = |R|_F of the last iteration's FP32 R (is_r) or |I - G|_F (SIMT Gram);
// NOT_CONVERGED when r is non-finite or 3/4 r^2 + 1/4 r^3 > tol (tol > 0)
int launch_converged_check(Plan& p, int is_r, float tol, void* stream);
void orth_plan_trace_free(Plan& p);   // abi.cu
// f2: spectral certificate (certify.cu); workspace bytes (-1: not applicable) and the launch
int64_t certify_workspace_bytes(const LayerInfo& L, int H, int W);
int launch_certify(const LayerInfo& L, const float* kernel, int H, int W, int iters, void* ws, double* out,
                   void* stream);
// f3 (soc.cu): skew part, AOL scalar, series sum (the powers are GemmPhases)
int launch_soc_skew(Plan& p, const float* ortho, void* stream);
int launch_soc_alpha(Plan& p, void* stream);
int launch_soc_sum(Plan& p, void* stream);
// f4 (sll.cu)
int launch_sll_scale(Plan& p, const float* ortho, void* stream);   // d_i -> s_i, then the rescaled tap-major kernel
int launch_blk_merge(Plan& p, void* stream);                 // M = [A | -2 B]
int launch_emit_list(Plan& p, const std::vector<EmitItem>& items, const EmitItem* d_items,
                     const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream);
int launch_relu_concat(const void* x, const void* h, void* z, int64_t pixels, int c, int cs, int io, void* stream);
// f1 (wgrad.cu): conv weight gradient; workspace bytes for the split partials (0: none needed)
int64_t wgrad_workspace_bytes(const LayerInfo& L, int N, int Ho, int Wo, int io);
int launch_wgrad(const LayerInfo& L, const void* x, const void* dy, float* dK, int N, int H, int W, int Ho, int Wo,
                 int io, void* ws, int64_t ws_bytes, void* stream);
// f1 (vjp.cu)
int launch_vjp_deemit(Plan& p, const float* dK, float* dortho, void* stream);
int launch_vjp_scatter(Plan& p, float* dortho, void* stream);
// a8: copy every unit from the gather layout to the final layout
int launch_assemble(Plan& p, const float* gf, float* kf, const uint16_t* gb, uint16_t* kb, void* stream);
// per-layer conv scratch (bytes) for calls up to N x Hbig x Wbig (forward-conv input grid), both
// directions: max(padded input copy of the TMA-window kernels, split-K partials); flags: tile flags
int64_t conv_scratch_need(const LayerInfo& L, int N, int Hbig, int Wbig, int64_t* flags);
// padded-copy bytes the stacked-window kernel would use for this forward-view call (0: not taken)
int64_t conv_stack_pad_bytes(const LayerInfo& L, int N, int H, int W, int Ho, int Wo);
int launch_emit(Plan& p, const float* const bufs[BUF_COUNT], float* kf32, uint16_t* kbf16, void* stream);
int launch_conv_fwd(const LayerInfo& L, const void* kernel, void* scratch, const float* bias, const void* x, void* y,
                    int N, int H, int W, int Ho, int Wo, int io, void* stream);
bool conv_fwd_tc_eligible(const LayerInfo& L);
int launch_conv_fwd_tc(const LayerInfo& L, const void* kernel, void* scratch, const float* bias, const void* x,
                       void* y, int N, int H, int W, int Ho, int Wo, void* stream);
int launch_conv_bwd(const LayerInfo& L, const void* kernel, void* wt_scratch, const float* bias, const void* y,
                    void* x, int N, int H, int W, int Ho, int Wo, int io, void* stream);
bool conv_bwd_tc_eligible(const LayerInfo& L);
int launch_conv_bwd_tc(const LayerInfo& L, const void* kernel, void* wt_scratch, const float* bias, const void* y,
                       void* x, int N, int H, int W, int Ho, int Wo, void* stream);

}  // namespace orth

struct orth_plan {
  orth::Plan p;
};
