// Compute entry points of the C ABI (include/orth.h).  Each validates
// synchronously, then enqueues its kernels on the caller's stream.
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdlib>
#include <vector>

#include "orth_internal.h"

using namespace orth;

// tracing state of a plan (orth_plan_trace): event pairs of the groups recorded since the last read
struct orth_trace_state {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Pending { orth_trace_rec_t rec; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

namespace orth {
void orth_plan_trace_free(Plan& p) {
  if (!p.trace) return;
  for (auto e : p.trace->pool) cudaEventDestroy(e);
  for (auto& r : p.trace->pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  delete p.trace;
  p.trace = nullptr;
}
}  // namespace orth

namespace {

orth_trace_state& tstate(Plan& P) {
  if (!P.trace) P.trace = new orth_trace_state();
  return *P.trace;
}

// NVTX range of one ABI call (always on; free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// One traced group of kernels: events around it on the call's stream when tracing is on.
struct Trace {
  Plan& P;
  int kind, layer;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  int64_t l0;
  Trace(Plan& p, int k, int lay, void* stream) : P(p), kind(k), layer(lay), s((cudaStream_t)stream), l0(p.launches) {
    g_conv_variant = 0;
    if (P.trace && P.trace->on) {
      a = P.trace->get();
      cudaEventRecord(a, s);
    }
  }
  ~Trace() {
    if (!a) return;
    cudaEvent_t b = P.trace->get();
    cudaEventRecord(b, s);
    orth_trace_rec_t r{kind, layer, (kind == ORTH_TK_CONV_FWD || kind == ORTH_TK_CONV_ADJ) ? g_conv_variant : 0,
                       (int32_t)(P.launches - l0), 0.f};
    P.trace->pending.push_back({r, a, b});
  }
};

orth_status_t cuda_fail(int e, const char* where) {
  if (e == 0) return ORTH_OK;
  set_error("%s: %s", where, cudaGetErrorString((cudaError_t)e));
  return ORTH_ERR_CUDA;
}

orth_status_t need_device(orth_plan_t plan) {
  if (!plan) { set_error("NULL plan"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (plan->p.device < 0) { set_error("host-only plan (device = -1) cannot compute"); return ORTH_ERR_NO_DEVICE; }
  return ORTH_OK;
}

int out_dim(int H, int k, int s, int d, int p0, int p1) { return (H + p0 + p1 - d * (k - 1) - 1) / s + 1; }

orth_status_t check_conv(Plan& P, int32_t layer, const void* kernel, const void* in, void* out, int N, int H, int W,
                         int io, int& Ho, int& Wo) {
  if (layer < 0 || layer >= (int)P.layers.size()) { set_error("layer %d out of range", layer); return ORTH_ERR_INVALID_ARGUMENT; }
  const LayerInfo& L = P.layers[layer];
  if (L.cons == CONS_DENSE) { set_error("dense layers have no conv forward (plain GEMM, out of scope)"); return ORTH_ERR_UNSUPPORTED_CONFIG; }
  // an empty batch (N = 0) is a valid no-op: its activation pointers may be NULL
  if (!kernel || (N != 0 && (!in || !out))) { set_error("NULL kernel/input/output"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (io != ORTH_F32 && io != ORTH_BF16) { set_error("bad io dtype %d", io); return ORTH_ERR_INVALID_ARGUMENT; }
  if (N < 0 || H < 1 || W < 1) { set_error("N >= 0, H, W >= 1 required"); return ORTH_ERR_SHAPE_MISMATCH; }
  if ((int64_t)N * (H + L.pt + L.pb) * (W + L.pl + L.pr) >= (1LL << 31)) {
    set_error("N*H*W (padded) must stay below 2^31 (32-bit pixel indices)");
    return ORTH_ERR_SHAPE_MISMATCH;
  }
  const int num = H + L.pt + L.pb - L.d * (L.k - 1) - 1, numw = W + L.pl + L.pr - L.d * (L.k - 1) - 1;
  if (num < 0 || numw < 0) { set_error("input %dx%d smaller than the dilated kernel", H, W); return ORTH_ERR_SHAPE_MISMATCH; }
  Ho = out_dim(H, L.k, L.s, L.d, L.pt, L.pb);
  Wo = out_dim(W, L.k, L.s, L.d, L.pl, L.pr);
  if (L.desc.padding_mode == ORTH_PAD_CIRCULAR && (H % L.s || W % L.s)) {
    set_error("circular padding needs s | H and s | W (s=%d, H=%d, W=%d; reading R11)", L.s, H, W);
    return ORTH_ERR_SHAPE_MISMATCH;
  }
  if (((uintptr_t)in | (uintptr_t)out | (uintptr_t)kernel) & 15) { set_error("buffers must be 16-byte aligned"); return ORTH_ERR_INVALID_ARGUMENT; }
  return ORTH_OK;
}

}  // namespace

extern "C" {

orth_status_t orth_orthogonalize(orth_plan_t plan, const float* params, float* ortho_out, float* power_cache,
                                 float* residual_out, void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  if (!params || !ortho_out) { set_error("NULL params or ortho_out"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (params == ortho_out) { set_error("params and ortho_out must not overlap"); return ORTH_ERR_INVALID_ARGUMENT; }
  NvtxRange nv("orth_orthogonalize");
  // SOC free kernels (role K) pass through unchanged: orth_compose_kernel reads every unit from ortho
  for (size_t i = 0; i + 1 < P.soc_copy.size(); i += 2) {
    const cudaError_t ce = cudaMemcpyAsync(ortho_out + P.soc_copy[i], params + P.soc_copy[i],
                                           (size_t)P.soc_copy[i + 1] * sizeof(float), cudaMemcpyDeviceToDevice,
                                           (cudaStream_t)stream);
    if (ce != cudaSuccess) return cuda_fail((int)ce, "orth_orthogonalize (SOC copy)");
  }
  if (P.mat_items.empty()) return ORTH_OK;
  const int T = P.opts.ns_iters;
  float* bufs[BUF_COUNT] = {ortho_out, P.d_scratch, P.d_gram, P.d_comp};
  // X0 goes where T swaps leave the result in ortho_out
  int par = (T % 2 == 0) ? 0 : 1;      // 0: X lives in BUF_X
  float* x0 = bufs[par == 0 ? BUF_X : BUF_Y];
  const int frob = P.opts.prescale == ORTH_PRESCALE_FROBENIUS;
  int e = 0;
  {  // pre-scaling: all power iterations (or the Frobenius pass) in one cooperative launch
    Trace tr(P, ORTH_TK_POWER, -1, stream);
    e = launch_power_fused(P, params, power_cache, (!frob && !power_cache) ? 1 : 0, frob, P.opts.power_iters,
                           frob ? nullptr : power_cache, stream);
  }
  const int mode = P.opts.compute;
  if (mode == ORTH_F32) {
    if (!e) {
      Trace tr(P, ORTH_TK_SCALE, -1, stream);
      e = launch_scale(P, params, x0, stream);
    }
    {
      Trace tr(P, ORTH_TK_NS, -1, stream);
      for (int t = 0; t < T && !e; ++t) {
        e = launch_gemm_f32(P.gram[par], bufs, stream);
        if (!e) e = launch_gemm_f32(P.update[par], bufs, stream);
        P.launches += 2;
        par ^= 1;
      }
    }
    // S:125 convergence check on the last iteration's own Gram G = X_{T-1}^T X_{T-1} (still in BUF_G)
    Trace tr(P, ORTH_TK_NS_CHECK, -1, stream);
    if (!e) e = launch_converged_check(P, 0, P.opts.ns_tol, stream);
    if (!e && residual_out) {
      e = launch_gemm_f32(P.gram[0], bufs, stream);
      if (!e) e = launch_residual(P, residual_out, stream);
      P.launches++;
    }
  } else {
    // tensor cores: Gram passes g(t), update passes u(t); operand copies carry lo halves when read by a 3-pass GEMM
    auto gp = [&](int t) { return (mode == ORTH_BF16X3 || t >= T - P.opts.polish_iters) ? 3 : 1; };
    auto up = [&](int t) { return mode == ORTH_BF16X3 ? 3 : 1; };
    auto x_lo = [&](int t) { return t >= T || gp(t) == 3 || up(t) == 3; };   // t == T: the residual Gram
    // The FP32 master X is updated IN PLACE in ortho_out (an update tile's epilogue is the only reader of
    // its FP32 C block, and it overwrites that block): only the BF16 operand copies ping-pong.  This keeps
    // the NS working set (FP32 X, BF16 hi/lo X x 2, R) inside the 126 MB L2 for ImageNet-size networks.
    if (!e) {
      Trace tr(P, ORTH_TK_SCALE, -1, stream);
      e = launch_scale_bf16(P, params, bufs[BUF_X], par, x_lo(0), stream);
    }
    static const bool phased = std::getenv("ORTH_NS_PHASED") != nullptr;   // A/B switch: per-phase kernels
    if (!e && P.nsp_ctas > 0 && 2 * T + 1 <= kNspMaxPhases && !phased) {
      // all 2T (+1 residual Gram) phases in one persistent cooperative launch
      uint8_t fl[kNspMaxPhases];
      int n = 0;
      for (int t = 0; t < T; ++t) {
        // the last iteration's Gram also writes its FP32 R = I - X^T X: the convergence check reads it
        const int wf = (t == T - 1 && !residual_out) ? 16 : 0;
        fl[n++] = (uint8_t)(1 | (gp(t) == 3 ? 2 : 0) | (par << 2) | (up(t) == 3 ? 8 : 0) | wf);
        fl[n++] = (uint8_t)((up(t) == 3 ? 2 : 0) | (par << 2) | (x_lo(t + 1) ? 8 : 0) | 16);
        par ^= 1;
      }
      if (residual_out) fl[n++] = (uint8_t)(1 | 2 | (par << 2) | 16);
      {
        Trace tr(P, ORTH_TK_NS, -1, stream);
        e = launch_ns_persist(P, bufs, fl, n, stream);
      }
      Trace tr(P, ORTH_TK_NS_CHECK, -1, stream);
      if (!e && residual_out) e = launch_residual_r(P, residual_out, stream);   // also checks R_T (tol)
      else if (!e) e = launch_converged_check(P, 1, P.opts.ns_tol, stream);
      return cuda_fail(e, "orth_orthogonalize");
    }
    {
      Trace tr(P, ORTH_TK_NS, -1, stream);
      for (int t = 0; t < T && !e; ++t) {
        e = launch_ns_tc(P, bufs, par, true, gp(t), up(t) == 3, t == T - 1 && !residual_out, stream);
        if (!e) e = launch_ns_tc(P, bufs, par, false, up(t), x_lo(t + 1), true, stream);
        par ^= 1;
      }
    }
    Trace tr(P, ORTH_TK_NS_CHECK, -1, stream);
    if (!e && residual_out) {
      e = launch_ns_tc(P, bufs, 0, true, 3, false, true, stream);
      if (!e) e = launch_residual_r(P, residual_out, stream);
    } else if (!e) {
      e = launch_converged_check(P, 1, P.opts.ns_tol, stream);
    }
  }
  return cuda_fail(e, "orth_orthogonalize");
}

orth_status_t orth_compose_kernel(orth_plan_t plan, const float* ortho, float* kernels_f32, void* kernels_bf16,
                                  void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  if (!ortho || !kernels_f32) { set_error("NULL ortho or kernels_f32"); return ORTH_ERR_INVALID_ARGUMENT; }
  NvtxRange nv("orth_compose_kernel");
  // BUF_Y = the output kernels: the SLL-block merges read the FP32 kernels the first emit wrote
  float* bufs[BUF_COUNT] = {const_cast<float*>(ortho), kernels_f32, nullptr, P.d_comp};
  int e = 0;
  // composition stays FP32-accurate: SIMT FFMA, or the 3-pass split on tensor cores
  auto gemm = [&](const GemmPhase& ph) {
    if (!ph.total_tiles || e) return;
    e = P.opts.compute == ORTH_F32 ? launch_gemm_f32(ph, bufs, stream) : launch_gemm_tc(ph, bufs, 3, stream);
    P.launches++;
  };
  {
    Trace tr(P, ORTH_TK_COMPOSE, -1, stream);
    if (P.opts.compute == ORTH_F32) {
      gemm(P.proj);
      for (auto& ph : P.chain) gemm(ph);
      gemm(P.aoc);
    } else {
      e = launch_compose_tc(P, ortho, stream);
    }
    if (!e && !P.soc.empty()) {   // f3: explicit exponentials of the SOC units
      e = launch_soc_skew(P, ortho, stream);
      for (auto& ph : P.soc_pow) gemm(ph);
      if (!e) e = launch_soc_alpha(P, stream);
      if (!e) e = launch_soc_sum(P, stream);
    }
    if (!e && !P.sll.empty()) {   // f4: AOL rescale of the SLL kernels
      gemm(P.sll_v);
      if (!e) e = launch_sll_scale(P, ortho, stream);
    }
  }
  if (!e) {
    Trace tr(P, ORTH_TK_EMIT, -1, stream);
    e = launch_emit(P, bufs, kernels_f32, (uint16_t*)kernels_bf16, stream);
  }
  if (!e && !P.blk.empty()) {   // f4: merge the SLL blocks' kernels once per update, then emit them
    Trace tr(P, ORTH_TK_COMPOSE, -1, stream);
    gemm(P.blk_mm);
    if (!e) e = launch_blk_merge(P, stream);
    if (!e) e = launch_emit_list(P, P.emit2, P.d_emit2, bufs, kernels_f32, (uint16_t*)kernels_bf16, stream);
  }
  return cuda_fail(e, "orth_compose_kernel");
}

orth_status_t orth_conv_forward(orth_plan_t plan, int32_t layer, const void* kernel, const float* bias, const void* x,
                                void* y, int32_t N, int32_t H, int32_t W, int32_t io, void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  int Ho = 0, Wo = 0;
  st = check_conv(P, layer, kernel, x, y, N, H, W, io, Ho, Wo);
  if (st != ORTH_OK || N == 0) return st;
  NvtxRange nv("orth_conv_forward");
  Trace tr(P, ORTH_TK_CONV_FWD, layer, stream);
  const LayerInfo& L = P.layers[layer];
  if (L.cons == CONS_SLL_BLOCK) {   // f4: y = M *_s [x | relu(C * x + bias)]
    if ((int64_t)N * H * W * 4 > L.blk_scratch_bytes) {
      set_error("SLL block %d: N*H*W exceeds the declared grid_h/grid_w x max_batch (its h and [x | h] scratch)", layer);
      return ORTH_ERR_SHAPE_MISMATCH;
    }
    const LayerInfo& Lc = P.blk_conv[2 * L.blk_id];
    const LayerInfo& Lm = P.blk_conv[2 * L.blk_id + 1];
    const size_t es = io == ORTH_BF16 ? 2 : 4;
    const void* km = static_cast<const char*>(kernel) + (size_t)L.m_off * es;
    int e = launch_conv_fwd(Lc, kernel, Lc.wt_scratch, bias, x, L.blk_h, N, H, W, H, W, io, stream);
    if (!e) e = launch_relu_concat(x, L.blk_h, L.blk_z, (int64_t)N * H * W, L.ci, L.blk_cs, io, stream);
    if (!e) e = launch_conv_fwd(Lm, km, Lm.wt_scratch, nullptr, L.blk_z, y, N, H, W, Ho, Wo, io, stream);
    P.launches += 3;
    return cuda_fail(e, "orth_conv_forward (SLL block)");
  }
  const int e = launch_conv_fwd(P.layers[layer], kernel, P.layers[layer].wt_scratch, bias, x, y, N, H, W, Ho, Wo, io, stream);
  P.launches++;
  return cuda_fail(e, "orth_conv_forward");
}

orth_status_t orth_conv_transpose(orth_plan_t plan, int32_t layer, const void* kernel, const float* bias,
                                  const void* y_small, void* x_big, int32_t N, int32_t H_big, int32_t W_big, int32_t io,
                                  void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  int Ho = 0, Wo = 0;
  st = check_conv(P, layer, kernel, y_small, x_big, N, H_big, W_big, io, Ho, Wo);
  if (st != ORTH_OK) return st;
  if (P.layers[layer].cons == CONS_SLL_BLOCK) { set_error("an SLL block is not linear: no adjoint"); return ORTH_ERR_UNSUPPORTED_CONFIG; }
  if (N == 0) return ORTH_OK;
  NvtxRange nv("orth_conv_transpose");
  Trace tr(P, ORTH_TK_CONV_ADJ, layer, stream);
  const int e = launch_conv_bwd(P.layers[layer], kernel, P.layers[layer].wt_scratch, bias, y_small, x_big, N, H_big, W_big, Ho,
                                Wo, io, stream);
  P.launches++;
  return cuda_fail(e, "orth_conv_transpose");
}

orth_status_t orth_kernels_assemble(orth_plan_t plan, const float* gathered_f32, float* kernels_f32,
                                    const void* gathered_bf16, void* kernels_bf16, void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  if (P.opts.world == 1) return ORTH_OK;
  if ((!gathered_f32) != (!kernels_f32) || (!gathered_bf16) != (!kernels_bf16)) {
    set_error("gathered / kernels pointers must be both set or both NULL per dtype");
    return ORTH_ERR_INVALID_ARGUMENT;
  }
  if ((gathered_f32 && (const void*)gathered_f32 == (const void*)kernels_f32) ||
      (gathered_bf16 && gathered_bf16 == kernels_bf16)) {
    set_error("gathered and final kernel buffers must not overlap");
    return ORTH_ERR_INVALID_ARGUMENT;
  }
  NvtxRange nv("orth_kernels_assemble");
  Trace tr(P, ORTH_TK_ASSEMBLE, -1, stream);
  const int e = launch_assemble(P, gathered_f32, kernels_f32, (const uint16_t*)gathered_bf16, (uint16_t*)kernels_bf16,
                                stream);
  P.launches++;
  return cuda_fail(e, "orth_kernels_assemble");
}

orth_status_t orth_conv_wgrad_workspace(orth_plan_t plan, int32_t layer, int32_t N, int32_t H, int32_t W, int32_t io,
                                        int64_t* bytes) {
  if (!plan || !bytes) { set_error("NULL plan or bytes"); return ORTH_ERR_INVALID_ARGUMENT; }
  Plan& P = plan->p;
  if (layer < 0 || layer >= (int)P.layers.size()) { set_error("layer %d out of range", layer); return ORTH_ERR_INVALID_ARGUMENT; }
  const LayerInfo& L = P.layers[layer];
  if (N < 0 || H < 1 || W < 1) { set_error("N >= 0, H, W >= 1 required"); return ORTH_ERR_SHAPE_MISMATCH; }
  const int Ho = out_dim(H, L.k, L.s, L.d, L.pt, L.pb), Wo = out_dim(W, L.k, L.s, L.d, L.pl, L.pr);
  *bytes = N == 0 ? 0 : wgrad_workspace_bytes(L, N, Ho, Wo, io);
  return ORTH_OK;
}

orth_status_t orth_conv_wgrad(orth_plan_t plan, int32_t layer, const void* x, const void* dy, float* dkernel_f32,
                              int32_t N, int32_t H, int32_t W, int32_t io, void* workspace, int64_t workspace_bytes,
                              void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  int Ho = 0, Wo = 0;
  st = check_conv(P, layer, dkernel_f32, x, const_cast<void*>(dy), N, H, W, io, Ho, Wo);
  if (st != ORTH_OK) return st;
  const LayerInfo& L = P.layers[layer];
  if (L.cons == CONS_SLL_BLOCK) { set_error("SLL blocks have no single weight gradient"); return ORTH_ERR_UNSUPPORTED_CONFIG; }
  if ((int64_t)N * H * W >= (1LL << 31)) { set_error("N*H*W must stay below 2^31 (32-bit pixel indices)"); return ORTH_ERR_SHAPE_MISMATCH; }
  if (N == 0)   // the gradient over an empty batch is zero
    return cuda_fail((int)cudaMemsetAsync(dkernel_f32, 0, (size_t)L.kernel_numel * 4, (cudaStream_t)stream),
                     "orth_conv_wgrad");
  NvtxRange nv("orth_conv_wgrad");
  Trace tr(P, ORTH_TK_WGRAD, layer, stream);
  const int e = launch_wgrad(L, x, dy, dkernel_f32, N, H, W, Ho, Wo, io, workspace, workspace_bytes, stream);
  P.launches += 2;
  return cuda_fail(e, "orth_conv_wgrad");
}

orth_status_t orth_compose_vjp(orth_plan_t plan, const float* ortho, const float* dkernels_f32, float* d_ortho,
                               void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  if (!P.opts.vjp || !P.d_vjp) { set_error("create the plan with opts.vjp = 1"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (!P.vjp_supported) { set_error("no VJP for SOC / SLL layers or SLL blocks"); return ORTH_ERR_UNSUPPORTED_CONFIG; }
  if (!ortho || !dkernels_f32 || !d_ortho) { set_error("NULL ortho, dkernels or d_ortho"); return ORTH_ERR_INVALID_ARGUMENT; }
  NvtxRange nv("orth_compose_vjp");
  Trace tr(P, ORTH_TK_COMPOSE_VJP, -1, stream);
  cudaStream_t s = (cudaStream_t)stream;
  float* bufs[BUF_COUNT] = {const_cast<float*>(ortho), P.d_vjp, d_ortho, P.d_comp};
  int e = 0;
  auto gemm = [&](const GemmPhase& ph) {
    if (!ph.total_tiles || e) return;
    e = P.opts.compute == ORTH_F32 ? launch_gemm_f32(ph, bufs, stream) : launch_gemm_tc(ph, bufs, 3, stream);
    P.launches++;
  };
  if (P.cv_zero_n > 0)
    e = (int)cudaMemsetAsync(P.d_vjp + P.cv_zero_off, 0, (size_t)P.cv_zero_n * sizeof(float), s);
  for (size_t i = 0; i + 2 < P.cv_qcopy.size() && !e; i += 3)
    e = (int)cudaMemcpyAsync(P.d_vjp + P.cv_qcopy[i + 1], ortho + P.cv_qcopy[i], (size_t)P.cv_qcopy[i + 2] * 4,
                             cudaMemcpyDeviceToDevice, s);
  gemm(P.proj);                                  // projectors P = U U^T (into comp, as in the forward)
  for (auto& ph : P.cv_fwd) gemm(ph);            // chain intermediates, one buffer per step
  if (!e) e = launch_vjp_deemit(P, dkernels_f32, d_ortho, stream);
  gemm(P.cv_dr);                                 // AOC: dR_ab
  if (!e) e = launch_vjp_scatter(P, d_ortho, stream);
  gemm(P.cv_dkb);                                // AOC: dK_BCOP
  for (size_t j = 0; j < P.cv_bwd_a.size(); ++j) {
    gemm(P.cv_bwd_a[j]);
    gemm(P.cv_bwd_b[j]);
    gemm(P.cv_bwd_c[j]);
  }
  return cuda_fail(e, "orth_compose_vjp");
}

orth_status_t orth_orthogonalize_vjp(orth_plan_t plan, const float* params, const float* d_ortho, float* d_params,
                                     void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  if (!P.opts.vjp || !P.d_vjp) { set_error("create the plan with opts.vjp = 1"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (!params || !d_ortho || !d_params) { set_error("NULL params, d_ortho or d_params"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (P.mat_items.empty()) return ORTH_OK;
  NvtxRange nv("orth_orthogonalize_vjp");
  Trace tr(P, ORTH_TK_NS_VJP, -1, stream);
  cudaStream_t s = (cudaStream_t)stream;
  float* bufs[BUF_COUNT] = {nullptr, P.d_vjp, nullptr, nullptr};
  int e = 0;
  auto gemm = [&](const GemmPhase& ph) {
    if (!ph.total_tiles || e) return;
    e = P.opts.compute == ORTH_F32 ? launch_gemm_f32(ph, bufs, stream) : launch_gemm_tc(ph, bufs, 3, stream);
    P.launches++;
  };
  e = launch_scale(P, params, P.d_vjp + P.vj_x_off, stream);   // X_0 = W / sigma (the forward's sigma)
  for (auto& ph : P.vj_fwd) gemm(ph);                          // X_1 .. X_{T-1}
  if (!e) e = (int)cudaMemcpyAsync(P.d_vjp + P.vj_g_off[1], d_ortho, (size_t)P.params_numel * 4,
                                   cudaMemcpyDeviceToDevice, s);
  for (auto& ph : P.vj_bwd) gemm(ph);
  if (!e) e = launch_scale(P, P.d_vjp + P.vj_g_off[P.vj_g_final], d_params, stream);   // d_params = G_0 / sigma
  return cuda_fail(e, "orth_orthogonalize_vjp");
}

orth_status_t orth_certify_workspace(orth_plan_t plan, int32_t layer, int32_t H, int32_t W, int64_t* bytes) {
  if (!plan || !bytes) { set_error("NULL plan or bytes"); return ORTH_ERR_INVALID_ARGUMENT; }
  Plan& P = plan->p;
  if (layer < 0 || layer >= (int)P.layers.size()) { set_error("layer %d out of range", layer); return ORTH_ERR_INVALID_ARGUMENT; }
  if (H < 1 || W < 1) { set_error("H, W must be >= 1"); return ORTH_ERR_SHAPE_MISMATCH; }
  const int64_t b = certify_workspace_bytes(P.layers[layer], H, W);
  if (b < 0) { set_error("grid %dx%d does not fit layer %d (s | H, s | W; dense: 1x1)", H, W, layer); return ORTH_ERR_SHAPE_MISMATCH; }
  *bytes = b;
  return ORTH_OK;
}

orth_status_t orth_certify(orth_plan_t plan, int32_t layer, const float* kernel_f32, int32_t H, int32_t W,
                           int32_t power_iters, void* workspace, int64_t workspace_bytes, double* out, void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  int64_t need = 0;
  st = orth_certify_workspace(plan, layer, H, W, &need);
  if (st != ORTH_OK) return st;
  if (!kernel_f32 || !workspace || !out) { set_error("NULL kernel, workspace or out"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (workspace_bytes < need) { set_error("workspace %lld < %lld bytes", (long long)workspace_bytes, (long long)need); return ORTH_ERR_INVALID_ARGUMENT; }
  if (power_iters < 0) { set_error("power_iters must be >= 0"); return ORTH_ERR_INVALID_ARGUMENT; }
  if (((uintptr_t)workspace | (uintptr_t)out) & 15) { set_error("workspace/out must be 16-byte aligned"); return ORTH_ERR_INVALID_ARGUMENT; }
  Plan& P = plan->p;
  NvtxRange nv("orth_certify");
  Trace tr(P, ORTH_TK_CERTIFY, layer, stream);
  const int e = launch_certify(P.layers[layer], kernel_f32, H, W, power_iters, workspace, out, stream);
  P.launches += 3;
  return cuda_fail(e, "orth_certify");
}

orth_status_t orth_plan_trace(orth_plan_t plan, int32_t enable) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  tstate(plan->p).on = enable != 0;
  return ORTH_OK;
}

orth_status_t orth_plan_trace_read(orth_plan_t plan, orth_trace_rec_t* out, int32_t cap, int32_t* n) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  if (!n || cap < 0) { set_error("NULL n or negative cap"); return ORTH_ERR_INVALID_ARGUMENT; }
  orth_trace_state& T = tstate(plan->p);
  *n = (int32_t)T.pending.size();
  int i = 0;
  for (auto& r : T.pending) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail((int)e, "orth_plan_trace_read");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    r.rec.ms = ms;
    if (out && i < cap) out[i] = r.rec;
    ++i;
    T.pool.push_back(r.a);
    T.pool.push_back(r.b);
  }
  T.pending.clear();
  return ORTH_OK;
}

orth_status_t orth_plan_check(orth_plan_t plan, void* stream) {
  orth_status_t st = need_device(plan);
  if (st != ORTH_OK) return st;
  Plan& P = plan->p;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail((int)e, "orth_plan_check");
  int32_t h = 0;
  e = cudaMemcpy(&h, P.d_status, sizeof(h), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(P.d_status, 0, sizeof(int32_t));
  if (e != cudaSuccess) return cuda_fail((int)e, "orth_plan_check");
  if (h != 0) set_error("device status %d", h);
  return (orth_status_t)h;
}

}  // extern "C"
