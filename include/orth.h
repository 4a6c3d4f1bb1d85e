/*
 * orth.h -- C ABI of the B200-native orthogonal-convolution hot path.
 *
 * The library turns free parameter matrices into exactly orthogonal conv
 * kernels and applies them (arXiv 2601.13776 "Orthogonium", AOC layers):
 *
 *   orth_plan_create     host: validate layers, derive the matrices of every
 *                        (layer, group) unit, packed layouts, workspace.
 *   orth_orthogonalize   a2+a3: pre-scaling (batched power iteration, P:100-101,
 *                        P:313, or Frobenius) then T Bjorck / Newton-Schulz
 *                        iterations W <- (1+b)W - b W W^T W.
 *   orth_compose_kernel  a4+a5: BCOP chain of projector blocks, RKO
 *                        reshape and AOC = RKO (*) K_BCOP, emitted
 *                        as FP32 PyTorch-layout and BF16 GEMM-layout kernels.
 *   orth_conv_forward    a6: strided / dilated / grouped conv with that kernel
 *                        ("a single call to torch.nn.Conv2d").
 *   orth_conv_transpose  a7: its exact adjoint (P:334 transposed convolutions).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R<k> = reading k of
 * DESIGN.md "Readings of the paper".  Everything computed here is defined by
 * the float64 oracle in oracle/orth_oracle.py, which shares no code with it.
 *
 * Conventions
 *  - Ownership: the caller owns every data buffer (params, ortho, power cache,
 *    kernels, x, y, bias).  They are DEVICE pointers on the plan's device,
 *    16-byte aligned (128 B preferred).  The plan owns its workspace (allocated
 *    in orth_plan_create, freed in orth_plan_destroy) and a device status word.
 *    No call allocates device memory after create: the per-layer conv scratch
 *    (split-K partials and flags, padded input copies, transposed / packed
 *    weights) is sized at create from the declared grid (grid_h, grid_w) of
 *    every layer and opts.max_batch, one private slice per layer.
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).  Compute calls are asynchronous: they validate
 *    arguments synchronously (enqueuing nothing on failure), enqueue kernels on
 *    `stream` and return.  None calls cudaDeviceSynchronize.  Calls on
 *    DIFFERENT layers may run concurrently on different streams (each layer
 *    owns its conv scratch); calls on the same layer, and the construction
 *    calls (orth_orthogonalize / orth_compose_kernel, which share the NS and
 *    composition workspace), must be ordered on one stream.
 *  - Device-side conditions (zero matrix; NS not converged, S:125:
 *    non-finite, or the residual bound of the last iteration above
 *    opts.ns_tol) set the plan's status word; orth_plan_check reports them.
 *  - Determinism: results are bitwise reproducible for fixed inputs, device
 *    type and (rank, world): no floating-point atomics, fixed reduction order.
 *  - Threading: a plan serves one host thread at a time.  orth_last_error is
 *    thread-local.
 */
#ifndef ORTH_H_
#define ORTH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orth_plan* orth_plan_t;

typedef enum {
  ORTH_OK = 0,
  ORTH_ERR_INVALID_ARGUMENT = 1,   /* null pointer, bad enum, dim < 1, g does not divide channels, beta not in (0, 1/2], T < 1 */
  ORTH_ERR_UNSUPPORTED_CONFIG = 2, /* k < s, gcd(s, d) != 1 (R10), non-square k/s/d, dense forward */
  ORTH_ERR_SHAPE_MISMATCH = 3,     /* N/H/W inconsistent with the layer, circular with s not dividing H or W (R11) */
  ORTH_ERR_ZERO_NORM = 4,          /* device: a zero parameter matrix */
  ORTH_ERR_NOT_CONVERGED = 5,      /* device: NS residual non-finite or its bound above ns_tol */
  ORTH_ERR_CUDA = 6,               /* CUDA runtime error; detail in orth_last_error() */
  ORTH_ERR_OUT_OF_MEMORY = 7,      /* workspace allocation failed */
  ORTH_ERR_NO_DEVICE = 8           /* compute call on a host-only plan (device = -1) */
} orth_status_t;

typedef enum { ORTH_F32 = 0, ORTH_BF16 = 1, ORTH_BF16X3 = 2 } orth_dtype_t;
typedef enum { ORTH_PAD_ZEROS = 0, ORTH_PAD_CIRCULAR = 1 } orth_pad_t;
typedef enum { ORTH_CONV2D = 0, ORTH_CONV_TRANSPOSE2D = 1, ORTH_DENSE = 2, ORTH_SOC = 3, ORTH_SLL = 4,
               ORTH_SLL_BLOCK = 5 } orth_kind_t;
typedef enum { ORTH_PRESCALE_POWER = 0, ORTH_PRESCALE_FROBENIUS = 1 } orth_prescale_t;

/* One orthogonal layer (S:35-40 ConvSpec + S:205-210 ConvLayerConfig).
 *  kind ORTH_CONV2D: AdaptiveOrthoConv2d, c_in -> c_out.
 *  kind ORTH_CONV_TRANSPOSE2D: AdaptiveOrthoConvTranspose2d, c_in (small
 *    spatial) -> c_out (large spatial); its kernel is that of the forward
 *    adjoint conv c_out -> c_in, PyTorch ConvTranspose2d weight layout
 *    (c_in, c_out/g, k, k) (R13).
 *  kind ORTH_DENSE: an OrthoLinear weight c_out x c_in; k = s = d = 1.
 *  kind ORTH_SOC: AdaptiveSOCConv2d (App. B.2): the free parameter of each group is a
 *    kernel (c/g, c/g, k, k) (k odd, c_in = c_out, s = 1), packed as one c/g x (c/g) k^2 "matrix" (role K)
 *    that orth_orthogonalize passes through unchanged; orth_compose_kernel builds the EXPLICIT exponential
 *    E = delta + L + L(*)L/2! + ... + L^(*)n/n!, L = alpha skew(K), alpha the scalar AOL bound (R25-R27),
 *    of spatial size k_eff = n (k - 1) + 1, n = soc_terms (0 -> 6); conv calls apply E ("same" padding of
 *    k_eff).  Circular padding makes the layer orthogonal up to the series tail e/(n+1)!.
 *  kind ORTH_SLL: the kernel K of an SLL layer ("W T^{-1/2} = Toeplitz(K)"), c_in -> c_out, k,
 *    s = d = g = 1: one free c_out x c_in k^2 matrix (role K) that orth_compose_kernel AOL-rescales per
 *    input channel (R28), so |T(K)| <= 1.
 *  kind ORTH_SLL_BLOCK: the fused SLL x AOC down-sampling block (App. B.3) over three EARLIER
 *    layers of the plan: blk_pre (ORTH_CONV2D c -> c, s = 1), blk_sll (ORTH_SLL c -> c_s) and blk_post
 *    (ORTH_CONV2D c -> c_out, stride s), all g = d = 1, circular; c_in = c, c_out and stride_h/w = s of the
 *    block must match (k_h/k_w are ignored).  orth_compose_kernel merges them once per update
 *    (P:399): C = K (*) K_pre (c_s x c) and M = [K_post (*) K_pre | -2 K_post (*) K^T] (c_out x (c + c_s)),
 *    stored back to back in the block's kernel region (ORTH_Q_LAYER_BLOCK_M_OFF); orth_conv_forward
 *    computes y = M *_s [x | relu(C * x + bias)] (bias: the SLL bias, c_s floats) -- two conv launches and
 *    one concat, with h and [x | h] in the layer's scratch (declare grid_h/grid_w and max_batch).  The
 *    block and its three layers are constructed on one rank.
 *  Square kernels/strides/dilations only (k_h == k_w, ...).  pad_* = -1 selects
 *  the "same" rule p_t = floor(d(k-1)/2), p_b = d(k-1) - p_t (R11).
 *  grid_h, grid_w: the largest spatial size the layer's conv calls will see on
 *  the forward-conv INPUT side (ORTH_CONV2D: its input; ORTH_CONV_TRANSPOSE2D:
 *  its large output grid, H_big of orth_conv_transpose).  Together with
 *  opts.max_batch they size the layer's conv scratch at create time; 0 = not
 *  declared (no scratch: calls still run, on the kernels that need none, and
 *  so does any call larger than the declaration -- same results up to FP32
 *  summation order).  */
typedef struct {
  int32_t kind;          /* orth_kind_t */
  int32_t c_in, c_out;
  int32_t k_h, k_w;
  int32_t stride_h, stride_w;
  int32_t dil_h, dil_w;
  int32_t groups;
  int32_t pad_t, pad_b, pad_l, pad_r;
  int32_t padding_mode;  /* orth_pad_t */
  int32_t grid_h, grid_w;
  int32_t soc_terms;     /* ORTH_SOC: highest power n of the series (0 -> 6); ignored otherwise */
  int32_t blk_pre, blk_sll, blk_post;   /* ORTH_SLL_BLOCK: layer indices (< this layer); ignored otherwise */
} orth_layer_desc_t;

/* OrthoParams, Bjorck only. */
typedef struct {
  int32_t ns_iters;      /* T >= 1, default 12 (R1) */
  float beta;            /* in (0, 1/2], default 0.5 */
  int32_t prescale;      /* orth_prescale_t, default power (R3) */
  int32_t power_iters;   /* P >= 1, default 3 (R2) */
  int32_t compute;       /* NS / composition contractions (R16):
                            ORTH_F32    FP32 FFMA (SIMT), FP32-accurate;
                            ORTH_BF16   tensor cores, BF16 operands, FP32 master X in residual form
                                        X <- X + b X (I - X^T X); the last polish_iters iterations and the
                                        composition use the 3-pass hi/lo split (~2^-16 products);
                            ORTH_BF16X3 tensor cores, 3-pass split everywhere (products to ~2^-16:
                                        measured 2e-5 relative on chained kernels, tested at 1e-4; only
                                        ORTH_F32 meets the 1e-5 FP32 tolerance). */
  int32_t polish_iters;  /* BF16 only: trailing iterations run FP32-accurate, default 2 */
  int32_t rank, world;   /* construction sharding by (layer, group) unit, LPT (R22); default 0, 1 */
  float ns_tol;          /* NOT_CONVERGED threshold on the bound 3/4 r^2 + 1/4 r^3 >= |I - X_T^T X_T|_F,
                            r = |I - X_{T-1}^T X_{T-1}|_F from the last iteration's own Gram (R20);
                            default 1e-3 (north star max|sigma - 1|); <= 0: non-finite check only */
  int32_t max_batch;     /* largest N of any conv call (sizes the per-layer scratch); default 0 */
  int32_t vjp;           /* 1: allocate the backward workspace (T x params floats for the NS iterates + the
                            composition chain's per-step buffers) for orth_compose_vjp / orth_orthogonalize_vjp */
} orth_opts_t;

/* Fill *opts with the defaults above. */
void orth_opts_default(orth_opts_t* opts);

/* Host-only validation of layer descriptors and options; needs no GPU.
 * Returns the first failing status; detail in orth_last_error(). */
orth_status_t orth_validate_desc(const orth_layer_desc_t* layers, int32_t n_layers, const orth_opts_t* opts);

/* Create a plan for n_layers layers on CUDA device `device` (>= 0), or a
 * host-only plan (device = -1) usable for orth_plan_query only.  Copies
 * `layers` and `opts` (opts may be NULL = defaults).  On success *plan owns
 * all workspace. */
orth_status_t orth_plan_create(const orth_layer_desc_t* layers, int32_t n_layers, const orth_opts_t* opts,
                               int32_t device, orth_plan_t* plan);
orth_status_t orth_plan_destroy(orth_plan_t plan);

/* Plan queries (int64 result in *out).  `index` is a layer index for the
 * ORTH_Q_LAYER_* queries, a global matrix index for ORTH_Q_MATRIX_* and a unit
 * index for ORTH_Q_UNIT_*. */
typedef enum {
  ORTH_Q_N_LAYERS = 0,
  ORTH_Q_N_MATRICES = 1,          /* total parameter matrices over all layers and groups */
  ORTH_Q_PARAMS_NUMEL = 2,        /* floats in the packed params / ortho buffers */
  ORTH_Q_CACHE_NUMEL = 3,         /* floats in the packed power-iteration cache */
  ORTH_Q_KERNELS_F32_NUMEL = 4,   /* floats in kernels_f32 (all ranks' segments) */
  ORTH_Q_KERNELS_BF16_NUMEL = 5,  /* bf16 elements in kernels_bf16 */
  ORTH_Q_WORKSPACE_BYTES = 6,
  ORTH_Q_NS_FLOPS = 7,            /* algorithmic NS flops 4 m n^2 T (m >= n) of this rank's matrices */
  ORTH_Q_KERNEL_SEGMENT_F32 = 8,  /* per-rank segment size (floats) of the gather layout (world > 1) */
  ORTH_Q_KERNEL_SEGMENT_BF16 = 9,
  ORTH_Q_N_UNITS = 10,            /* construction units (layer, group) over all layers */
  ORTH_Q_GATHER_F32_NUMEL = 11,   /* world * KERNEL_SEGMENT_F32 (world == 1: KERNELS_F32_NUMEL) */
  ORTH_Q_GATHER_BF16_NUMEL = 12,
  ORTH_Q_CONV_SCRATCH_BYTES = 13, /* plan-owned conv scratch over all layers */
  ORTH_Q_COMP_FLOPS = 14,         /* structured composition flops of this rank's units */
  ORTH_Q_LAYER_FIRST_MATRIX = 20, /* global index of the layer's first matrix */
  ORTH_Q_LAYER_MATS_PER_GROUP = 21,
  ORTH_Q_LAYER_KERNEL_OFF_F32 = 22,
  ORTH_Q_LAYER_KERNEL_OFF_BF16 = 23,
  ORTH_Q_LAYER_KERNEL_NUMEL = 24, /* elements of the layer kernel (same in both layouts) */
  ORTH_Q_LAYER_OWNER = 25,        /* rank that constructs the layer's group 0 (see ORTH_Q_UNIT_OWNER) */
  ORTH_Q_LAYER_C_MID = 26,        /* derived internal width (R7); 0 if none */
  ORTH_Q_LAYER_C_B = 27,          /* BCOP width; 0 if none */
  ORTH_Q_LAYER_KP = 28,           /* BCOP size k' (R8); 0 if none */
  ORTH_Q_LAYER_K_EFF = 32,        /* kernel size of the applied kernel (SOC: n (k - 1) + 1; SLL block: of M) */
  ORTH_Q_LAYER_BLOCK_KC = 33,     /* SLL block: size of C */
  ORTH_Q_LAYER_BLOCK_M_OFF = 34,  /* SLL block: element offset of M inside the layer's kernel region */
  ORTH_Q_LAYER_BLOCK_PADS = 35,   /* SLL block: top pad of C (low 16 bits) and of M (high 16 bits) */
  ORTH_Q_LAYER_SCRATCH_BYTES = 29,/* this layer's conv scratch slice */
  ORTH_Q_LAYER_NS_FLOPS = 30,     /* 4 m n^2 T over the layer's matrices (all groups) */
  ORTH_Q_LAYER_COMP_FLOPS = 31,   /* structured composition flops of the layer (all groups) */
  ORTH_Q_MATRIX_ROWS = 40,
  ORTH_Q_MATRIX_COLS = 41,
  ORTH_Q_MATRIX_OFFSET = 42,      /* float offset in params / ortho */
  ORTH_Q_MATRIX_CACHE_OFFSET = 43,/* float offset of its length-n vector in the power cache */
  ORTH_Q_MATRIX_LAYER = 44,
  ORTH_Q_MATRIX_GROUP = 45,
  ORTH_Q_MATRIX_ROLE = 46,        /* 0 Q, 1 U, 2 R, 3 W, 4 K (SOC free kernel, not orthogonalised) */
  ORTH_Q_UNIT_LAYER = 60,         /* units are ordered layer -> group */
  ORTH_Q_UNIT_GROUP = 61,
  ORTH_Q_UNIT_OWNER = 62,         /* rank that orthogonalises and composes this unit */
  ORTH_Q_UNIT_NUMEL = 63,         /* kernel elements of one unit: (c_out/g) (c_in/g) k^2 (forward view) */
  ORTH_Q_UNIT_GATHER_OFF_F32 = 64,/* offset in the gather layout (owner * segment + position) */
  ORTH_Q_UNIT_GATHER_OFF_BF16 = 65,
  ORTH_Q_UNIT_KERNEL_OFF_F32 = 66,/* offset in the final layout (= LAYER_KERNEL_OFF + group * numel) */
  ORTH_Q_UNIT_KERNEL_OFF_BF16 = 67
} orth_query_t;
orth_status_t orth_plan_query(orth_plan_t plan, int32_t what, int32_t index, int64_t* out);

/* a2+a3.  params: packed FP32 matrices, layer -> group -> [Q, U_1..U_2(k'-1), R]
 * (R15), each row-major at ORTH_Q_MATRIX_OFFSET (offsets 128 B aligned).
 * ortho_out: same layout; receives the orthogonalised matrices of this rank's
 * layers (others untouched).  power_cache: nullable in/out, one length-n
 * vector per matrix at ORTH_Q_MATRIX_CACHE_OFFSET (P:313 cached vector); NULL
 * starts every power iteration from ones/sqrt(n) (R2).  residual_out:
 * nullable, one float per matrix: |I - X^T X|_F of the result on the short
 * side.  Device-side zero matrices / non-finite residuals set the status word.
 * params and ortho_out must not overlap. */
orth_status_t orth_orthogonalize(orth_plan_t plan, const float* params, float* ortho_out, float* power_cache,
                                 float* residual_out, void* stream);

/* a4+a5.  ortho: the output of orth_orthogonalize.  kernels_f32: receives the
 * kernels in PyTorch weight layout (Conv2d: (c_out, c_in/g, k, k);
 * ConvTranspose2d: (c_in, c_out/g, k, k); dense: (c_out, c_in)).  kernels_bf16:
 * nullable; receives the GEMM layout (C_o, k, k, C_i/g) of the forward conv,
 * RNE-rounded.
 * world == 1: the final layout, layer l at ORTH_Q_LAYER_KERNEL_OFF_{F32,BF16}
 * (ORTH_Q_KERNELS_*_NUMEL elements).
 * world > 1: the GATHER layout (ORTH_Q_GATHER_*_NUMEL elements): this rank's
 * units only, at ORTH_Q_UNIT_GATHER_OFF_* inside its own rank-major segment
 * [rank * seg, (rank + 1) * seg) -- the input of one all-gather of equal
 * segments (R22), after which orth_kernels_assemble builds the final layout. */
orth_status_t orth_compose_kernel(orth_plan_t plan, const float* ortho, float* kernels_f32, void* kernels_bf16,
                                  void* stream);

/* a6.  Applies the conv of layer `layer`'s kernel: input (N, H, W, C_i) NHWC
 * -> output (N, H_out, W_out, C_o), H_out = floor((H + p_t + p_b - d(k-1) - 1)/s) + 1,
 * where (C_i, C_o) = (c_in, c_out) for ORTH_CONV2D and (c_out, c_in) for
 * ORTH_CONV_TRANSPOSE2D (whose forward adjoint this is).
 * io = ORTH_F32: x, y float32 and `kernel` the layer's FP32 PyTorch-layout kernel;
 * io = ORTH_BF16: x, y bfloat16 and `kernel` the layer's BF16 GEMM-layout kernel.
 * bias: nullable FP32[C_o].  Accumulation FP32.  Circular padding requires
 * s | H and s | W (R11).  Dense layers: ORTH_ERR_UNSUPPORTED_CONFIG.
 * N = 0 (an empty batch, e.g. a rank's empty shard) is a no-op: x and y may be
 * NULL; H, W must still be >= 1 (and so for orth_conv_transpose).  The padded
 * pixel count N (H + p_t + p_b)(W + p_l + p_r) must stay below 2^31 (32-bit
 * pixel indices; SHAPE_MISMATCH otherwise). */
orth_status_t orth_conv_forward(orth_plan_t plan, int32_t layer, const void* kernel, const float* bias,
                                const void* x, void* y, int32_t N, int32_t H, int32_t W, int32_t io, void* stream);

/* a7.  Exact adjoint of orth_conv_forward for the same layer and kernel:
 * y_small (N, H_out, W_out, C_o) -> x_big (N, H_big, W_big, C_i).  For an
 * ORTH_CONV_TRANSPOSE2D layer this is its forward (ConvTranspose2d); for an
 * ORTH_CONV2D layer it is the data gradient.  The large size is explicit, so
 * PyTorch's output_padding ambiguity does not arise.  bias: nullable FP32[C_i]. */
orth_status_t orth_conv_transpose(orth_plan_t plan, int32_t layer, const void* kernel, const float* bias,
                                  const void* y_small, void* x_big, int32_t N, int32_t H_big, int32_t W_big,
                                  int32_t io, void* stream);

/* a8 (world > 1).  Copies every unit from the all-gathered gather layout
 * (ORTH_Q_UNIT_GATHER_OFF_*) to its place in the final layout
 * (ORTH_Q_UNIT_KERNEL_OFF_*), so that each layer's kernel is contiguous for
 * orth_conv_forward.  Either pair (gathered_f32, kernels_f32) or
 * (gathered_bf16, kernels_bf16) may be NULL; the buffers must not overlap.
 * world == 1: nothing to do (returns ORTH_OK). */
orth_status_t orth_kernels_assemble(orth_plan_t plan, const float* gathered_f32, float* kernels_f32,
                                    const void* gathered_bf16, void* kernels_bf16, void* stream);

/* Synchronises `stream`, reads and clears the device status word; returns the
 * first device-side error since the last check (or a pending CUDA error). */
orth_status_t orth_plan_check(orth_plan_t plan, void* stream);

/* ---- f1: backward of the path (P:61, P:122 a TRAINING wall time; R31-R33).
 * Data gradient: orth_conv_transpose (the exact adjoint).  Weight gradient, in the layer's forward-conv view
 * (y = conv(x, K): x on the large grid (N, H, W, C_i), dy on the output grid (N, H_out, W_out, C_o); for an
 * ORTH_CONV_TRANSPOSE2D layer, whose forward is the adjoint, x is the gradient of its large output and dy its
 * small input):  dkernel_f32 = dK, PyTorch layout of the layer's FP32 kernel, defined by the bilinear form
 * <dy, conv(x, delta K)> = <dK, delta K>.  io = ORTH_BF16 with channels per group multiple of 8: tcgen05
 * GEMM over the pixels (M = c_out/g, N = c_in/g, up to 3 taps per CTA sharing the dy tile); otherwise
 * FP32 SIMT.  Both sum pixel splits in a fixed order through `workspace` (orth_conv_wgrad_workspace bytes,
 * caller-owned device memory; 0 bytes: none needed).  FP32 accumulation, deterministic.  N*H*W < 2^31.
 * N = 0: dK = 0 (x, dy may be NULL).  Not for SLL blocks or dense layers. */
orth_status_t orth_conv_wgrad_workspace(orth_plan_t plan, int32_t layer, int32_t N, int32_t H, int32_t W, int32_t io,
                                        int64_t* bytes);
orth_status_t orth_conv_wgrad(orth_plan_t plan, int32_t layer, const void* x, const void* dy, float* dkernel_f32,
                              int32_t N, int32_t H, int32_t W, int32_t io, void* workspace, int64_t workspace_bytes,
                              void* stream);

/* Composition VJP: d(ortho) of this rank's units from dkernels_f32, the gradient of the FP32 kernels in the
 * FINAL layout (all layers; with world > 1 the data-parallel gradient is all-reduced first).  ortho: the
 * matrices the kernels were composed from.  Writes every owned unit's matrices in d_ortho (packed like
 * ortho); other entries untouched.  Recomputes the chain's intermediates (R32), then runs the adjoint of
 * each step: slice -> zero padding, AOC block convolution (dR, dK_BCOP), BCOP steps K' = K_cur P + K_prev
 * (I - P) -> (dK, dP), P = U U^T -> dU = (dP + dP^T) U, RKO reshape -> reshape.  Needs opts.vjp; AOC /
 * BCOP / RKO / dense layers only (SOC / SLL / blocks: ORTH_ERR_UNSUPPORTED_CONFIG). */
orth_status_t orth_compose_vjp(orth_plan_t plan, const float* ortho, const float* dkernels_f32, float* d_ortho,
                               void* stream);
/* Orthogonalisation VJP: d_params of this rank's matrices from d_ortho.  The pre-scale sigma is a constant
 * (R31: the value the LAST orth_orthogonalize of this plan computed -- call it on the same params first);
 * the T iterates X_t = NS^t(W / sigma) are recomputed FP32-accurately (FP32 SIMT, or 3-pass tcgen05 in the
 * BF16 modes: the adjoint of the FP32 iteration, R32) and the adjoint step
 * G <- G + b (G R + X S'), R = I - X^T X, S' = -(X^T G + G^T X) (tall; the mirrored form for wide) runs
 * T times; d_params = G_0 / sigma.  Needs opts.vjp. */
orth_status_t orth_orthogonalize_vjp(orth_plan_t plan, const float* params, const float* d_ortho, float* d_params,
                                     void* stream);

/* ---- f2: GPU spectral certification (App. C "scalable spectral norm
 * estimation ... check that the produced bounds are valid").
 * For layer `layer`'s FP32 kernel (PyTorch layout, as orth_compose_kernel writes it) and the circular
 * operator of its forward conv on an H x W grid (s | H, s | W; dense layers: H = W = 1), per group and per
 * frequency (f1, f2) of the (H/s) x (W/s) polyphase grid: E = M^H M - I on the short side of the
 * symbol M (c_out/g x (c_in/g) s^2), computed in FP64 from the FP32 values.
 *   out[((g * H/s + f1) * W/s + f2) * 2 + 0] = |E|_F   -- certificate: max|sigma - 1| <= max|sigma^2 - 1|
 *                                                          = |E|_2 <= |E|_F at that frequency;
 *   out[... + 1]                             = |E z|    -- power_iters power iterations of E from a fixed
 *                                                          start: a lower bound converging to |E|_2.
 * out: caller-owned device FP64 array; workspace: caller-owned device memory of at least
 * orth_certify_workspace(...) bytes (16-byte aligned).  Asynchronous on `stream`.  Errors:
 * SHAPE_MISMATCH (s does not divide H or W, dense with H*W != 1), INVALID_ARGUMENT (NULLs, small
 * workspace, power_iters < 0). */
orth_status_t orth_certify_workspace(orth_plan_t plan, int32_t layer, int32_t H, int32_t W, int64_t* bytes);
orth_status_t orth_certify(orth_plan_t plan, int32_t layer, const float* kernel_f32, int32_t H, int32_t W,
                           int32_t power_iters, void* workspace, int64_t workspace_bytes, double* out, void* stream);

/* ---- tracing: per-call timing of the plan's kernel groups ----------------------------
 * orth_plan_trace(plan, 1) makes every compute call bracket each group of kernels it launches (the
 * power pass, the NS launch, the composition, the emit, one conv call, ...) with a pair of CUDA events
 * on the call's stream; orth_plan_trace_read synchronises on them and returns the records in launch
 * order (then forgets them).  Tracing adds event records between kernels (it defeats the programmatic
 * dependent launch overlap and is not meant for CUDA-graph capture): use it in a separate, eager
 * profiling pass, never inside a timed region.  Every ABI call is also an NVTX range
 * ("orth_conv_forward", ...) whether or not tracing is on. */
typedef enum {
  ORTH_TK_POWER = 1,        /* pre-scaling: power iterations or Frobenius norms (power_fused_kernel) */
  ORTH_TK_SCALE = 2,        /* X0 = W / sigma (+ BF16 operand copies) */
  ORTH_TK_NS = 3,           /* the T Bjorck / NS iterations (one persistent launch, or 2T phases) */
  ORTH_TK_NS_CHECK = 4,     /* convergence check / residual reduction */
  ORTH_TK_COMPOSE = 5,      /* projectors + BCOP chain + RKO (*) BCOP */
  ORTH_TK_EMIT = 6,         /* kernels into the FP32 / BF16 layouts */
  ORTH_TK_CONV_FWD = 7,     /* one orth_conv_forward (variant = orth_conv_variant_t) */
  ORTH_TK_CONV_ADJ = 8,     /* one orth_conv_transpose */
  ORTH_TK_ASSEMBLE = 9,     /* orth_kernels_assemble */
  ORTH_TK_CERTIFY = 10,     /* orth_certify */
  ORTH_TK_WGRAD = 11,       /* orth_conv_wgrad */
  ORTH_TK_COMPOSE_VJP = 12, /* orth_compose_vjp */
  ORTH_TK_NS_VJP = 13       /* orth_orthogonalize_vjp */
} orth_trace_kind_t;
typedef enum {             /* which conv kernel a conv call ran */
  ORTH_CV_NONE = 0, ORTH_CV_SIMT = 1, ORTH_CV_SMALLK = 2, ORTH_CV_STEM = 3,
  ORTH_CV_WINDOW_SWAP = 4,  /* conv_pad<64, swapped>: TMA window, M = 64 channels x N = 256 pixels */
  ORTH_CV_WINDOW = 5,       /* conv_pad<BN>: TMA window, M = 128 pixels */
  ORTH_CV_STACK = 6,        /* conv_stack: padded copy + stacked windows, M = 128 ch x N = 256 px */
  ORTH_CV_TMA = 7,          /* conv_tma (experimental, ORTH_CONV_TMA=1) */
  ORTH_CV_GATHER256 = 8, ORTH_CV_GATHER128 = 9, ORTH_CV_GATHER64 = 10, ORTH_CV_GATHER32 = 11,  /* conv_ws<BN> */
  ORTH_CV_GATHER_PAIR = 12, /* conv_pair (experimental, ORTH_CONV_PAIR=1) */
  ORTH_CV_WINDOW_ROW = 13   /* conv_pad<64, row>: TMA window, M = 128 pixels x N = k * 64 (one kernel row's taps);
                               opt-in (ORTH_CONV_ROW=1) */
} orth_conv_variant_t;
typedef struct {
  int32_t kind;      /* orth_trace_kind_t */
  int32_t layer;     /* conv calls: the layer; else -1 */
  int32_t variant;   /* conv calls: orth_conv_variant_t; else 0 */
  int32_t launches;  /* kernels in the group */
  float ms;          /* CUDA-event time of the group */
} orth_trace_rec_t;
orth_status_t orth_plan_trace(orth_plan_t plan, int32_t enable);
/* Synchronises on the recorded events; copies up to `cap` records into `out` (NULL: none), sets *n to
 * the number of records available, and clears them. */
orth_status_t orth_plan_trace_read(orth_plan_t plan, orth_trace_rec_t* out, int32_t cap, int32_t* n);

/* Number of kernel launches enqueued by this plan since creation (all calls). */
int64_t orth_plan_launch_count(orth_plan_t plan);

const char* orth_status_string(orth_status_t status);
/* Build description, e.g. "sm_100a experimental=0" (experimental=1: the opt-in conv_tma / conv_pair kernels
 * that measured no faster are compiled in, ORTH_EXPERIMENTAL=1 at build time). */
const char* orth_build_info(void);
const char* orth_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ORTH_H_ */
