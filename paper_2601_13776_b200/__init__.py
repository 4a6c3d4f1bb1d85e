"""Python binding of the C-ABI library ``liborth.so`` (include/orth.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no CPU or PyTorch fallback: if the library is missing
the import fails, and compute calls on a host-only plan raise.

Module-level functions carry the ABI names (``orth_plan_create``,
``orth_orthogonalize``, ``orth_compose_kernel``, ``orth_conv_forward``,
``orth_conv_transpose``, ...); ``Plan`` wraps them for convenience.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborth.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is not built; run `python paper_2601_13776_b200/build.py` "
                      "(or __graft_entry__.build()). There is no fallback path.")
_lib = C.CDLL(_LIB_PATH)

# ---------------------------------------------------------------- ABI types
OK, INVALID_ARGUMENT, UNSUPPORTED_CONFIG, SHAPE_MISMATCH, ZERO_NORM, NOT_CONVERGED, CUDA_ERR, OOM, NO_DEVICE = range(9)
F32, BF16, BF16X3 = 0, 1, 2
PAD_ZEROS, PAD_CIRCULAR = 0, 1
CONV2D, CONV_TRANSPOSE2D, DENSE, SOC, SLL, SLL_BLOCK = 0, 1, 2, 3, 4, 5
PRESCALE_POWER, PRESCALE_FROBENIUS = 0, 1
Q = dict(N_LAYERS=0, N_MATRICES=1, PARAMS_NUMEL=2, CACHE_NUMEL=3, KERNELS_F32_NUMEL=4, KERNELS_BF16_NUMEL=5,
         WORKSPACE_BYTES=6, NS_FLOPS=7, KERNEL_SEGMENT_F32=8, KERNEL_SEGMENT_BF16=9, N_UNITS=10,
         GATHER_F32_NUMEL=11, GATHER_BF16_NUMEL=12, CONV_SCRATCH_BYTES=13, COMP_FLOPS=14,
         LAYER_FIRST_MATRIX=20, LAYER_MATS_PER_GROUP=21, LAYER_KERNEL_OFF_F32=22, LAYER_KERNEL_OFF_BF16=23,
         LAYER_KERNEL_NUMEL=24, LAYER_OWNER=25, LAYER_C_MID=26, LAYER_C_B=27, LAYER_KP=28, LAYER_SCRATCH_BYTES=29, LAYER_NS_FLOPS=30, LAYER_COMP_FLOPS=31, LAYER_K_EFF=32,
         LAYER_BLOCK_KC=33, LAYER_BLOCK_M_OFF=34, LAYER_BLOCK_PADS=35,
         MATRIX_ROWS=40, MATRIX_COLS=41, MATRIX_OFFSET=42, MATRIX_CACHE_OFFSET=43, MATRIX_LAYER=44,
         MATRIX_GROUP=45, MATRIX_ROLE=46, UNIT_LAYER=60, UNIT_GROUP=61, UNIT_OWNER=62, UNIT_NUMEL=63,
         UNIT_GATHER_OFF_F32=64, UNIT_GATHER_OFF_BF16=65, UNIT_KERNEL_OFF_F32=66, UNIT_KERNEL_OFF_BF16=67)
ROLES = {0: "Q", 1: "U", 2: "R", 3: "W", 4: "K"}
_KIND = {"conv": CONV2D, "convT": CONV_TRANSPOSE2D, "dense": DENSE, "soc": SOC, "sll": SLL, "sll_block": SLL_BLOCK}
_MODE = {"zeros": PAD_ZEROS, "circular": PAD_CIRCULAR}


TRACE_KINDS = {1: "power", 2: "scale", 3: "ns", 4: "ns_check", 5: "compose", 6: "emit", 7: "conv_fwd",
               8: "conv_adj", 9: "assemble", 10: "certify", 11: "wgrad", 12: "compose_vjp", 13: "ns_vjp"}
CONV_VARIANTS = {0: "none", 1: "conv_fwd_simt/conv_bwd_simt", 2: "conv_fwd_smallk", 3: "conv_stem_tc",
                 4: "conv_pad<64,swapped>", 5: "conv_pad<BN>", 6: "conv_stack (+pad_kernel)", 7: "conv_tma",
                 8: "conv_ws<256>", 9: "conv_ws<128>", 10: "conv_ws<64>", 11: "conv_ws<32>", 12: "conv_pair",
                 13: "conv_pad<64,row>"}


class TraceRec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("variant", C.c_int32), ("launches", C.c_int32),
                ("ms", C.c_float)]


class LayerDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "c_in", "c_out", "k_h", "k_w", "stride_h", "stride_w", "dil_h",
                                         "dil_w", "groups", "pad_t", "pad_b", "pad_l", "pad_r", "padding_mode",
                                         "grid_h", "grid_w", "soc_terms", "blk_pre", "blk_sll", "blk_post")]


class Opts(C.Structure):
    _fields_ = [("ns_iters", C.c_int32), ("beta", C.c_float), ("prescale", C.c_int32), ("power_iters", C.c_int32),
                ("compute", C.c_int32), ("polish_iters", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("ns_tol", C.c_float), ("max_batch", C.c_int32), ("vjp", C.c_int32)]


_P = C.c_void_p
_sig = {
    "orth_opts_default": (None, [C.POINTER(Opts)]),
    "orth_validate_desc": (C.c_int, [C.POINTER(LayerDesc), C.c_int32, C.POINTER(Opts)]),
    "orth_plan_create": (C.c_int, [C.POINTER(LayerDesc), C.c_int32, C.POINTER(Opts), C.c_int32, C.POINTER(_P)]),
    "orth_plan_destroy": (C.c_int, [_P]),
    "orth_plan_query": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "orth_orthogonalize": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "orth_compose_kernel": (C.c_int, [_P, _P, _P, _P, _P]),
    "orth_conv_forward": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "orth_conv_transpose": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "orth_kernels_assemble": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "orth_plan_check": (C.c_int, [_P, _P]),
    "orth_compose_vjp": (C.c_int, [_P, _P, _P, _P, _P]),
    "orth_orthogonalize_vjp": (C.c_int, [_P, _P, _P, _P, _P]),
    "orth_conv_wgrad_workspace": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.POINTER(C.c_int64)]),
    "orth_conv_wgrad": (C.c_int, [_P, C.c_int32, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64,
                                  _P]),
    "orth_certify_workspace": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "orth_certify": (C.c_int, [_P, C.c_int32, _P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64, _P, _P]),
    "orth_plan_trace": (C.c_int, [_P, C.c_int32]),
    "orth_plan_trace_read": (C.c_int, [_P, C.POINTER(TraceRec), C.c_int32, C.POINTER(C.c_int32)]),
    "orth_plan_launch_count": (C.c_int64, [_P]),
    "orth_status_string": (C.c_char_p, [C.c_int]),
    "orth_build_info": (C.c_char_p, []),
    "orth_last_error": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
EXPORTED = tuple(_sig)


class OrthError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.orth_status_string(status).decode()
        detail = (_lib.orth_last_error() or b"").decode()
        super().__init__(f"{where}: {msg}: {detail}")


def _check(st: int, where: str):
    if st != OK:
        raise OrthError(st, where)


def layer_grid(d: Dict):
    """Declared forward-conv input grid (grid_h, grid_w) of a layer dict: ``grid`` if given, else from
    synth's ``H`` (the call's input size; a transposed layer's large grid is H * s), else (0, 0)."""
    if d.get("grid"):
        return tuple(d["grid"])
    H = d.get("H", 0) or 0
    if d.get("kind") == "convT":
        H *= d.get("s", 1)
    return (H, H)


def layer_desc(d: Dict) -> LayerDesc:
    """Marshal a synth.configs-style dict into orth_layer_desc_t."""
    pads = d.get("pad") or (-1, -1, -1, -1)
    k, s, dl = d.get("k", 3), d.get("s", 1), d.get("d", 1)
    gh, gw = layer_grid(d) if d.get("kind", "conv") != "dense" else (0, 0)
    return LayerDesc(_KIND[d.get("kind", "conv")], d["c_in"], d["c_out"], k, k, s, s, dl, dl, d.get("g", 1),
                     pads[0], pads[1], pads[2], pads[3], _MODE[d.get("padding_mode", "circular")], gh, gw,
                     d.get("terms", 0), d.get("pre", 0), d.get("sll", 0), d.get("post", 0))


def make_opts(**kw) -> Opts:
    o = Opts()
    _lib.orth_opts_default(C.byref(o))
    for k, v in kw.items():
        if k == "compute" and isinstance(v, str):
            v = {"f32": F32, "bf16": BF16, "bf16x3": BF16X3}[v]
        if k == "prescale" and isinstance(v, str):
            v = {"power": PRESCALE_POWER, "frobenius": PRESCALE_FROBENIUS}[v]
        setattr(o, k, v)
    return o


def orth_validate_desc(layers: Sequence[Dict], **opts) -> int:
    arr = (LayerDesc * len(layers))(*[layer_desc(d) for d in layers])
    o = make_opts(**opts)
    return _lib.orth_validate_desc(arr, len(layers), C.byref(o))


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    import torch
    return torch.cuda.current_stream().cuda_stream


def orth_plan_create(layers: Sequence[Dict], device: int = 0, **opts) -> int:
    arr = (LayerDesc * len(layers))(*[layer_desc(d) for d in layers])
    o = make_opts(**opts)
    h = _P()
    _check(_lib.orth_plan_create(arr, len(layers), C.byref(o), device, C.byref(h)), "orth_plan_create")
    return h.value


def orth_plan_destroy(h: int):
    _check(_lib.orth_plan_destroy(h), "orth_plan_destroy")


def orth_plan_query(h: int, what, index: int = 0) -> int:
    out = C.c_int64()
    w = Q[what] if isinstance(what, str) else what
    _check(_lib.orth_plan_query(h, w, index, C.byref(out)), "orth_plan_query")
    return out.value


def orth_orthogonalize(h: int, params, ortho_out, power_cache=None, residual_out=None, stream=None):
    _check(_lib.orth_orthogonalize(h, _ptr(params), _ptr(ortho_out), _ptr(power_cache), _ptr(residual_out),
                                   _stream(stream)), "orth_orthogonalize")


def orth_compose_kernel(h: int, ortho, kernels_f32, kernels_bf16=None, stream=None):
    _check(_lib.orth_compose_kernel(h, _ptr(ortho), _ptr(kernels_f32), _ptr(kernels_bf16), _stream(stream)),
           "orth_compose_kernel")


def orth_conv_forward(h: int, layer: int, kernel, x, y, N: int, H: int, W: int, io: int, bias=None, stream=None):
    _check(_lib.orth_conv_forward(h, layer, _ptr(kernel), _ptr(bias), _ptr(x), _ptr(y), N, H, W, io,
                                  _stream(stream)), "orth_conv_forward")


def orth_conv_transpose(h: int, layer: int, kernel, y_small, x_big, N: int, H_big: int, W_big: int, io: int,
                        bias=None, stream=None):
    _check(_lib.orth_conv_transpose(h, layer, _ptr(kernel), _ptr(bias), _ptr(y_small), _ptr(x_big), N, H_big, W_big,
                                    io, _stream(stream)), "orth_conv_transpose")


def orth_kernels_assemble(h: int, gathered_f32, kernels_f32, gathered_bf16=None, kernels_bf16=None, stream=None):
    _check(_lib.orth_kernels_assemble(h, _ptr(gathered_f32), _ptr(kernels_f32), _ptr(gathered_bf16),
                                      _ptr(kernels_bf16), _stream(stream)), "orth_kernels_assemble")


def orth_compose_vjp(h: int, ortho, dkernels_f32, d_ortho, stream=None):
    _check(_lib.orth_compose_vjp(h, _ptr(ortho), _ptr(dkernels_f32), _ptr(d_ortho), _stream(stream)),
           "orth_compose_vjp")


def orth_orthogonalize_vjp(h: int, params, d_ortho, d_params, stream=None):
    _check(_lib.orth_orthogonalize_vjp(h, _ptr(params), _ptr(d_ortho), _ptr(d_params), _stream(stream)),
           "orth_orthogonalize_vjp")


def orth_conv_wgrad_workspace(h: int, layer: int, N: int, H: int, W: int, io: int) -> int:
    out = C.c_int64()
    _check(_lib.orth_conv_wgrad_workspace(h, layer, N, H, W, io, C.byref(out)), "orth_conv_wgrad_workspace")
    return out.value


def orth_conv_wgrad(h: int, layer: int, x, dy, dkernel, N: int, H: int, W: int, io: int, workspace=None,
                    stream=None):
    nb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.orth_conv_wgrad(h, layer, _ptr(x), _ptr(dy), _ptr(dkernel), N, H, W, io, _ptr(workspace), nb,
                                _stream(stream)), "orth_conv_wgrad")


def orth_certify_workspace(h: int, layer: int, H: int, W: int) -> int:
    out = C.c_int64()
    _check(_lib.orth_certify_workspace(h, layer, H, W, C.byref(out)), "orth_certify_workspace")
    return out.value


def orth_certify(h: int, layer: int, kernel_f32, H: int, W: int, power_iters: int, workspace, out, stream=None):
    _check(_lib.orth_certify(h, layer, _ptr(kernel_f32), H, W, power_iters, _ptr(workspace),
                             workspace.numel() * workspace.element_size(), _ptr(out), _stream(stream)),
           "orth_certify")


def orth_plan_check(h: int, stream=None):
    _check(_lib.orth_plan_check(h, _stream(stream)), "orth_plan_check (device status)")


def orth_plan_trace(h: int, enable: bool):
    _check(_lib.orth_plan_trace(h, 1 if enable else 0), "orth_plan_trace")


def orth_plan_trace_read(h: int) -> List[Dict]:
    n = C.c_int32()
    cap = 4096
    buf = (TraceRec * cap)()
    _check(_lib.orth_plan_trace_read(h, buf, cap, C.byref(n)), "orth_plan_trace_read")
    return [dict(kind=TRACE_KINDS.get(r.kind, str(r.kind)), layer=r.layer, variant=CONV_VARIANTS.get(r.variant, ""),
                 launches=r.launches, ms=r.ms) for r in buf[: min(n.value, cap)]]


def experimental() -> bool:
    return b"experimental=1" in _lib.orth_build_info()


def orth_plan_launch_count(h: int) -> int:
    return _lib.orth_plan_launch_count(h)


def out_size(H: int, k: int, s: int, d: int, p0: int, p1: int) -> int:
    return (H + p0 + p1 - d * (k - 1) - 1) // s + 1


class Plan:
    """Owns an orth_plan_t.  ``layers``: synth.configs-style dicts."""

    def __init__(self, layers: Sequence[Dict], device: int = 0, **opts):
        self.layers = [dict(d) for d in layers]
        self.device = device
        self.h = orth_plan_create(self.layers, device, **opts)
        q = lambda w, i=0: orth_plan_query(self.h, w, i)
        self.n_layers = q("N_LAYERS")
        self.n_matrices = q("N_MATRICES")
        self.params_numel = q("PARAMS_NUMEL")
        self.cache_numel = q("CACHE_NUMEL")
        self.kf32_numel = q("KERNELS_F32_NUMEL")
        self.kbf16_numel = q("KERNELS_BF16_NUMEL")
        self.workspace_bytes = q("WORKSPACE_BYTES")
        self.ns_flops = q("NS_FLOPS")
        self.world = opts.get("world", 1)
        self.rank = opts.get("rank", 0)
        self.gf32_numel = q("GATHER_F32_NUMEL")
        self.gbf16_numel = q("GATHER_BF16_NUMEL")
        self.seg_f32 = q("KERNEL_SEGMENT_F32")
        self.seg_bf16 = q("KERNEL_SEGMENT_BF16")
        self.conv_scratch_bytes = q("CONV_SCRATCH_BYTES")
        self.units = [dict(layer=q("UNIT_LAYER", u), group=q("UNIT_GROUP", u), owner=q("UNIT_OWNER", u),
                           numel=q("UNIT_NUMEL", u), gat_f32=q("UNIT_GATHER_OFF_F32", u),
                           gat_bf16=q("UNIT_GATHER_OFF_BF16", u), fin_f32=q("UNIT_KERNEL_OFF_F32", u),
                           fin_bf16=q("UNIT_KERNEL_OFF_BF16", u)) for u in range(q("N_UNITS"))]
        self.matrices = [dict(m=q("MATRIX_ROWS", i), n=q("MATRIX_COLS", i), off=q("MATRIX_OFFSET", i),
                              cache_off=q("MATRIX_CACHE_OFFSET", i), layer=q("MATRIX_LAYER", i),
                              group=q("MATRIX_GROUP", i), role=ROLES[q("MATRIX_ROLE", i)])
                         for i in range(self.n_matrices)]
        self.layer_info = [dict(first_matrix=q("LAYER_FIRST_MATRIX", l), mats_per_group=q("LAYER_MATS_PER_GROUP", l),
                                kf32_off=q("LAYER_KERNEL_OFF_F32", l), kbf16_off=q("LAYER_KERNEL_OFF_BF16", l),
                                numel=q("LAYER_KERNEL_NUMEL", l), owner=q("LAYER_OWNER", l),
                                c_mid=q("LAYER_C_MID", l), c_b=q("LAYER_C_B", l), kp=q("LAYER_KP", l),
                                scratch=q("LAYER_SCRATCH_BYTES", l), k_eff=q("LAYER_K_EFF", l),
                                kc=q("LAYER_BLOCK_KC", l), m_off=q("LAYER_BLOCK_M_OFF", l),
                                pads=q("LAYER_BLOCK_PADS", l))
                           for l in range(self.n_layers)]

    # -- shapes ---------------------------------------------------------
    def fwd_channels(self, l: int):
        d = self.layers[l]
        return (d["c_out"], d["c_in"]) if d.get("kind") == "convT" else (d["c_in"], d["c_out"])

    def kernel_shape(self, l: int):
        d = self.layers[l]
        if d.get("kind") == "dense":
            return (d["c_out"], d["c_in"])
        ci, co = self.fwd_channels(l)
        k = self.layer_info[l]["k_eff"]
        return (co, ci // d.get("g", 1), k, k)

    def block_kernels(self, kbuf, l: int):
        """SLL block l: views (C, M) of its merged kernels in kbuf (FP32 PyTorch layout (c_s, c, kC, kC) and
        (c_out, c + c_s, kM, kM), or BF16 GEMM layout (C_o, k, k, C_i) when kbuf is bfloat16)."""
        d, info = self.layers[l], self.layer_info[l]
        c, co = d["c_in"], d["c_out"]
        cs = self.layers[d["sll"]]["c_out"]
        kc, km = info["kc"], info["k_eff"]
        off = info["kbf16_off"] if str(kbuf.dtype) == "torch.bfloat16" else info["kf32_off"]
        C = kbuf[off: off + cs * c * kc * kc]
        M = kbuf[off + info["m_off"]: off + info["m_off"] + co * (c + cs) * km * km]
        if str(kbuf.dtype) == "torch.bfloat16":
            return C.view(cs, kc, kc, c), M.view(co, km, km, c + cs)
        return C.view(cs, c, kc, kc), M.view(co, c + cs, km, km)

    def kernel_f32(self, kf32, l: int):
        info = self.layer_info[l]
        return kf32[info["kf32_off"]: info["kf32_off"] + info["numel"]].view(self.kernel_shape(l))

    def kernel_bf16(self, kbf16, l: int):
        info = self.layer_info[l]
        sh = self.kernel_shape(l)
        v = kbf16[info["kbf16_off"]: info["kbf16_off"] + info["numel"]]
        return v.view(sh) if len(sh) == 2 else v.view(sh[0], sh[2], sh[3], sh[1])

    def out_hw(self, l: int, H: int, W: int):
        d = self.layers[l]
        k, s, dl = self.layer_info[l]["k_eff"], d.get("s", 1), d.get("d", 1)
        pads = d.get("pad")
        if d.get("kind") == "sll_block":
            pm = self.layer_info[l]["pads"] >> 16
            pads = (pm, k - 1 - pm, pm, k - 1 - pm)
        if pads is None:
            e = dl * (k - 1)
            pads = (e // 2, e - e // 2, e // 2, e - e // 2)
        return out_size(H, k, s, dl, pads[0], pads[1]), out_size(W, k, s, dl, pads[2], pads[3])

    # -- compute ----------------------------------------------------------
    def orthogonalize(self, params, ortho_out, power_cache=None, residual_out=None, stream=None):
        orth_orthogonalize(self.h, params, ortho_out, power_cache, residual_out, stream)

    def compose(self, ortho, kernels_f32, kernels_bf16=None, stream=None):
        """world == 1: final layout (kf32_numel / kbf16_numel); world > 1: this rank's units into its
        segment of the gather layout (gf32_numel / gbf16_numel)."""
        orth_compose_kernel(self.h, ortho, kernels_f32, kernels_bf16, stream)

    def assemble(self, gathered_f32, kernels_f32, gathered_bf16=None, kernels_bf16=None, stream=None):
        """a8: all-gathered gather layout -> final layout (world > 1)."""
        orth_kernels_assemble(self.h, gathered_f32, kernels_f32, gathered_bf16, kernels_bf16, stream)

    def conv_forward(self, l: int, kernel, x, y, bias=None, stream=None):
        """x: NHWC (N, H, W, C_i) float32 or bfloat16 CUDA tensor; y preallocated."""
        io = BF16 if str(x.dtype) == "torch.bfloat16" else F32
        N, H, W, _ = x.shape
        orth_conv_forward(self.h, l, kernel, x, y, N, H, W, io, bias, stream)

    def conv_transpose(self, l: int, kernel, y_small, x_big, bias=None, stream=None):
        io = BF16 if str(y_small.dtype) == "torch.bfloat16" else F32
        N, H, W, _ = x_big.shape
        orth_conv_transpose(self.h, l, kernel, y_small, x_big, N, H, W, io, bias, stream)

    def check(self, stream=None):
        orth_plan_check(self.h, stream)

    def compose_vjp(self, ortho, dkernels_f32, d_ortho, stream=None):
        orth_compose_vjp(self.h, ortho, dkernels_f32, d_ortho, stream)

    def orthogonalize_vjp(self, params, d_ortho, d_params, stream=None):
        orth_orthogonalize_vjp(self.h, params, d_ortho, d_params, stream)

    def conv_wgrad(self, l: int, x, dy, dkernel, workspace=None, stream=None):
        """f1: dK (FP32 PyTorch layout, preallocated) of layer l's forward-conv view from x (large grid, NHWC)
        and dy (output grid); the split workspace is allocated here if not given (caller-owned memory)."""
        import torch
        io = BF16 if str(x.dtype) == "torch.bfloat16" else F32
        N, H, W, _ = x.shape
        nb = orth_conv_wgrad_workspace(self.h, l, N, H, W, io)
        if workspace is None and nb > 0:
            workspace = torch.empty(nb, dtype=torch.uint8, device=x.device)
        orth_conv_wgrad(self.h, l, x, dy, dkernel, N, H, W, io, workspace, stream)

    def certify(self, l: int, kernel_f32, H: int, W: int, power_iters: int = 30, workspace=None, stream=None):
        """f2: per (group, frequency) [|E|_F, power estimate of |E|_2] (FP64 tensor on the kernel's device),
        shape (g, H/s, W/s, 2); E = M^H M - I of the circular operator's symbol on the short side."""
        import torch
        nb = orth_certify_workspace(self.h, l, H, W)
        if workspace is None:
            workspace = torch.empty(nb, dtype=torch.uint8, device=kernel_f32.device)
        d = self.layers[l]
        s = 1 if d.get("kind") == "dense" else d.get("s", 1)
        g = 1 if d.get("kind") == "dense" else d.get("g", 1)
        out = torch.empty((g, H // s, W // s, 2), dtype=torch.float64, device=kernel_f32.device)
        orth_certify(self.h, l, kernel_f32, H, W, power_iters, workspace, out, stream)
        return out

    def trace(self, enable: bool = True):
        orth_plan_trace(self.h, enable)

    def trace_read(self) -> List[Dict]:
        return orth_plan_trace_read(self.h)

    @property
    def launches(self) -> int:
        return orth_plan_launch_count(self.h)

    def close(self):
        if getattr(self, "h", None):
            orth_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
