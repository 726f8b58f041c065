"""Python driver of libdpg.so (include/dpg.h) — plumbing for tests, smoke() and bench.py.

The product is the C ABI and the sm_100a kernels behind it; this module only passes device
pointers of torch CUDA tensors (torch is used for device memory and streams) and maps status
codes onto exception classes named after the reference's (errors.hpp:12-72). Class and method
names mirror the reference API: GradSampleModule.forward_backward, DpOptimizer.{virtual_step,
step, step_empty_batch, zero_grad, last_clip_summary}, per_sample_rule_{linear,conv2d,embedding},
clip_and_sum, add_noise.

There is no fallback: if libdpg.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import torch

from .configs import LayerDesc, c_layers, params_meta

HERE = os.path.dirname(os.path.abspath(__file__))
# DPG_LIB: an alternative in-tree build of the same sources (A/B experiments only)
LIB_PATH = os.path.join(HERE, os.environ.get("DPG_LIB", "libdpg.so"))

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int


class DpgError(RuntimeError):
    code = -1

    def __init__(self, msg: str):
        super().__init__(msg)
        self.msg = msg


class DimensionError(DpgError):
    code = 1


class ParameterError(DpgError):
    code = 2


class LifecycleError(DpgError):
    code = 3


class RegistryError(DpgError):
    code = 4


class NumericError(DpgError):
    code = 5


class CudaError(DpgError):
    code = 6


class NcclError(DpgError):
    code = 7


_ERRS = {c.code: c for c in (DimensionError, ParameterError, LifecycleError, RegistryError,
                             NumericError, CudaError, NcclError)}


class dpg_conv2d_spec(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("in_channels", "out_channels", "kernel_h", "kernel_w", "stride", "padding")]


class dpg_optimizer_config(ctypes.Structure):
    _fields_ = [("noise_multiplier", ctypes.c_double), ("max_grad_norm", ctypes.c_double),
                ("learning_rate", ctypes.c_double), ("expected_batch_size", ctypes.c_double),
                ("noise_seed", ctypes.c_uint64), ("materialise_grad_sample", ctypes.c_int32),
                ("clipped_sum_from_record", ctypes.c_int32)]


# exported symbols and their argument types (everything include/dpg.h declares)
_SIGS = {
    "dpg_abi_version": (ctypes.c_int, []),
    "dpg_tg_gemm_selftest": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32]),
    "dpg_tg_gemm_selftest_split": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32]),
    "dpg_noise_schedule_init": (_I32, [_P, _I32, _D, _D, _D, ctypes.c_uint64, _P, _I64]),
    "dpg_noise_schedule_sigma_at": (_D, [_P, ctypes.c_uint64]),
    "dpg_schedule_noise": (_I32, [_P, ctypes.c_uint64, _P, _P]),
    "dpg_rdp_subsampled_gaussian": (_I32, [_D, _D, _I32, _P]),
    "dpg_accountant_create": (_I32, [_P, _I32, ctypes.POINTER(_P)]),
    "dpg_accountant_destroy": (None, [_P]),
    "dpg_accountant_num_orders": (_I32, [_P]),
    "dpg_accountant_step": (_I32, [_P, _D, _D, _I64]),
    "dpg_accountant_rdp": (_I32, [_P, _P, _P]),
    "dpg_accountant_epsilon": (_I32, [_P, _D, _P, _P]),
    "dpg_get_noise_multiplier": (_I32, [_D, _D, _D, _I64, _D, _D, _P]),
    "dpg_grad_sample_export": (_I32, [_P, _I32, _P, _I64]),
    "dpg_ctx_create": (_I32, [_I32, _P, ctypes.POINTER(_P)]),
    "dpg_ctx_destroy": (None, [_P]),
    "dpg_ctx_stream": (_P, [_P]),
    "dpg_last_error": (ctypes.c_char_p, [_P]),
    "dpg_ctx_sync": (_I32, [_P]),
    "dpg_ctx_kernel_launches": (_I64, [_P]),
    "dpg_ctx_set_profiling": (_I32, [_P, _I32]),
    "dpg_ctx_profile_read": (ctypes.c_char_p, [_P]),
    "dpg_ctx_set_timeline": (_I32, [_P, _I32]),
    "dpg_ctx_timeline_read": (ctypes.c_char_p, [_P]),
    "dpg_nccl_unique_id": (_I32, [ctypes.c_char_p]),
    "dpg_ctx_init_comm": (_I32, [_P, _I32, _I32, ctypes.c_char_p]),
    "dpg_allreduce_sum": (_I32, [_P, _P, _I64]),
    "dpg_grad_sample_linear": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "dpg_grad_sample_conv2d": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P]),
    "dpg_grad_sample_embedding": (_I32, [_P, _P, _P, _I64, _I64, _I64, _I64, _P, _P]),
    "dpg_clip_factors": (_I32, [_P, _P, _I32, _I64, _D, _P, _P, _P]),
    "dpg_clipped_sum_linear": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _I32]),
    "dpg_clipped_sum_conv2d": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _I32]),
    "dpg_clipped_sum_embedding": (_I32, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I32]),
    "dpg_clip_and_sum_materialised": (_I32, [_P, _P, _P, _I32, _I64, _D, _P, _P, _P, _P, _I32]),
    "dpg_noise_update": (_I32, [_P, _P, _P, _P, _I64, _D, _D, _D, _D, _U64, _U64, _P]),
    "dpg_gaussian": (_I32, [_P, _P, _I64, _D, _U64, _U64]),
    "dpg_model_create": (_I32, [_P, _P, _I32, _P, _I32, _I64, ctypes.POINTER(_P)]),
    "dpg_model_destroy": (None, [_P]),
    "dpg_model_parameter_count": (_I64, [_P]),
    "dpg_model_num_param_tensors": (_I32, [_P]),
    "dpg_model_param_info": (_I32, [_P, _I32, _P, _P, _P, _P]),
    "dpg_model_params": (_P, [_P]),
    "dpg_model_load_params": (_I32, [_P, _P]),
    "dpg_model_store_params": (_I32, [_P, _P]),
    "dpg_model_output_width": (_I64, [_P]),
    "dpg_optimizer_create": (_I32, [_P, _P, ctypes.POINTER(_P)]),
    "dpg_optimizer_peer_handle": (_I32, [_P, _P]),
    "dpg_grad_sample_linear_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _I64]),
    "dpg_grad_sample_conv2d_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _P]),
    "dpg_grad_sample_embedding_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _I64]),
    "dpg_clipped_sum_linear_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _I64]),
    "dpg_clipped_sum_conv2d_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _P]),
    "dpg_clipped_sum_embedding_workspace_size": (ctypes.c_size_t, [_I64, _I64, _I64, _I64]),
    "dpg_ctx_reserve_workspace": (_I32, [_P, ctypes.c_size_t]),
    "dpg_optimizer_set_peers": (_I32, [_P, ctypes.c_int, ctypes.c_int, _P]),
    "dpg_optimizer_destroy": (None, [_P]),
    "dpg_forward_backward": (_I32, [_P, _P, _P, _I64, _P]),
    "dpg_virtual_step": (_I32, [_P]),
    "dpg_step": (_I32, [_P]),
    "dpg_step_empty_batch": (_I32, [_P]),
    "dpg_zero_grad": (_I32, [_P]),
    "dpg_set_noise_multiplier": (_I32, [_P, _D]),
    "dpg_set_expected_batch_size": (_I32, [_P, _D]),
    "dpg_set_injected_noise": (_I32, [_P, _P]),
    "dpg_last_clip_summary": (_I32, [_P, _P, _P, _P]),
    "dpg_grad_sample": (_P, [_P]),
    "dpg_summed_grad": (_P, [_P]),
    "dpg_grad": (_P, [_P]),
    "dpg_accumulated_samples": (_I64, [_P]),
    "dpg_train_step_host": (_I32, [_P, _P, _P, _I64, _P]),
    "dpg_train_step_host_async": (_I32, [_P, _P, _P, _I64, _P]),
    "dpg_train_step": (_I32, [_P, _P, _P, _I64, _P, _I32]),
    "dpg_grad_sample_layer_norm": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "dpg_grad_sample_group_norm": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libdpg.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with __graft_entry__.build()")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def exported_symbols() -> List[str]:
    return list(_SIGS)


def _check(code: int, ctx=None):
    if code != 0:
        msg = lib().dpg_last_error(ctx).decode()
        raise _ERRS.get(code, DpgError)(msg)


def _p(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return ctypes.c_void_p(t.data_ptr())


class _Handle:
    """A native handle shared by its Python owner and the owner's parent, so the handles of a
    garbage cycle (context <- model <- optimizer, collected in arbitrary order) are still
    destroyed children first: whichever finaliser runs first destroys the handle and its
    children, the other finds it dead."""

    def __init__(self, h, destroy: str):
        self.h = h
        self.destroy_fn = destroy
        self.children: List["_Handle"] = []

    def destroy(self):
        if self.h is None:
            return
        for c in reversed(self.children):
            c.destroy()
        self.children = []
        if _lib is not None:
            getattr(_lib, self.destroy_fn)(self.h)
        self.h = None


class Context:
    """dpg_ctx on one GPU, bound to torch's current stream so ordering with torch ops holds."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        self.device = device
        torch.cuda.set_device(device)
        s = stream if stream is not None else torch.cuda.current_stream(device)
        if s.cuda_stream == 0:
            # the legacy default stream cannot be graph-captured: give torch and libdpg one
            # shared side stream so their work stays ordered
            s = torch.cuda.Stream(device)
            torch.cuda.set_stream(s)
        self.stream = s
        h = _P()
        _check(lib().dpg_ctx_create(device, ctypes.c_void_p(s.cuda_stream), ctypes.byref(h)))
        self.h = h
        self._handle = _Handle(h, "dpg_ctx_destroy")

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            self._handle.destroy()
            self.h = None

    def sync(self):
        _check(lib().dpg_ctx_sync(self.h), self.h)

    def reserve_workspace(self, nbytes: int):
        """Pre-size the operator workspace arena (dpg_ctx_reserve_workspace)."""
        _check(lib().dpg_ctx_reserve_workspace(self.h, nbytes), self.h)

    @property
    def kernel_launches(self) -> int:
        return int(lib().dpg_ctx_kernel_launches(self.h))

    def set_profiling(self, on: bool):
        _check(lib().dpg_ctx_set_profiling(self.h, int(on)), self.h)

    def profile(self):
        """{stage: {"ms": total, "count": n, "bytes": algorithmic bytes total, "flops": ...,
        "kernels": launches total, "seq": enqueue order of the first occurrence}}"""
        txt = lib().dpg_ctx_profile_read(self.h).decode()
        out = {}
        for line in txt.strip().splitlines():
            name, ms, cnt, by, fl, kern, seq = line.split()
            out[name] = {"ms": float(ms), "count": int(cnt), "bytes": float(by), "flops": float(fl),
                         "kernels": int(kern), "seq": int(seq)}
        return out

    def set_timeline(self, on: bool):
        """Record the stage scopes of steps captured from now on as graph event nodes."""
        _check(lib().dpg_ctx_set_timeline(self.h, int(on)), self.h)

    def timeline(self):
        """[(stage, start_ms, duration_ms, kernels)] of the last replay, in capture order."""
        txt = lib().dpg_ctx_timeline_read(self.h).decode()
        out = []
        for line in txt.strip().splitlines():
            name, t0, dt, kern = line.split()
            out.append((name, float(t0), float(dt), int(kern)))
        return out

    def init_comm(self, nranks: int, rank: int, uid: bytes):
        _check(lib().dpg_ctx_init_comm(self.h, nranks, rank, uid), self.h)

    def allreduce_sum(self, buf: torch.Tensor):
        _check(lib().dpg_allreduce_sum(self.h, _p(buf), buf.numel()), self.h)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().dpg_nccl_unique_id(buf))
        return buf.raw


# ---------------------------------------------------------------------------------------------
# Operator ABI (per-layer rules, clip, noise) — the GradSampleRule / clip_and_sum / add_noise
# entry points of the reference.
# ---------------------------------------------------------------------------------------------

def _f32(shape, device):
    return torch.empty(shape, dtype=torch.float32, device=device)


def per_sample_rule_linear(ctx: Context, acts: torch.Tensor, highway: torch.Tensor, bias=True,
                           grad=True, norms=True):
    """grad_sample.hpp:53-59. acts [b, mid..., d], highway [b, mid..., r] ->
    (gw [b, r, d] | None, gb [b, r] | None, sq_w [b] | None, sq_b [b] | None)."""
    b, d, r = acts.shape[0], acts.shape[-1], highway.shape[-1]
    mid = acts.numel() // max(1, b * d)
    dev = acts.device
    gw = _f32((b, r, d), dev) if grad else None
    gb = _f32((b, r), dev) if (grad and bias) else None
    sw = torch.empty(b, dtype=torch.float64, device=dev) if norms else None
    sb = torch.empty(b, dtype=torch.float64, device=dev) if (norms and bias) else None
    _check(lib().dpg_grad_sample_linear(ctx.h, _p(acts), _p(highway), b, mid, d, r, _p(gw), _p(gb),
                                        _p(sw), _p(sb)), ctx.h)
    return gw, gb, sw, sb


def _spec(ic, oc, kh, kw, stride, pad):
    return dpg_conv2d_spec(ic, oc, kh, kw, stride, pad)


def workspace_size(op: str, *extents) -> int:
    """Context-arena bytes an operator takes (dpg_<op>_workspace_size; host-only, no GPU needed).
    conv2d ops take (b, h, w, ic, oc, kh, kw, stride, pad), the others their ABI extents."""
    fn = getattr(lib(), f"dpg_{op}_workspace_size")
    if op.endswith("conv2d"):
        b, h, w, ic, oc, kh, kw, stride, pad = extents
        spec = _spec(ic, oc, kh, kw, stride, pad)
        return int(fn(b, h, w, ctypes.byref(spec)))
    return int(fn(*extents))


def per_sample_rule_conv2d(ctx: Context, x: torch.Tensor, highway: torch.Tensor, kh: int, kw: int,
                           stride: int, pad: int, bias=True, grad=True, norms=True):
    """grad_sample.hpp:135-150. x [b, ic, h, w], highway [b, oc, oh, ow]."""
    b, ic, h, w = x.shape
    oc = highway.shape[1]
    dev = x.device
    gw = _f32((b, oc, ic, kh, kw), dev) if grad else None
    gb = _f32((b, oc), dev) if (grad and bias) else None
    sw = torch.empty(b, dtype=torch.float64, device=dev) if norms else None
    sb = torch.empty(b, dtype=torch.float64, device=dev) if (norms and bias) else None
    spec = _spec(ic, oc, kh, kw, stride, pad)
    _check(lib().dpg_grad_sample_conv2d(ctx.h, _p(x), _p(highway), b, h, w, ctypes.byref(spec),
                                        _p(gw), _p(gb), _p(sw), _p(sb)), ctx.h)
    return gw, gb, sw, sb


def per_sample_rule_embedding(ctx: Context, idx: torch.Tensor, highway: torch.Tensor, vocab: int,
                              dense=True, norms=True):
    """grad_sample.hpp:64-82. idx [b, t] float ids, highway [b, t, dim] -> (g [b, V, dim] | None, sq)."""
    b, t = idx.shape
    dim = highway.shape[-1]
    g = _f32((b, vocab, dim), idx.device) if dense else None
    sq = torch.empty(b, dtype=torch.float64, device=idx.device) if norms else None
    _check(lib().dpg_grad_sample_embedding(ctx.h, _p(idx), _p(highway), b, t, vocab, dim, _p(g),
                                           _p(sq)), ctx.h)
    return g, sq


def per_sample_rule_layer_norm(ctx: Context, normalized: torch.Tensor, highway: torch.Tensor):
    """grad_sample.hpp:87-108. normalized / highway [b, ..., m] -> (ggamma [b, m], gbeta [b, m],
    sq_gamma [b], sq_beta [b])."""
    b, m = normalized.shape[0], normalized.shape[-1]
    positions = normalized.numel() // max(1, b * m)
    dev = normalized.device
    gg, gb = _f32((b, m), dev), _f32((b, m), dev)
    sg = torch.empty(b, dtype=torch.float64, device=dev)
    sb = torch.empty(b, dtype=torch.float64, device=dev)
    _check(lib().dpg_grad_sample_layer_norm(ctx.h, _p(normalized), _p(highway), b, positions, m, _p(gg),
                                            _p(gb), _p(sg), _p(sb)), ctx.h)
    return gg, gb, sg, sb


def per_sample_rule_group_norm(ctx: Context, normalized: torch.Tensor, highway: torch.Tensor):
    """grad_sample.hpp:110-131. normalized / highway [b, C, ...] -> (ggamma [b, C], gbeta [b, C], ...)."""
    b, c = normalized.shape[0], normalized.shape[1]
    spatial = normalized.numel() // max(1, b * c)
    dev = normalized.device
    gg, gb = _f32((b, c), dev), _f32((b, c), dev)
    sg = torch.empty(b, dtype=torch.float64, device=dev)
    sb = torch.empty(b, dtype=torch.float64, device=dev)
    _check(lib().dpg_grad_sample_group_norm(ctx.h, _p(normalized), _p(highway), b, c, spatial, _p(gg),
                                            _p(gb), _p(sg), _p(sb)), ctx.h)
    return gg, gb, sg, sb


def clip_factors(ctx: Context, sq: torch.Tensor, c: float):
    """optimizer.hpp:67-98. sq [nparams, b] float64 -> (norms f64 [b], scale f32 [b], num_clipped)."""
    nparams, b = sq.shape
    norms = torch.empty(b, dtype=torch.float64, device=sq.device)
    scale = torch.empty(b, dtype=torch.float32, device=sq.device)
    nclip = torch.zeros(1, dtype=torch.int64, device=sq.device)
    _check(lib().dpg_clip_factors(ctx.h, _p(sq.contiguous()), nparams, b, c, _p(norms), _p(scale),
                                  _p(nclip)), ctx.h)
    return norms, scale, nclip


def clipped_sum_linear(ctx, acts, highway, scale, bias=True, out_w=None, out_b=None, accumulate=False):
    b, d, r = acts.shape[0], acts.shape[-1], highway.shape[-1]
    mid = acts.numel() // max(1, b * d)
    sw = out_w if out_w is not None else _f32((r, d), acts.device)
    sb = out_b if out_b is not None else (_f32((r,), acts.device) if bias else None)
    _check(lib().dpg_clipped_sum_linear(ctx.h, _p(acts), _p(highway), _p(scale), b, mid, d, r,
                                        _p(sw), _p(sb), int(accumulate)), ctx.h)
    return sw, sb


def clipped_sum_conv2d(ctx, x, highway, scale, kh, kw, stride, pad, bias=True, out_w=None,
                       out_b=None, accumulate=False):
    b, ic, h, w = x.shape
    oc = highway.shape[1]
    sw = out_w if out_w is not None else _f32((oc, ic, kh, kw), x.device)
    sb = out_b if out_b is not None else (_f32((oc,), x.device) if bias else None)
    spec = _spec(ic, oc, kh, kw, stride, pad)
    _check(lib().dpg_clipped_sum_conv2d(ctx.h, _p(x), _p(highway), _p(scale), b, h, w,
                                        ctypes.byref(spec), _p(sw), _p(sb), int(accumulate)), ctx.h)
    return sw, sb


def clipped_sum_embedding(ctx, idx, highway, scale, vocab, out=None, accumulate=False):
    b, t = idx.shape
    dim = highway.shape[-1]
    s = out if out is not None else _f32((vocab, dim), idx.device)
    _check(lib().dpg_clipped_sum_embedding(ctx.h, _p(idx), _p(highway), _p(scale), b, t, vocab, dim,
                                           _p(s), int(accumulate)), ctx.h)
    return s


def clip_and_sum(ctx: Context, grads: Sequence[torch.Tensor], c: float, accumulate_into=None):
    """clip_and_sum (optimizer.hpp:62-116) over materialised per-sample gradients."""
    n = len(grads)
    b = grads[0].shape[0]
    gs = [g.contiguous() for g in grads]
    numel = (ctypes.c_int64 * n)(*[g.numel() // b for g in gs])
    summed = accumulate_into or [_f32(g.shape[1:], g.device) for g in gs]
    gp = (_P * n)(*[g.data_ptr() for g in gs])
    sp = (_P * n)(*[s.data_ptr() for s in summed])
    norms = torch.empty(b, dtype=torch.float64, device=gs[0].device)
    scale = torch.empty(b, dtype=torch.float32, device=gs[0].device)
    nclip = torch.zeros(1, dtype=torch.int64, device=gs[0].device)
    _check(lib().dpg_clip_and_sum_materialised(ctx.h, gp, numel, n, b, c, sp, _p(norms), _p(scale),
                                               _p(nclip), int(accumulate_into is not None)), ctx.h)
    return summed, norms, scale, nclip


def noise_update(ctx, params, summed, sigma, c, expected_batch, lr, seed, step, grad=None,
                 injected=None):
    """add_noise + finish_step (optimizer.hpp:120-133, 256-271), in place on params."""
    _check(lib().dpg_noise_update(ctx.h, _p(params), _p(summed), _p(grad), params.numel(), sigma, c,
                                  expected_batch, lr, seed, step, _p(injected)), ctx.h)


def gaussian(ctx, n, std, seed, step, device="cuda"):
    out = _f32((n,), device)
    _check(lib().dpg_gaussian(ctx.h, _p(out), n, std, seed, step), ctx.h)
    return out


# ---------------------------------------------------------------------------------------------
# Engine ABI
# ---------------------------------------------------------------------------------------------

class Model:
    """Device ModelGraph (layers.hpp:227-245) with parameters in (layer, slot) order."""

    def __init__(self, ctx: Context, layers: Sequence[LayerDesc], in_shape: Sequence[int],
                 max_batch: int):
        self.ctx = ctx
        self.layers = list(layers)
        self.in_shape = tuple(in_shape)
        self.max_batch = max_batch
        shp = (ctypes.c_int64 * len(in_shape))(*in_shape)
        h = _P()
        self._cl = c_layers(layers)
        _check(lib().dpg_model_create(ctx.h, self._cl, len(layers), shp, len(in_shape), max_batch,
                                      ctypes.byref(h)), ctx.h)
        self.h = h
        self._handle = _Handle(h, "dpg_model_destroy")
        ctx._handle.children.append(self._handle)
        self.L = int(lib().dpg_model_parameter_count(h))
        self.meta = params_meta(layers)

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            self._handle.destroy()
            self.h = None

    def parameter_count(self) -> int:
        return self.L

    def load_params(self, host):
        import numpy as np
        a = np.ascontiguousarray(host, dtype=np.float32)
        assert a.size == self.L
        _check(lib().dpg_model_load_params(self.h, a.ctypes.data_as(_P)), self.ctx.h)

    def store_params(self):
        import numpy as np
        a = np.empty(self.L, dtype=np.float32)
        _check(lib().dpg_model_store_params(self.h, a.ctypes.data_as(_P)), self.ctx.h)
        return a

    def params_ptr(self) -> int:
        return int(lib().dpg_model_params(self.h))

    def output_width(self) -> int:
        return int(lib().dpg_model_output_width(self.h))


class _CudaArray:
    """Minimal __cuda_array_interface__ holder so torch can wrap a libdpg device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _view(ptr: int, n: int, dtype=torch.float32) -> Optional[torch.Tensor]:
    """A copy of n elements at a libdpg device pointer (None for NULL)."""
    if not ptr:
        return None
    typestr = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device="cuda").clone()


class DpOptimizer:
    """DpOptimizer (optimizer.hpp:138-278) + GradSampleModule.forward_backward on the device."""

    def __init__(self, model: Model, noise_multiplier=1.0, max_grad_norm=1.0, learning_rate=0.1,
                 expected_batch_size=1.0, noise_seed=3, materialise_grad_sample=True,
                 clipped_sum_from_record=False):
        self.model = model
        self.ctx = model.ctx
        cfg = dpg_optimizer_config(noise_multiplier, max_grad_norm, learning_rate,
                                   expected_batch_size, noise_seed, int(materialise_grad_sample),
                                   int(clipped_sum_from_record))
        h = _P()
        _check(lib().dpg_optimizer_create(model.h, ctypes.byref(cfg), ctypes.byref(h)), self.ctx.h)
        self.h = h
        self._handle = _Handle(h, "dpg_optimizer_destroy")
        model._handle.children.append(self._handle)
        self._b = 0

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            self._handle.destroy()
            self.h = None

    def forward_backward(self, x: torch.Tensor, targets: torch.Tensor, loss: Optional[torch.Tensor] = None):
        """compute_grad_samples + set_grad_sample (grad_sample.hpp:328-343, optimizer.hpp:147-161)."""
        self._b = x.shape[0]
        self._x, self._y = x, targets  # keep alive until the fold
        _check(lib().dpg_forward_backward(self.h, _p(x), _p(targets), x.shape[0], _p(loss)), self.ctx.h)

    PEER_HANDLE_BYTES = 128  # DPG_PEER_HANDLE_BYTES

    def peer_handle(self) -> bytes:
        """This rank's handle for the peer-memory clipped-sum exchange (dpg_optimizer_peer_handle)."""
        buf = ctypes.create_string_buffer(self.PEER_HANDLE_BYTES)
        _check(lib().dpg_optimizer_peer_handle(self.h, ctypes.cast(buf, _P)), self.ctx.h)
        return buf.raw

    def set_peers(self, rank: int, handles) -> None:
        """Sum the clipped sums of all ranks over peer memory inside step() (instead of NCCL).
        `handles`: every rank's peer_handle() in rank order; a single handle turns it off."""
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib().dpg_optimizer_set_peers(self.h, rank, len(handles), ctypes.cast(buf, _P)), self.ctx.h)

    def virtual_step(self):
        _check(lib().dpg_virtual_step(self.h), self.ctx.h)

    def step(self):
        _check(lib().dpg_step(self.h), self.ctx.h)

    def step_empty_batch(self):
        _check(lib().dpg_step_empty_batch(self.h), self.ctx.h)

    def zero_grad(self):
        _check(lib().dpg_zero_grad(self.h), self.ctx.h)

    def set_noise_multiplier(self, sigma: float):
        _check(lib().dpg_set_noise_multiplier(self.h, sigma), self.ctx.h)

    def set_expected_batch_size(self, e: float):
        _check(lib().dpg_set_expected_batch_size(self.h, e), self.ctx.h)

    def set_injected_noise(self, noise: Optional[torch.Tensor]):
        self._noise = noise
        _check(lib().dpg_set_injected_noise(self.h, _p(noise)), self.ctx.h)

    def last_clip_summary(self):
        import numpy as np
        b = self._b
        norms = np.empty(b, dtype=np.float64)
        scales = np.empty(b, dtype=np.float64)
        n = ctypes.c_int64(0)
        _check(lib().dpg_last_clip_summary(self.h, norms.ctypes.data_as(_P), scales.ctypes.data_as(_P),
                                           ctypes.byref(n)), self.ctx.h)
        return norms, scales, int(n.value)

    def grad_sample(self) -> Optional[torch.Tensor]:
        return _view(lib().dpg_grad_sample(self.h), self._b * self.model.L)

    def grad_sample_export(self, param: int):
        """Parameter `param`'s per-sample gradients [b, ...param] on the host (dpg_grad_sample_export)."""
        import numpy as np
        numel = self.model.meta[param][4]
        out = np.empty(self._b * numel, dtype=np.float32)
        _check(lib().dpg_grad_sample_export(self.h, param, out.ctypes.data_as(ctypes.c_void_p), out.size), self.ctx.h)
        return out.reshape((self._b,) + tuple(self.model.meta[param][3]))

    def summed_grad(self) -> Optional[torch.Tensor]:
        return _view(lib().dpg_summed_grad(self.h), self.model.L)

    def grad(self) -> Optional[torch.Tensor]:
        return _view(lib().dpg_grad(self.h), self.model.L)

    def accumulated_samples(self) -> int:
        return int(lib().dpg_accumulated_samples(self.h))

    def train_step(self, x: torch.Tensor, targets: torch.Tensor, loss: Optional[torch.Tensor] = None,
                   use_graph: bool = True):
        self._b = x.shape[0]
        self._x, self._y = x, targets
        _check(lib().dpg_train_step(self.h, _p(x), _p(targets), x.shape[0], _p(loss), int(use_graph)),
               self.ctx.h)

    def train_step_host_async(self, x_host, targets_host, loss_host=None):
        """Pipelined host step (dpg_train_step_host_async): returns before the step finishes;
        the host buffers must stay alive until ctx.sync()."""
        def hp(a):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                return ctypes.c_void_p(a.data_ptr())
            return a.ctypes.data_as(_P)
        b = x_host.shape[0]
        self._b = b
        _check(lib().dpg_train_step_host_async(self.h, hp(x_host), hp(targets_host), b, hp(loss_host)),
               self.ctx.h)

    def train_step_host(self, x_host, targets_host, loss_host=None):
        """One step from HOST buffers (numpy or pinned torch CPU tensors): H2D, step, D2H."""
        def hp(a):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                return ctypes.c_void_p(a.data_ptr())
            return a.ctypes.data_as(_P)
        b = x_host.shape[0]
        self._b = b
        _check(lib().dpg_train_step_host(self.h, hp(x_host), hp(targets_host), b, hp(loss_host)),
               self.ctx.h)


def tg_gemm_selftest(ctx: Context, a: torch.Tensor, b: torch.Tensor, bn: int = 64, bk: int = 32) -> torch.Tensor:
    """D = A B^T through the TMA-fed tcgen05 GEMM core (dpg_tg_gemm_selftest; diagnostics)."""
    m, k = a.shape
    n = b.shape[1] if bk < 0 else b.shape[0]  # bk < 0: b is B transposed, [k][n]
    d = torch.empty(m, n, device=a.device, dtype=torch.float32)
    _check(lib().dpg_tg_gemm_selftest(ctx.h, _p(a), _p(b), _p(d), m, n, k, bn, bk), ctx.h)
    return d


def tg_gemm_selftest_split(ctx: Context, a: torch.Tensor, b: torch.Tensor, bn: int = 64, ck: int = 2) -> torch.Tensor:
    """D = A B^T with the K blocks split over a cluster of ck CTAs (dpg_tg_gemm_selftest_split)."""
    m, k = a.shape
    n = b.shape[0]
    d = torch.empty(m, n, device=a.device, dtype=torch.float32)
    _check(lib().dpg_tg_gemm_selftest_split(ctx.h, _p(a), _p(b), _p(d), m, n, k, bn, ck), ctx.h)
    return d


# ---------------------------------------------------------------------------------------------
# Privacy bookkeeping (host side): NoiseSchedule, RDP accountant (include/dpg.h)
# ---------------------------------------------------------------------------------------------

class _CSchedule(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("initial_sigma", ctypes.c_double), ("gamma", ctypes.c_double),
                ("factor", ctypes.c_double), ("period", ctypes.c_uint64), ("table", ctypes.c_void_p),
                ("table_len", ctypes.c_int64), ("current", ctypes.c_double)]


class NoiseSchedule:
    """NoiseSchedule (optimizer.hpp:280-351) over dpg_noise_schedule; factories validate like the
    reference's (ParameterError)."""
    CONSTANT, EXPONENTIAL, STEP, CUSTOM = range(4)

    def __init__(self, kind, sigma0=1.0, gamma=1.0, factor=1.0, period=1, table=None):
        self._table = None
        ptr, n = None, 0
        if table is not None:
            self._table = (ctypes.c_double * len(table))(*table)
            ptr, n = ctypes.cast(self._table, ctypes.c_void_p), len(table)
        self.s = _CSchedule()
        _check(lib().dpg_noise_schedule_init(ctypes.byref(self.s), kind, sigma0, gamma, factor, period, ptr, n))

    @classmethod
    def constant(cls, sigma):
        return cls(cls.CONSTANT, sigma)

    @classmethod
    def exponential(cls, sigma0, gamma):
        return cls(cls.EXPONENTIAL, sigma0, gamma=gamma)

    @classmethod
    def step(cls, sigma0, factor, period):
        return cls(cls.STEP, sigma0, factor=factor, period=period)

    @classmethod
    def custom(cls, table):
        return cls(cls.CUSTOM, table=list(table))

    @property
    def current(self) -> float:
        return self.s.current

    def sigma_at(self, epoch: int) -> float:
        return lib().dpg_noise_schedule_sigma_at(ctypes.byref(self.s), epoch)

    def schedule_noise(self, epoch: int, optimizer=None) -> float:
        """schedule_noise (optimizer.hpp:354-358); applies sigma to `optimizer` when given."""
        out = ctypes.c_double()
        _check(lib().dpg_schedule_noise(ctypes.byref(self.s), epoch, optimizer.h if optimizer else None,
                                        ctypes.byref(out)), optimizer.ctx.h if optimizer else None)
        return out.value


def rdp_subsampled_gaussian(q: float, sigma: float, alpha: int) -> float:
    out = ctypes.c_double()
    _check(lib().dpg_rdp_subsampled_gaussian(q, sigma, alpha, ctypes.byref(out)))
    return out.value


def get_noise_multiplier(target_eps: float, delta: float, q: float, steps: int, sigma_min: float = 0.01,
                         sigma_max: float = 100.0) -> float:
    out = ctypes.c_double()
    _check(lib().dpg_get_noise_multiplier(target_eps, delta, q, steps, sigma_min, sigma_max, ctypes.byref(out)))
    return out.value


class RdpAccountant:
    """RdpAccountant over dpg_accountant."""

    def __init__(self, orders: Optional[Sequence[int]] = None):
        h = _P()
        arr = (ctypes.c_int * len(orders))(*orders) if orders else None
        _check(lib().dpg_accountant_create(arr, len(orders) if orders else 0, ctypes.byref(h)))
        self._handle = _Handle(h, "dpg_accountant_destroy")
        self.h = h

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            self._handle.destroy()

    def step(self, sigma: float, q: float, steps: int = 1):
        _check(lib().dpg_accountant_step(self.h, sigma, q, steps))

    def rdp(self):
        n = lib().dpg_accountant_num_orders(self.h)
        orders = (ctypes.c_int * n)()
        curve = (ctypes.c_double * n)()
        _check(lib().dpg_accountant_rdp(self.h, orders, curve))
        return list(orders), list(curve)

    def epsilon(self, delta: float):
        eps, best = ctypes.c_double(), ctypes.c_int()
        _check(lib().dpg_accountant_epsilon(self.h, delta, ctypes.byref(eps), ctypes.byref(best)))
        return eps.value, best.value
