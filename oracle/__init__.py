"""Python driver for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two implementations with identical signatures:
  * `restatement` — oracle/build/libdpg_oracle.so, the C restatement of the reference's DP-SGD
    step (oracle/dpg_oracle*.c), built by oracle/Makefile;
  * `reference`   — oracle/_ref/libdpgref.so, the real reference (/root/reference/proj/core)
    compiled from its own sources by the same Makefile, called through oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this package; the
product (paper_2109_12298_b200, libdpg.so) never does.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import numpy as np

from paper_2109_12298_b200.configs import LayerDesc, c_layers, param_count, params_meta

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "build", "libdpg_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libdpgref.so")
REFERENCE_FAST_SO = os.path.join(HERE, "_ref", "libdpgref_fast.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_U64 = ctypes.c_uint64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_P)


class _Impl:
    """One loaded library (restatement or reference), with numpy-facing wrappers."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.path = path
        self.prefix = prefix
        self.lib = ctypes.CDLL(path)
        err = getattr(self.lib, f"{prefix}_last_error")
        err.restype = ctypes.c_char_p
        self._err = err

    def fn(self, name: str, dtype=None):
        sfx = "" if dtype is None else ("_f32" if np.dtype(dtype) == np.float32 else "_f64")
        return getattr(self.lib, f"{self.prefix}_{name}{sfx}")

    def check(self, code: int):
        if code != 0:
            raise OracleError(code, self._err().decode())

    # ---- rng ----
    def gaussian(self, seed: int, n: int, std: float, dtype=np.float32) -> np.ndarray:
        out = np.empty(n, dtype=dtype)
        if self.prefix == "dpgref":
            self.check(self.fn("gaussian", dtype)(_U64(seed), _I64(n), _D(std), _ptr(out)))
        else:
            rng = self.rng(seed)
            self.fn("gaussian", dtype)(ctypes.byref(rng), _I64(n), _D(std), _ptr(out))
        return out

    def rng(self, seed: int):
        st = (ctypes.c_uint8 * 4096)()
        self.lib.dpgo_rng_seed(ctypes.byref(st), _U64(seed))
        return st

    def normals(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        if self.prefix == "dpgref":
            self.check(self.lib.dpgref_rng_normal(_U64(seed), _I64(n), _ptr(out)))
        else:
            st = self.rng(seed)
            f = self.lib.dpgo_rng_normal
            f.restype = ctypes.c_double
            for i in range(n):
                out[i] = f(ctypes.byref(st))
        return out

    def u64(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        if self.prefix == "dpgref":
            self.check(self.lib.dpgref_rng_u64(_U64(seed), _I64(n), _ptr(out)))
        else:
            st = self.rng(seed)
            f = self.lib.dpgo_rng_next_u64
            f.restype = ctypes.c_uint64
            for i in range(n):
                out[i] = f(ctypes.byref(st))
        return out

    def below(self, seed: int, n: int, bound: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        if self.prefix == "dpgref":
            self.check(self.lib.dpgref_rng_below(_U64(seed), _I64(n), _U64(bound), _ptr(out)))
        else:
            st = self.rng(seed)
            f = self.lib.dpgo_rng_below
            f.restype = ctypes.c_uint64
            for i in range(n):
                out[i] = f(ctypes.byref(st), _U64(bound))
        return out

    def build_params(self, layers: Sequence[LayerDesc], seed: int, dtype=np.float32) -> np.ndarray:
        out = np.empty(param_count(layers), dtype=dtype)
        cl = c_layers(layers)
        if self.prefix == "dpgref":
            self.check(self.fn("build_params", dtype)(cl, len(layers), _U64(seed), _ptr(out)))
        else:
            st = self.rng(seed)
            self.check(self.fn("build_params", dtype)(cl, len(layers), ctypes.byref(st), _ptr(out)))
        return out

    # ---- per-sample rules ----
    def rule_linear(self, acts: np.ndarray, hw: np.ndarray, bias: bool = True):
        b, mid, d = acts.shape
        r = hw.shape[-1]
        gw = np.empty((b, r, d), dtype=acts.dtype)
        gb = np.empty((b, r), dtype=acts.dtype) if bias else None
        self.check(self.fn("rule_linear", acts.dtype)(_ptr(acts), _ptr(hw), _I64(b), _I64(mid),
                                                      _I64(d), _I64(r), _ptr(gw), _ptr(gb)))
        return gw, gb

    def rule_conv2d(self, x: np.ndarray, hw: np.ndarray, kh: int, kw: int, stride: int, pad: int):
        b, ic, h, w = x.shape
        oc = hw.shape[1]
        gw = np.empty((b, oc, ic, kh, kw), dtype=x.dtype)
        gb = np.empty((b, oc), dtype=x.dtype)
        self.check(self.fn("rule_conv2d", x.dtype)(
            _ptr(x), _ptr(hw), _I64(b), _I64(ic), _I64(h), _I64(w), _I64(oc), _I64(kh), _I64(kw),
            _I64(stride), _I64(pad), _ptr(gw), _ptr(gb)))
        return gw, gb

    def rule_norm(self, normalized: np.ndarray, hw: np.ndarray, group: bool):
        """per_sample_rule_layer_norm ([b, q, c], group=False) / _group_norm ([b, c, q]); reference only."""
        assert self.prefix == "dpgref"
        b = normalized.shape[0]
        c = normalized.shape[1] if group else normalized.shape[-1]
        q = normalized.size // (b * c)
        gg = np.empty((b, c), dtype=normalized.dtype)
        gb = np.empty((b, c), dtype=normalized.dtype)
        self.check(self.fn("rule_norm", normalized.dtype)(
            ctypes.c_int(int(group)), _ptr(np.ascontiguousarray(normalized)), _ptr(np.ascontiguousarray(hw)),
            _I64(b), _I64(c), _I64(q), _ptr(gg), _ptr(gb)))
        return gg, gb

    def rule_embedding(self, idx: np.ndarray, hw: np.ndarray, vocab: int):
        b, t = idx.shape
        dim = hw.shape[-1]
        out = np.empty((b, vocab, dim), dtype=hw.dtype)
        self.check(self.fn("rule_embedding", hw.dtype)(_ptr(idx.astype(hw.dtype)), _ptr(hw), _I64(b),
                                                       _I64(t), _I64(vocab), _I64(dim), _ptr(out)))
        return out

    def clip_and_sum(self, grads: Sequence[np.ndarray], c: float):
        dtype = grads[0].dtype
        b = grads[0].shape[0]
        n = len(grads)
        gs = [np.ascontiguousarray(g.reshape(b, -1)) for g in grads]
        numel = np.array([g.shape[1] for g in gs], dtype=np.int64)
        summed = [np.empty(g.shape[1], dtype=dtype) for g in gs]
        gptr = (_P * n)(*[g.ctypes.data for g in gs])
        sptr = (_P * n)(*[s.ctypes.data for s in summed])
        norms = np.empty(b, dtype=np.float64)
        scales = np.empty(b, dtype=np.float64)
        nclip = ctypes.c_int64(0)
        if self.prefix == "dpgref":
            self.check(self.fn("clip_and_sum", dtype)(gptr, _ptr(numel), n, _I64(b), _D(c), sptr,
                                                      _ptr(norms), _ptr(scales), ctypes.byref(nclip)))
        else:
            bp, bs = ctypes.c_int64(-1), ctypes.c_int64(-1)
            self.check(self.fn("clip_and_sum", dtype)(gptr, _ptr(numel), n, _I64(b), _D(c), sptr,
                                                      _ptr(norms), _ptr(scales), ctypes.byref(nclip),
                                                      ctypes.byref(bp), ctypes.byref(bs)))
        return summed, norms, scales, int(nclip.value)

    def add_noise(self, summed: np.ndarray, sigma: float, c: float, seed: int) -> np.ndarray:
        out = np.empty_like(summed)
        if self.prefix == "dpgref":
            self.check(self.fn("add_noise", summed.dtype)(_ptr(summed), _I64(summed.size), _D(sigma),
                                                          _D(c), _U64(seed), _ptr(out)))
        else:
            st = self.rng(seed)
            self.check(self.fn("add_noise", summed.dtype)(_ptr(summed), _I64(summed.size), _D(sigma),
                                                          _D(c), ctypes.byref(st), _ptr(out)))
        return out

    # ---- the whole logical step ----
    def dpsgd_step(self, layers: Sequence[LayerDesc], in_shape: Sequence[int], params: np.ndarray,
                   x: np.ndarray, targets: np.ndarray, sigma: float, c: float, lr: float,
                   expected_batch: float, noise_seed: int = 3, injected_noise=None,
                   shards: Optional[Sequence[int]] = None, want_record: bool = True) -> Dict:
        dtype = params.dtype
        b = x.shape[0]
        L = param_count(layers)
        k = _out_classes(layers)
        p = params.copy()
        res = {
            "record": np.empty(b * L, dtype=dtype) if want_record else None,
            "summed": np.empty(L, dtype=dtype),
            "grad": np.empty(L, dtype=dtype),
            "norms": np.empty(b, dtype=np.float64),
            "scales": np.empty(b, dtype=np.float64),
            "loss": np.empty(b, dtype=dtype),
            "logits": np.empty((b, k), dtype=dtype),
        }
        nclip = ctypes.c_int64(0)
        shp = np.array(in_shape, dtype=np.int64)
        sh = None if shards is None else np.array(shards, dtype=np.int64)
        inj = None if injected_noise is None else np.ascontiguousarray(injected_noise, dtype=dtype)
        xx = np.ascontiguousarray(x, dtype=dtype)
        yy = np.ascontiguousarray(targets, dtype=dtype)
        self.check(self.fn("dpsgd_step", dtype)(
            c_layers(layers), len(layers), _ptr(shp), len(in_shape), _I64(b), _ptr(sh),
            0 if sh is None else len(sh), _ptr(p), _ptr(xx), _ptr(yy), _D(sigma), _D(c), _D(lr),
            _D(expected_batch), _U64(noise_seed), _ptr(inj), _ptr(res["record"]), _ptr(res["summed"]),
            _ptr(res["grad"]), _ptr(res["norms"]), _ptr(res["scales"]), ctypes.byref(nclip),
            _ptr(res["loss"]), _ptr(res["logits"])))
        res["params"] = p
        res["num_clipped"] = int(nclip.value)
        return res

    def dpsgd_step_threads(self, layers, in_shape, params, x, targets, sigma, c, lr, expected_batch,
                           noise_seed: int, nthreads: int) -> np.ndarray:
        """The sample-sharded host thread pool over the reference (reference only)."""
        assert self.prefix == "dpgref"
        dtype = params.dtype
        p = params.copy()
        shp = np.array(in_shape, dtype=np.int64)
        self.check(self.fn("dpsgd_step_threads", dtype)(
            c_layers(layers), len(layers), _ptr(shp), len(in_shape), _I64(x.shape[0]), nthreads,
            _ptr(p), _ptr(np.ascontiguousarray(x, dtype=dtype)),
            _ptr(np.ascontiguousarray(targets, dtype=dtype)), _D(sigma), _D(c), _D(lr),
            _D(expected_batch), _U64(noise_seed)))
        return p

    def microbatch_oracle(self, layers, in_shape, params, x, targets) -> np.ndarray:
        assert self.prefix == "dpgref"
        dtype = params.dtype
        b = x.shape[0]
        out = np.empty(b * param_count(layers), dtype=dtype)
        shp = np.array(in_shape, dtype=np.int64)
        self.check(self.fn("microbatch_oracle", dtype)(
            c_layers(layers), len(layers), _ptr(shp), len(in_shape), _I64(b), _ptr(params),
            _ptr(np.ascontiguousarray(x, dtype=dtype)), _ptr(np.ascontiguousarray(targets, dtype=dtype)),
            _ptr(out)))
        return out


def _out_classes(layers: Sequence[LayerDesc]) -> int:
    for l in reversed(layers):
        if l.kind == 0:
            return l.out_features
    raise ValueError("model must end in a linear layer for softmax cross-entropy")


_cache: Dict[str, _Impl] = {}


def restatement() -> _Impl:
    if "r" not in _cache:
        _cache["r"] = _Impl(RESTATEMENT_SO, "dpgo")
    return _cache["r"]


def reference(fast: bool = False) -> _Impl:
    key = "f" if fast else "ref"
    if key not in _cache:
        _cache[key] = _Impl(REFERENCE_FAST_SO if fast else REFERENCE_SO, "dpgref")
    return _cache[key]


def reference_available(fast: bool = False) -> bool:
    return os.path.exists(REFERENCE_FAST_SO if fast else REFERENCE_SO)


def record_split(record: np.ndarray, layers: Sequence[LayerDesc], b: int):
    """Split a flat record (per (l,k): [b, numel]) into per-parameter [b, *shape] arrays."""
    out = []
    for (li, k, name, shape, n, off) in params_meta(layers):
        out.append(record[b * off: b * (off + n)].reshape((b,) + tuple(shape)))
    return out


def synth_inputs(workload, seed_model: int = 1, seed_data: int = 2, dtype=np.float32, b=None,
                 impl: Optional[_Impl] = None):
    """Synthetic parameters / inputs / targets exactly as SURVEY.md §8(d) pins them:
    params = build_model(RngStream::standard(seed_model)); activations = gaussian(1.0) from
    RngStream::standard(seed_data); class targets = below(k) and token ids = below(V) from
    RngStream::standard(seed_data + 1)."""
    impl = impl or restatement()
    b = b or workload.batch
    params = impl.build_params(workload.layers, seed_model, dtype)
    per = int(np.prod(workload.in_shape))
    if workload.tokens:
        ids = impl.below(seed_data, b * per, workload.tokens).astype(dtype)
        x = ids.reshape((b,) + tuple(workload.in_shape))
    else:
        x = impl.gaussian(seed_data, b * per, 1.0, dtype).reshape((b,) + tuple(workload.in_shape))
    y = impl.below(seed_data + 1, b, workload.classes).astype(dtype)
    return params, x, y
