"""ReLU-kink screening for full-batch parity tests (test infrastructure).

A ReLU's derivative is discontinuous at 0, so a pre-activation whose fp64 value lies within the
rounding error of an fp32 contraction of zero has a mask that no fp32 implementation determines:
the reference's own fp32 path, the device's 3xTF32 path and a re-ordered sum can each land on
either side. One such element flips a whole row of the highway below it and moves that sample's
per-sample gradients by O(1e-2) of their maximum — a discontinuity of the function, not an error
of the contraction. (Synthetic CIFAR batch, seed 2, sample 126: a conv2 pre-activation of
9.0e-8 against terms of O(1); the device's no-split and split-K sums land on different sides.)

`kink_samples` finds those samples with an fp64 numpy forward (reference layers.hpp:389-467,
552-560): an element is a kink when |pre| <= rel * sum_k |x_k w_k| (+|bias|), the error bound of
an fp32-faithful sum of those terms. `redraw_kinks` replaces their inputs by fresh draws until
the batch is kink-free, so the full-size tests pin every launch at the sizes the bench runs
with inputs on which the reference function is well conditioned.
"""
import numpy as np

from paper_2109_12298_b200.configs import CONV2D, FLATTEN, LINEAR, RELU, params_meta

REL = 1e-6


def _conv(x, W, b, s, p):
    n, c, h, w = x.shape
    oc, ic, kh, kw = W.shape
    oh = (h + 2 * p - kh) // s + 1
    ow = (w + 2 * p - kw) // s + 1
    xp = np.zeros((n, c, h + 2 * p, w + 2 * p))
    xp[:, :, p:p + h, p:p + w] = x
    out = np.zeros((n, oc, oh, ow))
    for ki in range(kh):
        for kj in range(kw):
            patch = xp[:, :, ki:ki + s * oh:s, kj:kj + s * ow:s]
            out += np.einsum("nchw,oc->nohw", patch, W[:, :, ki, kj], optimize=True)
    return out if b is None else out + b[None, :, None, None]


def kink_samples(w, params, x, rel=REL):
    """Indices of samples with a ReLU pre-activation inside the fp32 rounding band of zero."""
    layers = w.layers
    if any(l.kind not in (CONV2D, LINEAR, RELU, FLATTEN) for l in layers):
        return np.zeros(0, dtype=np.int64)  # embedding / norm models here have no ReLU
    P = {}
    for (li, k, name, shape, numel, off) in params_meta(layers):
        P[(li, name)] = params[off:off + numel].astype(np.float64).reshape(shape)
    a = x.astype(np.float64)
    bad = np.zeros(x.shape[0], dtype=bool)
    pre = bound = None
    for li, l in enumerate(layers):
        if l.kind == CONV2D:
            W, bb = P[(li, "weight")], P.get((li, "bias"))
            pre = _conv(a, W, bb, l.stride, l.padding)
            bound = _conv(np.abs(a), np.abs(W), None if bb is None else np.abs(bb), l.stride, l.padding)
            a = pre
        elif l.kind == LINEAR:
            a2 = a.reshape(a.shape[0], -1)
            W, bb = P[(li, "weight")], P.get((li, "bias"))
            pre = a2 @ W.T + (0 if bb is None else bb)
            bound = np.abs(a2) @ np.abs(W).T + (0 if bb is None else np.abs(bb))
            a = pre
        elif l.kind == RELU:
            near = (np.abs(pre) <= rel * bound).reshape(pre.shape[0], -1).any(axis=1)
            bad |= near
            a = np.maximum(a, 0.0)
        elif l.kind == FLATTEN:
            a = a.reshape(a.shape[0], -1)
    return np.nonzero(bad)[0]


def redraw_kinks(w, params, x, seed=11, rel=REL, max_rounds=8):
    """x with kink samples replaced by fresh N(0,1) draws (kept dtype); returns (x, replaced)."""
    x = x.copy()
    rng = np.random.default_rng(seed)
    replaced = []
    for _ in range(max_rounds):
        ks = kink_samples(w, params, x, rel)
        if ks.size == 0:
            return x, replaced
        replaced.extend(int(k) for k in ks)
        x[ks] = rng.standard_normal((ks.size,) + x.shape[1:]).astype(x.dtype)
    raise AssertionError("could not draw a kink-free batch")
