"""Per-stage parity diagnosis of one device step against the fp64 oracle (GPU box).

  python tools/diag_parity.py cifar_b512 512 [c]

Prints, per parameter, the max-scaled error of the record, the clipped sum and the loss / norm
errors, so a parity failure at a full-size config can be localised to a layer.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from conftest import maxscaled_err  # noqa: E402
from paper_2109_12298_b200 import dpg  # noqa: E402
from paper_2109_12298_b200.configs import WORKLOADS, params_meta  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cifar_b512"
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    c = float(sys.argv[3]) if len(sys.argv) > 3 else 1.48
    w = WORKLOADS[name]
    params, x, y = oracle.synth_inputs(w, b=b)
    if os.environ.get("DIAG_REDRAW"):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from kinks import redraw_kinks
        x, _ = redraw_kinks(w, params, x)
    ctx = dpg.Context(0)
    m = dpg.Model(ctx, w.layers, w.in_shape, max_batch=b)
    m.load_params(params)
    o = dpg.DpOptimizer(m, noise_multiplier=0.0, max_grad_norm=c, learning_rate=0.1,
                        expected_batch_size=float(b), noise_seed=3)
    loss = torch.zeros(b, device="cuda")
    o.forward_backward(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), loss)
    rec = o.grad_sample().cpu().numpy()
    o.step()
    norms, scales, nclip = o.last_clip_summary()
    summed = o.summed_grad().cpu().numpy()
    ctx.sync()
    if os.environ.get("DIAG_ISOLATE"):
        # clipped sums recomputed in fp64 from the device's own record and scales: isolates the
        # clipped-sum kernels from upstream (forward / dgrad / rule) error
        sc = np.asarray(scales, dtype=np.float32).astype(np.float64)
        for (li, k, pname, shape, numel, off) in params_meta(w.layers):
            g = rec[b * off: b * (off + numel)].reshape(b, numel).astype(np.float64)
            ref = sc @ g
            print(f"  isolated csum layer {li} {pname}: {maxscaled_err(summed[off:off + numel], ref):.3e}")
        if os.environ.get("DIAG_ISOLATE") == "only":
            return
    r64 = oracle.restatement().dpsgd_step(w.layers, w.in_shape, params.astype(np.float64), x.astype(np.float64),
                                          y.astype(np.float64), 0.0, c, 0.1, float(b), noise_seed=3)
    r32 = oracle.restatement().dpsgd_step(w.layers, w.in_shape, params, x, y, 0.0, c, 0.1, float(b), noise_seed=3)
    print(f"{name} b={b} C={c} ksplit={os.environ.get('DPG_KSPLIT', 'default')}")
    print(f"  loss  maxrel {np.abs(loss.cpu().numpy() - r64['loss']).max() / np.abs(r64['loss']).max():.3e}")
    nr = np.abs(np.asarray(norms) - r64["norms"]) / r64["norms"]
    print(f"  norms maxrel {nr.max():.3e} at sample {int(nr.argmax())} (gpu {norms[int(nr.argmax())]:.8g} "
          f"ref {r64['norms'][int(nr.argmax())]:.8g}); clipped {nclip} vs {r64['num_clipped']}")
    for (li, k, pname, shape, numel, off) in params_meta(w.layers):
        sl = slice(b * off, b * (off + numel))
        g = rec[sl].reshape(b, numel)
        r = r64["record"][sl].reshape(b, numel)
        e = maxscaled_err(g, r)
        per = np.abs(g - r).max(axis=1) / max(np.abs(r).max(), 1e-300)
        bad = np.nonzero(per > 1e-5)[0]
        es = maxscaled_err(summed[off:off + numel], r64["summed"][off:off + numel])
        r3 = r32["record"][sl].reshape(b, numel)
        per32 = np.abs(r3 - r).max(axis=1) / max(np.abs(r).max(), 1e-300)
        bad32 = np.nonzero(per32 > 1e-5)[0]
        print(f"  layer {li} {pname:6s} record {e:.3e} (bad samples {len(bad)}: {bad[:8].tolist()})  summed {es:.3e}"
              f" | fp32 oracle record {maxscaled_err(r3, r):.3e} (bad {len(bad32)}: {bad32[:8].tolist()})"
              f" summed {maxscaled_err(r32['summed'][off:off + numel], r64['summed'][off:off + numel]):.3e}")


if __name__ == "__main__":
    main()
