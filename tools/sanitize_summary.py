"""profiles/r02_sanitize.md from the compute-sanitizer logs of tools/gpurun/r02_final.sh."""
import os
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
rows = []
for tool in ("memcheck", "racecheck", "synccheck"):
    for kind, name in (("", "default paths"), ("optin_", "opt-in paths (DPG_TG_CK=4 DPG_TG_CSUM=1 DPG_TG_RULE=1)")):
        path = os.path.join(d, f"sanitize_{kind}{tool}.log")
        if not os.path.exists(path):
            continue
        txt = open(path).read()
        summ = re.findall(r"=+ (?:ERROR|RACECHECK) SUMMARY: [^\n]*", txt)
        tests = re.findall(r"\d+ passed[^\n]*", txt)
        rows.append(f"| {tool} | {name} | {tests[-1] if tests else '?'} | `{summ[-1] if summ else 'no summary'}` |")
print("""# Sanitizers, round 2 (compute-sanitizer on a B200, `tools/gpurun/r02_final.sh`)

Default paths: `compute-sanitizer --tool T python -m pytest tests/test_gpu_tg.py
tests/test_gpu_step.py::test_step_matches_oracle tests/test_gpu_rules.py -k "not embedding_large"` —
the TMA-fed tcgen05 core on its own (TMA loads, mbarrier transaction counts, TMEM alloc / ld / st,
TS-mode MMA with paired B, MN-major B, the cluster split-K with its distributed-shared-memory
exchange), the whole engine step of every model (register-gather tcgen05 kernels, TMA-fed conv
forward / dgrad, thin conv forward, rules, clip factors, clipped sums, noise + update, PDL
launches) and the per-layer rule / clip / noise operators.
Opt-in paths: the step suite with the cluster split-K, the clipped sums and the conv2 rule on
the TMA core.

| tool | paths | tests | result |
|---|---|---|---|""")
print("\n".join(rows))
print("""
The cross-process peer-memory flags (`noise.cu`) are exercised by `tests/test_gpu_p2p.py`, which
spawns processes and is not run under the sanitizer.""")
