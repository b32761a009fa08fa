#!/usr/bin/env python
"""Timing experiments on the fused step (not a bench: no parity, variants are broken on purpose).

Builds libw2v variants with ablation macros (hogbatch.cu: W2V_ABL_NOCOMPUTE,
W2V_ABL_NOWAIT, W2V_MINB=...) and times `w2v_train` on a cfg3 prefix for each, plus occupancy
sweeps through the `ctas_per_sm` option. Prints one JSON line per (variant, option set).

  python tools/ablate.py build            # here (nvcc cross-compile)
  python tools/ablate.py run [--tokens N] # on the GPU box
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "paper_1611_06172_b200", "build", "abl")

VARIANTS = {
    "base": [],
    "nocompute": ["-DW2V_ABL_NOCOMPUTE"],
    "nowait": ["-DW2V_ABL_NOWAIT"],
    "nocompute_nowait": ["-DW2V_ABL_NOCOMPUTE", "-DW2V_ABL_NOWAIT"],
}


def build(names):
    from paper_1611_06172_b200 import _build
    os.makedirs(OUT, exist_ok=True)
    for n in names:
        print(n, _build.build(out=os.path.join(OUT, f"libw2v_{n}.so"), extra=VARIANTS[n]), flush=True)


def one(so, tokens, opts, reps):
    import numpy as np  # noqa: F401
    import torch
    os.environ["W2V_LIBRARY"] = so
    import inputs
    from paper_1611_06172_b200 import binding as w2v
    cfg = inputs.CONFIGS[3]
    host = torch.empty(tokens, dtype=torch.int32, pin_memory=True)
    cfg.corpus().tokens(0, tokens, out=host.numpy())
    dev = host.cuda()
    w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
    w2v.set_option("sentence_len", cfg.L)
    for k, v in opts.items():
        w2v.set_option(k, v)
    best = None
    for _ in range(reps):
        w2v.train(dev, tokens, 1)
        st = w2v.get_stats()
        if best is None or st["ms_step"] < best["ms_step"]:
            best = st
    w2v.finalize()
    return {"words_per_s": tokens / (best["ms_step"] / 1e3), "ms_step": best["ms_step"],
            "row_GBps": best["bytes_row"] / (best["ms_step"] / 1e3) / 1e9, "ms_batch": best["ms_batch"]}


def run(names, tokens, sweeps, reps):
    for n in names:
        so = os.path.join(OUT, f"libw2v_{n}.so")
        for opts in sweeps:
            code = (f"import sys, json; sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.dirname(__file__)!r});"
                    f"import ablate; print(json.dumps(ablate.one({so!r}, {tokens}, {opts!r}, {reps})))")
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
            print(json.dumps({"variant": n, "opts": opts, "result": line}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["build", "run"])
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--tokens", type=int, default=1 << 27)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--occ", default="0", help="comma list of ctas_per_sm values (0 = max)")
    a = ap.parse_args()
    names = a.variants.split(",")
    if a.what == "build":
        build(names)
    else:
        sweeps = [{"ctas_per_sm": int(x)} if int(x) else {} for x in a.occ.split(",")]
        run(names, a.tokens, sweeps, a.reps)
