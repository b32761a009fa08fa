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
    "nogather": ["-DW2V_ABL_NOGATHER"],
    "g_ldgsts": ["-DW2V_GATHER_LDGSTS"],
    "s_red": ["-DW2V_SCATTER_RED"],
    "s_red_fence": ["-DW2V_SCATTER_RED", "-DW2V_RED_FENCE"],
    "ldgsts_red_fence": ["-DW2V_GATHER_LDGSTS", "-DW2V_SCATTER_RED", "-DW2V_RED_FENCE"],
    "noscatter": ["-DW2V_ABL_NOSCATTER"],
    "phase": ["-DW2V_PHASE_TIMING"],
    "fulltile": ["-DW2V_DOT_FULL_TILE"],
    "minb9": ["-DW2V_MINB=9"],
    "a1mb20": ["-DW2V_A1_MINB=20"],
    "a1mb24": ["-DW2V_A1_MINB=24"],
    "minb8": ["-DW2V_MINB=8"],
    "nohot16": ["-DW2V_ABL_NOHOT=16"],
    "nohot256": ["-DW2V_ABL_NOHOT=256"],
    "nohot4096": ["-DW2V_ABL_NOHOT=4096"],
}


def build(names):
    from paper_1611_06172_b200 import _build
    os.makedirs(OUT, exist_ok=True)
    for n in names:
        print(n, _build.build(out=os.path.join(OUT, f"libw2v_{n}.so"), extra=VARIANTS[n]), flush=True)


def one(so, tokens, opts, reps, vmod=0, config=3):
    import numpy as np  # noqa: F401
    import torch
    os.environ["W2V_LIBRARY"] = so
    import inputs
    from paper_1611_06172_b200 import binding as w2v
    cfg = inputs.CONFIGS[config]
    host = torch.empty(tokens, dtype=torch.int32, pin_memory=True)
    cfg.corpus().tokens(0, tokens, out=host.numpy())
    V = cfg.V
    if vmod:  # (experiment) fold the vocabulary so the whole model fits in L2
        host.remainder_(vmod)
        V = vmod
    dev = host.cuda()
    w2v.init(V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
    w2v.set_option("sentence_len", cfg.L)
    w2v.set_option("check_finite", 0)  # ablation variants may compute on junk on purpose
    for k, v in opts.items():
        if k == "dp1":  # (experiment) the data-parallel path on a 1-rank NCCL communicator
            if v:
                w2v.dist_init(0, 1, w2v.dist_unique_id())
            continue
        w2v.set_option(k, v)
    best = None
    for _ in range(reps):
        w2v.train(dev, tokens, 1)
        st = w2v.get_stats()
        if best is None or st["ms_step"] < best["ms_step"]:
            best = st
    w2v.finalize()
    return {"words_per_s": tokens / (best["ms_step"] / 1e3), "ms_step": best["ms_step"], "ms_sync": best["ms_sync"],
            "ms_total": best["ms_total"], "syncs": best["syncs"], "syncs_hot": best["syncs_hot"],
            "units_per_sm": best["units_per_sm"],

            "row_GBps": best["bytes_row"] / (best["ms_step"] / 1e3) / 1e9, "ms_batch": best["ms_batch"],
            "l2_window_MB": best["l2_window_bytes"] / 2**20, "l2_carve_MB": best["l2_carve_bytes"] / 2**20}


def run(names, tokens, sweeps, reps, vmod=0, config=3):
    for n in names:
        so = os.path.join(OUT, f"libw2v_{n}.so") if n != "main" else \
            os.path.join(ROOT, "paper_1611_06172_b200", "libw2v.so")
        for opts in sweeps:
            code = (f"import sys, json; sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.dirname(__file__)!r});"
                    f"import ablate; print(json.dumps(ablate.one({so!r}, {tokens}, {opts!r}, {reps}, {vmod}, {config})))")
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
            print(json.dumps({"variant": n, "opts": opts, "result": line}), flush=True)
            for ln in r.stderr.splitlines():
                if ln.startswith("[phase]"):
                    print("   ", ln, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["build", "run"])
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--tokens", type=int, default=1 << 27)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--occ", default="0", help="comma list of ctas_per_sm values (0 = max)")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--vmod", type=int, default=0, help="experiment: ids %% vmod, V = vmod")
    ap.add_argument("--opts", default="", help="extra option sets: 'k=v,k=v;k=v' (each ';' part is one run)")
    a = ap.parse_args()
    names = a.variants.split(",")
    if a.what == "build":
        build(names)
    else:
        sweeps = [{"ctas_per_sm": int(x)} if int(x) else {} for x in a.occ.split(",")]
        if a.opts:
            sweeps = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in part.split(",")) for part in a.opts.split(";")]
        run(names, a.tokens, sweeps, a.reps, a.vmod, a.config)
