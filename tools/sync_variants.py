"""Every a9 variant at full cfg3 size on a 1-rank NCCL communicator (the only one a one-GPU box can
build): no communicator; C13 via ncclAllReduce; C13 via the C17 device kernel; C15 (in flight)
via NCCL; C15 via the C17 kernel on the comm stream. At W = 1 every average is the identity, so
this measures what each variant costs on the GPU that trains (HBM traffic and launch overhead of
763 averages of the 2.56 GB model per epoch), checks that each runs at full size, and that all
five leave the same model. Prints one JSON line.

    python tools/sync_variants.py [--steps 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

VARIANTS = {  # name: (communicator, sync_device, sync_overlap)
    "no_comm": (False, 0, 0),
    "c13_nccl": (True, 0, 0),
    "c13_c17": (True, 1, 0),
    "c15_nccl": (True, 0, 1),
    "c15_c17": (True, 1, 1),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--config", type=int, default=3)
    a = ap.parse_args()
    from paper_1611_06172_b200 import binding as w2v
    cfg = inputs.CONFIGS[a.config]
    dev = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    cfg.corpus().tokens_cuda(0, cfg.n, dev)
    torch.cuda.synchronize()
    out, ref = {}, None
    for name, (comm, sd, ovl) in VARIANTS.items():
        w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
        w2v.set_option("sentence_len", cfg.L)
        w2v.set_option("mode", 0)
        w2v.set_option("sync_overlap", ovl)
        w2v.set_option("sync_device", sd)
        w2v.dist_init(0, 1, w2v.dist_unique_id() if comm else None)
        s = torch.cuda.current_stream()
        w2v.set_stream(s.cuda_stream)
        w2v.train(dev, cfg.n, 1)   # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        ms_sync = 0.0
        for _ in range(a.steps):
            w2v.train(dev, cfg.n, 1)
            ms_sync += w2v.get_stats()["ms_sync"]
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        st = w2v.get_stats()
        M = np.empty((cfg.V, cfg.D), np.float32)
        w2v.get_embeddings(0, M)
        finite = bool(np.isfinite(M).all())
        out[name] = {"words_per_s": cfg.n / (ms / 1e3), "ms_per_step": ms, "ms_sync_per_step": ms_sync / a.steps,
                     "syncs": st["syncs"], "sync_path": st["sync_path"], "launches": st["launches"],
                     "finite": finite}
        w2v.finalize()
    print(json.dumps({"tool": "sync_variants", "world": 1, "config": a.config, "n_tokens": cfg.n,
                      "mode": "hogwild", "variants": out}))


if __name__ == "__main__":
    main()
