#!/usr/bin/env python
"""A small run of every kernel of the library, for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per invocation):

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

Covers: setup kernels, the batch kernel (HogBatch and Alg.1 negatives), the four step kernels
(rows, window, window warp-specialised, ring with TMEM originals) in Hogwild and deterministic
mode, the conflict-ticketed mode 2, Alg.1, the rowpath measurement mode, the overlapped batch
stream, the long-chunk kept-list ring (cfg4 shape), the on-device input generator, and the
1-rank data-parallel path with C13/C14/C15 sync.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1611_06172_b200 import binding as w2v  # noqa: E402


def run(ids, cfg, opts, dp=False, n_tokens=None):
    w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
    w2v.set_option("sentence_len", cfg.L)
    for k, v in opts.items():
        w2v.set_option(k, v)
    if dp:
        w2v.dist_init(0, 1, w2v.dist_unique_id())
    dev = torch.from_numpy(ids).cuda()
    w2v.train(dev, n_tokens or ids.size, 1)
    st = w2v.get_stats()
    M = np.empty((cfg.V, cfg.D), np.float32)
    w2v.get_embeddings(0, M)
    w2v.finalize()
    assert np.isfinite(M).all()
    return st


def main():
    torch.cuda.set_device(0)
    c1 = inputs.CONFIGS[1]
    ids1 = c1.corpus().tokens(0, 6000)
    c2 = inputs.CONFIGS[2]
    ids2 = c2.corpus().tokens(0, 6000)
    c4 = inputs.CONFIGS[4]
    ids4 = c4.corpus().tokens(0, 9000)   # L = 1000: long chunks (kept-list ring), window 8, K = 15
    gen = torch.empty(4096, dtype=torch.int32, device="cuda")
    c2.corpus().tokens_cuda(0, 4096, gen)
    inputs.CONFIGS[5].corpus().tokens_cuda(7_000_000_000, 4096, gen)
    cases = [
        (ids1, c1, {"mode": 0}), (ids1, c1, {"mode": 1, "debug_base": 0, "debug_len": 6000}),
        (ids2, c2, {"mode": 0, "kernel": 1}), (ids2, c2, {"mode": 0, "kernel": 2}), (ids2, c2, {"mode": 0, "kernel": 3}),
        (ids2, c2, {"mode": 1, "kernel": 3}), (ids2, c2, {"mode": 0, "algorithm": 1}),
        (ids2, c2, {"mode": 0, "rowpath_only": 1}), (ids1, c1, {"mode": 0, "overlap_batch": 1, "launch_words": 1000}),
        (ids2, c2, {"mode": 0, "kernel": 4}), (ids2, c2, {"mode": 1, "kernel": 4}),
        (ids2, c2, {"mode": 1, "kernel": 4, "ring_writeback": 1}), (ids2, c2, {"mode": 0, "kernel": 4, "rowpath_only": 1}),
        (ids1, c1, {"mode": 2}), (ids2, c2, {"mode": 2}),
        (ids4, c4, {"mode": 0}), (ids4, c4, {"mode": 1}),
    ]
    for ids, cfg, opts in cases:
        st = run(ids, cfg, opts)
        print("ok", cfg.idx, opts, st["targets"], flush=True)
    for opts in ({"sync_period_words": 1000}, {"sync_period_words": 1000, "sync_hot_rows": 100, "sync_cold_every": 2,
                                                "sync_overlap": 1},
                 {"sync_period_words": 1000, "sync_device": 1},
                 {"sync_period_words": 1000, "sync_hot_rows": 100, "sync_cold_every": 2, "sync_overlap": 1,
                  "sync_device": 1}):
        st = run(ids1, c1, dict(opts, mode=1), dp=True)
        print("ok dp", opts, st["syncs"], st["syncs_hot"], flush=True)
    print("sanitize_run done")


if __name__ == "__main__":
    main()
