"""Hogwild at FULL size against the sequential algorithm (opt-in: W2V_FULLSIZE=1; select configs
with W2V_FULLSIZE_CONFIGS=3,4). cfg4 (D = 128, K = 15, window 8) runs the TMA gather4 path.

cfg3 (V = 1M, D = 300, window 5, K = 5, t = 1e-4, 800M planted-Zipf tokens), one epoch:
  * Hogwild: the bench's launch configuration (all SMs, the default rows kernel; and the ring);
  * sequential: the library's deterministic mode 1 (one work unit, targets in corpus order, R17),
    which the parity tests hold to the fp64 oracle (<= 1e-5 relative L2 up to the cfg3 shape at
    2^20 tokens, within 1.25x the fp32 oracle's error) — the sequential CPU oracle itself would
    need ~3 h for 800M tokens, the GPU's mode 1 ~30 min.
north_star's Hogwild bar (final-10% training loss and held-out loss within 1% of the sequential
run, Hogwild's stale reads may slow convergence) at 40x the size of
test_gpu_parity.py::test_cfg3_hogwild_prefix_loss_gate. Held-out loss: the frozen models on 200K
tokens beyond the corpus, evaluated by the oracle (identical batches for every model).

Not part of the default `-m gpu` run (it takes ~35 GPU-minutes): W2V_FULLSIZE=1 enables it.
"""
import os

import numpy as np
import pytest
import torch

import inputs
from test_gpu_parity import heldout_loss, w2v  # noqa: F401

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("W2V_FULLSIZE") != "1", reason="opt-in: W2V_FULLSIZE=1 (~35 min)")]


def _train(w2v, dev, cfg, mode, kernel, tail_from):  # noqa: F811
    w2v.finalize()
    w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
    w2v.set_option("sentence_len", cfg.L)
    w2v.set_option("mode", mode)
    w2v.set_option("kernel", kernel)
    w2v.set_option("loss_tail_from", tail_from)
    w2v.train(dev, cfg.n, 1)
    st = w2v.get_stats()
    M_in = np.empty((cfg.V, cfg.D), np.float32)
    M_out = np.empty((cfg.V, cfg.D), np.float32)
    w2v.get_embeddings(0, M_in)
    w2v.get_embeddings(1, M_out)
    return st, M_in, M_out


@pytest.mark.parametrize("config", [3, 4])
def test_cfg3_fullsize_hogwild_vs_sequential(w2v, config):  # noqa: F811
    """cfg3 (the headline) and cfg4 (D = 128, K = 15, window 8: the TMA gather4 path)."""
    if os.environ.get("W2V_FULLSIZE_CONFIGS") and str(config) not in os.environ["W2V_FULLSIZE_CONFIGS"].split(","):
        pytest.skip("not selected in W2V_FULLSIZE_CONFIGS")
    cfg = inputs.CONFIGS[config]
    dev = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    cfg.corpus().tokens_cuda(0, cfg.n, dev)
    tail_from = (cfg.n * 9 // 10) // cfg.L * cfg.L
    res = {}
    for name, mode, kernel in (("sequential (mode 1)", 1, 1), ("hogwild rows", 0, 1), ("hogwild ring", 0, 4)):
        st, M_in, M_out = _train(w2v, dev, cfg, mode, kernel, tail_from)
        tail = st["loss_tail_sum"] / st["loss_tail_pairs"]
        whole = st["loss_sum"] / st["loss_pairs"]
        held = heldout_loss(M_in, M_out, cfg, cfg.n, 200_000)
        res[name] = (whole, tail, held, st["row_touches"], st["ms_total"])
        print(f"cfg{config} full {name}: loss/pair whole {whole:.6f}, final 10% {tail:.6f}, held-out {held:.6f}; "
              f"row_touches {st['row_touches']}, {st['ms_total'] / 1e3:.1f} s")
    seq = res["sequential (mode 1)"]
    for name in ("hogwild rows", "hogwild ring"):
        assert res[name][3] == seq[3]               # the same batch stream: identical row touches
    rows = res["hogwild rows"]                      # the default kernel: the north_star gate
    assert abs(rows[1] / seq[1] - 1) < 0.01 and abs(rows[2] / seq[2] - 1) < 0.01, (rows, seq)
    ring = res["hogwild ring"]
    ring_ok = abs(ring[1] / seq[1] - 1) < 0.01 and abs(ring[2] / seq[2] - 1) < 0.01
    if config == 4 and not ring_ok:
        # known limitation of the (opt-in) ring kernel, r02: at cfg4 (window 8, K = 15, L = 1000)
        # a slot holds a Zipf-hot context row for 2w+1 = 17 targets while ~1,600 other units
        # update it; the deltas written back from those stale copies overshoot early in the run
        # (whole-run loss 1.67 vs 0.23) and the final-10% / held-out loss end 2.6% / 2.1% high
        pytest.xfail(f"ring kernel at cfg4: final 10% {ring[1]:.6f} vs {seq[1]:.6f}, held-out {ring[2]:.6f} vs "
                     f"{seq[2]:.6f} (DESIGN.md §8, NEXT-1 limitation)")
    assert ring_ok, (ring, seq)
