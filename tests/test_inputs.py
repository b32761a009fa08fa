"""Pins of the seeded input generator (inputs/): the recipe DESIGN.md §5 states."""
import numpy as np
import pytest
from scipy import stats

import inputs


def test_iid_zipf_marginal():
    cor = inputs.Corpus("iid", 200, 1.07, 3)
    ids = cor.tokens(0, 400_000)
    assert ids.min() >= 0 and ids.max() < 200
    zq = cor.zipf_weights().astype(np.float64)
    ref = np.power(np.arange(1, 201, dtype=np.float64), -1.07)
    assert np.allclose(zq / zq.sum(), ref / ref.sum(), rtol=1e-9)
    hist = np.bincount(ids, minlength=200)
    assert stats.chisquare(hist, zq / zq.sum() * ids.size).pvalue > 1e-4


def test_slices_are_position_keyed():
    cor = inputs.Corpus("iid", 1000, 1.0, 11)
    full = cor.tokens(0, 50_000, threads=1)
    assert np.array_equal(cor.tokens(12_345, 1_000), full[12_345:13_345])
    assert np.array_equal(cor.tokens(0, 50_000, threads=7), full)
    pl = inputs.Corpus("planted", 1000, 1.07, 11, 37, 20)
    fullp = pl.tokens(0, 40_000, threads=1)
    assert np.array_equal(pl.tokens(20_013, 977), fullp[20_013:20_990])
    assert np.array_equal(pl.tokens(0, 40_000, threads=5), fullp)


def test_planted_sentences_and_marginal():
    V, C, Lg = 700, 35, 20
    cor = inputs.Corpus("planted", V, 1.07, 5, C, Lg)
    ids = cor.tokens(0, 600_000)
    sent = ids.reshape(-1, Lg) % C
    assert np.all(sent == sent[:, :1])               # one cluster per sentence
    zq = cor.zipf_weights().astype(np.float64)
    ref = np.power(np.arange(1, V + 1, dtype=np.float64), -1.07)
    assert np.allclose(zq / zq.sum(), ref / ref.sum(), rtol=1e-9)
    # marginal over words = Zipf(s) exactly in expectation (reading B)
    hist = np.bincount(ids, minlength=V)
    top = 50
    e = zq / zq.sum() * ids.size
    assert np.all(np.abs(hist[:top] - e[:top]) < 6 * np.sqrt(e[:top] * Lg))


def test_configs_match_baseline():
    import json, os
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    b = json.load(open(os.path.join(here, "BASELINE.json")))
    assert len(b["configs"]) == 5
    c = inputs.CONFIGS
    assert (c[1].V, c[1].D, c[1].n, c[1].window, c[1].K, c[1].t) == (1000, 32, 20000, 2, 3, 0.0)
    assert (c[3].V, c[3].D, c[3].n, c[3].window, c[3].K, c[3].t) == (1_000_000, 300, 800_000_000, 5, 5, 1e-4)
    assert (c[4].V, c[4].D, c[4].window, c[4].K, c[4].t) == (1_000_000, 128, 8, 15, 1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_idx,i0,n", [(5, 0, 300_000), (5, 7_999_000_000, 200_000), (3, 123_456_789, 250_000),
                                          (1, 0, 20_000), (4, 5_000_000, 100_000)])
def test_gpu_generator_bitexact(cfg_idx, i0, n):
    """The on-device generator (gen_cuda.cu; BASELINE cfg5 is generated on-device) reproduces the
    host generator bit for bit on slices of the iid and planted corpora."""
    import torch
    cfg = inputs.CONFIGS[cfg_idx]
    c = cfg.corpus()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    c.tokens_cuda(i0, n, out)
    assert np.array_equal(out.cpu().numpy(), c.tokens(i0, n))
