"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it follows. None of them re-types the oracle's own formula: they
use printed values (tests/golden/, cited), closed forms (the SGNS loss gradient), equivalences
the paper states (HogBatch = Alg.1 at N=1), library routines (numpy searchsorted / power),
invariants and statistics.
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- RNG (C1) ---------
def _kat():
    rows = []
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[0:4], w[4:6], tuple(w[6:10])))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answers(ctr, key, out):
    assert oracle.philox(ctr, key) == out
    assert inputs.philox4x32_10(ctr, key) == out


def test_rng_counter_layout():
    # counter = (p lo, p hi, e, tag<<24 | idx), key = (seed lo, seed hi)   (C1)
    seed, p = 0x0123456789ABCDEF, (7 << 32) | 5
    assert oracle.rng_block(seed, 2, 3, p, 9) == oracle.philox([5, 7, 3, (2 << 24) | 9],
                                                               [0x89ABCDEF, 0x01234567])
    o = oracle.rng_block(seed, 2, 3, p, 4)
    assert oracle.rng_u64(seed, 2, 3, p, 8) == (o[1] << 32) | o[0]
    assert oracle.rng_u64(seed, 2, 3, p, 9) == (o[3] << 32) | o[2]


# ---------------------------------------------------------------- Alg.1 worked example --------
def test_alg1_spec_worked_example():
    """Alg.1, D=1, alpha=0.1 — line 15 before line 17."""
    g = _gold("spec_alg1_d1.json")
    M_in = np.zeros((3, 1)); M_out = np.zeros((3, 1))
    w, t, n = 0, 1, 2
    M_in[w, 0], M_out[t, 0], M_out[n, 0] = g["m_in_w"], g["m_out_t"], g["m_out_n"]
    oracle.alg1_step(M_in, M_out, [w], t, [[n]], g["alpha"])
    tol = g["tolerance"]
    assert abs(M_out[t, 0] - g["m_out_t_after"]) < tol
    assert abs(M_out[n, 0] - g["m_out_n_after"]) < tol
    assert abs(M_in[w, 0] - g["m_in_w_after"]) < tol
    # the errors printed at SPEC.md:257/337 follow from the row changes: dOut = alpha*err*m_in
    assert abs((M_out[t, 0] - g["m_out_t"]) / (g["alpha"] * g["m_in_w"]) - g["err_pos"]) < tol
    assert abs((M_out[n, 0] - g["m_out_n"]) / (g["alpha"] * g["m_in_w"]) - g["err_neg"]) < tol


def test_hogbatch_spec_worked_example():
    """the same example through HogBatch (N=1, K=1, distinct ids) is identical."""
    g = _gold("spec_alg1_d1.json")
    M_in = np.zeros((3, 1)); M_out = np.zeros((3, 1))
    M_in[0, 0], M_out[1, 0], M_out[2, 0] = g["m_in_w"], g["m_out_t"], g["m_out_n"]
    oracle.hogbatch_step(M_in, M_out, [0], [1, 2], g["alpha"])
    tol = g["tolerance"]
    assert abs(M_out[1, 0] - g["m_out_t_after"]) < tol
    assert abs(M_out[2, 0] - g["m_out_n_after"]) < tol
    assert abs(M_in[0, 0] - g["m_in_w_after"]) < tol


def test_sigmoid_values_and_zero_input():
    """SPEC.md:142-143 sigma(0)=0.5, sigma(6)=0.997527; SPEC.md:335 C=0 => E=+-0.5."""
    g = _gold("spec_values.json")
    a = 0.5
    # N=1, K=0, D=1: A=[[1]], B=[[6]] -> dIn = alpha*(1-sigma(6))*6, dOut = alpha*(1-sigma(6))*1
    M_in = np.array([[1.0]]); M_out = np.array([[6.0]])
    oracle.hogbatch_step(M_in, M_out, [0], [0], a)
    sig6 = 1.0 - (M_in[0, 0] - 1.0) / (a * 6.0)
    assert abs(sig6 - g["sigma6"]) < g["sigma_tol"]
    # zero input rows: C = 0 -> err = 0.5 (target) / -0.5 (negatives); M_out unchanged
    D = 4
    rng = np.random.default_rng(0)
    M_in = np.zeros((2, D)); M_out = rng.normal(size=(4, D))
    Mo0 = M_out.copy()
    oracle.hogbatch_step(M_in, M_out, [1], [0, 2, 3], a)
    assert np.array_equal(M_out, Mo0)
    expect = a * (g["sigma0"] * Mo0[0] - g["sigma0"] * Mo0[2] - g["sigma0"] * Mo0[3])
    assert np.allclose(M_in[1], expect, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- gradient (closed form) -----
def _sgns_loss(M_in, M_out, ctx, outs):
    """The SGNS minibatch objective: sum_i -log s(C_i0) - sum_j>=1 log s(-C_ij)."""
    A, B = M_in[ctx], M_out[outs]
    C = A @ B.T
    lab = np.zeros(len(outs)); lab[0] = 1.0
    return float(np.sum(np.logaddexp(0, -C) * lab + np.logaddexp(0, C) * (1 - lab)))


def test_update_is_minus_alpha_gradient_fd():
    """Alg.1 l.13-20 / HogBatch: dIn = -alpha dL/dA, dOut = -alpha dL/dB,
    central finite differences in fp64 over random tiny instances incl. duplicate ids."""
    rng = np.random.default_rng(1)
    worst = 0.0
    for trial in range(200):
        V, D = int(rng.integers(2, 12)), int(rng.integers(1, 9))
        N, K = int(rng.integers(1, 11)), int(rng.integers(0, 11))
        ctx = rng.integers(0, V, N).astype(np.int32)
        outs = rng.integers(0, V, K + 1).astype(np.int32)
        M_in = rng.normal(scale=0.5, size=(V, D)); M_out = rng.normal(scale=0.5, size=(V, D))
        alpha = 1e-3
        mi, mo = M_in.copy(), M_out.copy()
        oracle.hogbatch_step(mi, mo, ctx, outs, alpha)
        # the *first-order* step equals -alpha * grad of the loss w.r.t. the whole model
        h = 1e-6
        for M, upd in ((M_in, mi - M_in), (M_out, mo - M_out)):
            g = np.zeros_like(M)
            for idx in np.ndindex(*M.shape):
                if not (np.any(ctx == idx[0]) if M is M_in else np.any(outs == idx[0])):
                    continue
                Mp, Mm = M.copy(), M.copy()
                Mp[idx] += h; Mm[idx] -= h
                lp = _sgns_loss(Mp, M_out, ctx, outs) if M is M_in else _sgns_loss(M_in, Mp, ctx, outs)
                lm = _sgns_loss(Mm, M_out, ctx, outs) if M is M_in else _sgns_loss(M_in, Mm, ctx, outs)
                g[idx] = (lp - lm) / (2 * h)
            ref = -alpha * g
            den = max(np.linalg.norm(ref), 1e-12)
            rel = np.linalg.norm(upd - ref) / den
            worst = max(worst, rel)
    assert worst < 1e-4, worst


def test_hogbatch_equals_alg1_when_N1_distinct():
    """N=1 and distinct outputs -> HogBatch bit-equals Alg.1 in fp64
    (PAPER.md:116-126 vs 37-63; line 15 reads M_out before line 17 writes it)."""
    rng = np.random.default_rng(2)
    for trial in range(300):
        V, D, K = 20, int(rng.integers(1, 9)), int(rng.integers(0, 10))
        outs = rng.choice(V, K + 1, replace=False).astype(np.int32)
        ctx = np.array([rng.integers(0, V)], np.int32)
        M_in = rng.normal(size=(V, D)); M_out = rng.normal(size=(V, D))
        a1_in, a1_out = M_in.copy(), M_out.copy()
        hb_in, hb_out = M_in.copy(), M_out.copy()
        oracle.alg1_step(a1_in, a1_out, ctx, outs[0], outs[1:].reshape(1, K), 0.05)
        oracle.hogbatch_step(hb_in, hb_out, ctx, outs, 0.05)
        assert np.allclose(a1_out, hb_out, rtol=0, atol=1e-15)
        # M_in: Alg.1 does alpha*sum(err*B) vs HogBatch sum((alpha*err)*B): equal up to rounding
        assert np.allclose(a1_in, hb_in, rtol=1e-14, atol=1e-15)


def test_hogbatch_equals_stale_read_scalar():
    """for general N, HogBatch = Alg.1 with every read taken from the batch-start
    snapshot (reading R11), over random instances with duplicates."""
    rng = np.random.default_rng(3)
    sig = lambda x: 1.0 / (1.0 + math.exp(-x))
    for trial in range(300):
        V, D = int(rng.integers(2, 50)), int(rng.integers(1, 9))
        N, K = int(rng.integers(1, 11)), int(rng.integers(0, 11))
        ctx = rng.integers(0, V, N).astype(np.int32)
        outs = rng.integers(0, V, K + 1).astype(np.int32)
        M_in = rng.normal(size=(V, D)); M_out = rng.normal(size=(V, D))
        snap_in, snap_out = M_in.copy(), M_out.copy()
        ref_in, ref_out = M_in.copy(), M_out.copy()
        a = float(np.float32(0.025))            # alpha is fp32 by contract (C8)
        for i in range(N):                      # Alg.1 loop structure, stale reads
            temp = np.zeros(D)
            for k in range(K + 1):
                tw, label = outs[k], (1.0 if k == 0 else 0.0)
                inn = float(np.dot(snap_in[ctx[i]], snap_out[tw]))
                err = label - sig(inn)
                temp += err * snap_out[tw]
                ref_out[tw] += a * err * snap_in[ctx[i]]
            ref_in[ctx[i]] += a * temp
        oracle.hogbatch_step(M_in, M_out, ctx, outs, a)
        assert np.allclose(M_in, ref_in, rtol=1e-12, atol=1e-14)
        assert np.allclose(M_out, ref_out, rtol=1e-12, atol=1e-14)


def test_only_touched_rows_change_and_zero_error():
    """SPEC.md:217 (only named rows change) and SPEC.md:345 (E=0 -> model unchanged)."""
    rng = np.random.default_rng(4)
    V, D = 30, 6
    M_in = rng.normal(size=(V, D)); M_out = rng.normal(size=(V, D))
    ctx, outs = np.array([3, 5, 3], np.int32), np.array([7, 9, 9, 11], np.int32)
    mi, mo = M_in.copy(), M_out.copy()
    oracle.hogbatch_step(mi, mo, ctx, outs, 0.1)
    chg_in = np.where(np.any(mi != M_in, axis=1))[0]
    chg_out = np.where(np.any(mo != M_out, axis=1))[0]
    assert set(chg_in) <= {3, 5} and set(chg_out) <= {7, 9, 11}
    # huge positive dot on the target and huge negative on negatives -> err ~ 0 in fp64? use alpha=0
    mi, mo = M_in.copy(), M_out.copy()
    oracle.hogbatch_step(mi, mo, ctx, outs, 0.0)
    assert np.array_equal(mi, M_in) and np.array_equal(mo, M_out)


def test_loss_decreases_repeated_batch():
    """repeating one batch with small alpha strictly decreases its SGNS loss."""
    rng = np.random.default_rng(5)
    V, D = 20, 8
    M_in = rng.normal(scale=0.3, size=(V, D)); M_out = rng.normal(scale=0.3, size=(V, D))
    ctx, outs = np.array([1, 2, 3, 4], np.int32), np.array([5, 6, 7, 8, 9, 10], np.int32)
    prev = None
    for it in range(100):
        cur = _sgns_loss(M_in, M_out, ctx, outs)
        ret = oracle.hogbatch_step(M_in, M_out, ctx, outs, 0.01)
        assert abs(ret - cur) < 1e-9 * max(1, cur)       # returned loss = pre-update loss
        if prev is not None:
            assert cur < prev
        prev = cur


# ---------------------------------------------------------------- sampler (C3) --------------
def test_sampler_weights_and_invcdf_vs_library():
    """Reading R1: q[w] = floor(c^0.75 * 2^20) with c^0.75 = sqrt(c)*sqrt(sqrt(c));
    invcdf is numpy.searchsorted on the prefix; every w is hit by exactly q[w] values of x."""
    rng = np.random.default_rng(6)
    c = rng.integers(0, 5000, 300).astype(np.int64)
    c[[0, 17, 299]] = 0
    P = oracle.sampler(c)
    q = np.diff(P).astype(np.float64)
    ref = np.power(c.astype(np.float64), 0.75) * 2**20
    assert np.all(np.abs(q - ref) <= 1.0 + 1e-9 * ref)
    assert np.all(q[c == 0] == 0)
    xs = [int(x) for x in rng.integers(0, int(P[-1]), 2000, dtype=np.uint64)]
    for w in np.nonzero(q)[0]:
        xs += [int(P[w]), int(P[w + 1]) - 1]
    for x in xs:
        w = oracle.invcdf(P, x)
        assert w == int(np.searchsorted(P[1:], np.uint64(x), side="right"))
        assert P[w] <= x < P[w + 1]


def test_sampler_two_word_share():
    """counts {a:4, b:1}, power 0.75 -> share(a) = 0.7388."""
    g = _gold("spec_values.json")
    P = oracle.sampler(np.array([4, 1], np.int64))
    assert abs(int(P[1]) / int(P[2]) - g["share_a4_b1"]) < g["share_tol"]


def test_negative_draws_chi2_and_exclusion():
    """Alg.1 l.10 with readings R1/R2: draws follow q/P[V] renormalised without the target
    (chi-square), never equal the target; allow_target_negative restores literal l.10."""
    from scipy import stats
    c = np.array([50, 30, 10, 5, 3, 1, 1, 0, 7, 2], np.int64)
    P = oracle.sampler(c)
    q = np.diff(P).astype(np.float64)
    tw = 1
    draws = []
    for p in range(4000):
        draws += oracle.draw_negatives(77, 0, p, P, tw, 5)
    draws = np.array(draws)
    assert not np.any(draws == tw)
    hist = np.bincount(draws, minlength=10).astype(np.float64)
    pexp = q.copy(); pexp[tw] = 0; pexp /= pexp.sum()
    m = pexp > 0
    chi2 = stats.chisquare(hist[m], pexp[m] * hist.sum())
    assert chi2.pvalue > 1e-4
    assert hist[~m].sum() == 0
    lit = []
    for p in range(2000):
        lit += oracle.draw_negatives(77, 0, p, P, tw, 5, allow_target_negative=True)
    assert np.any(np.array(lit) == tw)


def test_negative_fallback_after_100_tries():
    """Reading R2: if only the target has mass, 100 tries fail and (tw+1) mod V is returned."""
    P = oracle.sampler(np.array([0, 0, 9], np.int64))
    assert oracle.draw_negatives(1, 0, 0, P, 2, 3) == [0, 0, 0]


# ---------------------------------------------------------------- subsampling / window -------
def test_keep_thresholds_spec_values():
    """z=4 -> 0.75, z=1 -> 1 (clamp), sample=0 -> 1 (reading R5)."""
    g = _gold("spec_values.json")
    T = 10_000
    thr = oracle.thresholds(np.array([4, 1, 10_000], np.int64), T, 1e-4)
    assert abs(int(thr[0]) / 2**32 - g["keep_z4"]) < 1e-6
    assert int(thr[1]) == 2**32 and g["keep_z1"] == 1.0
    z = 10_000 / (float(np.float32(1e-4)) * T)
    assert abs(int(thr[2]) / 2**32 - (math.sqrt(z) + 1) / z) < 1e-9
    assert np.all(oracle.thresholds(np.array([4, 1, 10_000], np.int64), T, 0.0) == 2**32)


def test_keep_rate_and_window_distribution():
    """Subsampling keep-rate per word matches thr/2^32 (binomial z-test) and b is uniform on
    {1..window} (SPEC.md:134 chi-square)."""
    from scipy import stats
    cfg = inputs.CONFIGS[1]
    ids = inputs.Corpus("iid", 50, 1.0, 42).tokens(0, 200_000)
    V, window, t = 50, 5, 1e-2
    _, _, _, dbg = oracle.train(ids, V, 4, window, 1, 0.0, t, 9, 1000, debug=(0, ids.size))
    c = oracle.counts(ids, V)
    thr = oracle.thresholds(c, ids.size, t)
    for w in range(8):
        m = ids == w
        p = int(thr[w]) / 2**32
        k = int(dbg.keep[m].sum()); n = int(m.sum())
        zsc = (k - n * p) / math.sqrt(max(n * p * (1 - p), 1e-9))
        assert abs(zsc) < 5, (w, k, n, p)
    b = dbg.b[dbg.keep == 1]
    assert b.min() >= 1 and b.max() <= window
    hist = np.bincount(b, minlength=window + 1)[1:]
    assert stats.chisquare(hist).pvalue > 1e-4
    assert abs(hist[0] / hist.sum() - 0.2) < 0.01


def test_batch_construction_rules():
    """Reading R6/R7: ctx = kept neighbours within b on the compacted chunk, never crossing a
    chunk; N = |ctx|; positions with N=0 are not trained; row_touches = sum(N+K+1)."""
    ids = inputs.Corpus("iid", 40, 1.0, 5).tokens(0, 3_000)
    V, window, K, L = 40, 3, 2, 100
    _, _, st, dbg = oracle.train(ids, V, 4, window, K, 0.01, 5e-2, 11, L, debug=(0, ids.size))
    touches = 0
    for s in range(0, ids.size, L):
        kept = [p for p in range(s, min(s + L, ids.size)) if dbg.keep[p]]
        for m, p in enumerate(kept):
            b = int(dbg.b[p])
            nb = [ids[kept[j]] for j in range(max(0, m - b), min(len(kept), m + b + 1)) if j != m]
            assert int(dbg.N[p]) == len(nb)
            assert list(dbg.ctx[p, :len(nb)]) == nb
            assert np.all(dbg.ctx[p, len(nb):] == -1)
            if nb:
                touches += len(nb) + K + 1
                assert np.all(dbg.neg[p] != ids[p])
    assert st["row_touches"] == touches
    assert np.all(dbg.b[dbg.keep == 0] == 0)


def test_update_count_hogbatch_vs_alg1():
    """PAPER.md:140-149 (HogBatch "cut[s] down on the total number of updates"); SPEC.md:360:
    row writes N+(K+1) per target for HogBatch vs N(K+1)+N for Alg.1, exactly."""
    ids = inputs.Corpus("iid", 60, 1.0, 8).tokens(0, 5_000)
    V, window, K = 60, 2, 3
    _, _, hb, dbg = oracle.train(ids, V, 4, window, K, 0.01, 0.0, 3, 500, debug=(0, ids.size))
    _, _, a1, _ = oracle.train(ids, V, 4, window, K, 0.01, 0.0, 3, 500, algorithm=1)
    Ns = dbg.N[dbg.N > 0].astype(np.int64)
    assert hb["row_touches"] == int(np.sum(Ns + K + 1))
    assert a1["row_touches"] == int(np.sum(Ns * (K + 1) + Ns))
    assert hb["targets"] == a1["targets"] == Ns.size
    assert hb["row_touches"] < a1["row_touches"]


def test_alg1_per_input_negatives():
    """Alg.1 l.10 draws its negatives per input word (reading R4 contrasts HogBatch's shared set):
    O-A1's recorded per-input negatives never equal the target, follow q/P[V] renormalised without
    the target (chi-square over all inputs), differ between the inputs of one target (independent
    draws), and the training step they feed is Alg.1 verbatim (loss pairs N(K+1))."""
    from scipy import stats
    V, window, K = 10, 3, 5
    ids = inputs.Corpus("iid", V, 0.7, 5).tokens(0, 6_000)
    _, _, st, dbg = oracle.train(ids, V, 4, window, K, 0.01, 0.0, 9, 200, algorithm=1, debug=(0, ids.size))
    c = oracle.counts(ids, V)
    q = np.diff(oracle.sampler(c)).astype(np.float64)
    hist = np.zeros(V)
    distinct_inputs = 0
    for p in np.flatnonzero(dbg.N):
        N = int(dbg.N[p])
        negs = dbg.a1neg[p, :N, :]
        assert np.all(negs >= 0) and np.all(negs != ids[p])
        assert np.all(dbg.a1neg[p, N:, :] == -1)
        distinct_inputs += int(len({tuple(r) for r in negs}) == N)
        hist += np.bincount(negs.ravel(), minlength=V)
    assert distinct_inputs > 0.95 * np.count_nonzero(dbg.N)
    # pooled over targets the expected share of w is sum_t q_w / (P - q_t) (w != t)
    exp = np.zeros(V)
    for p in np.flatnonzero(dbg.N):
        pexp = q.copy(); pexp[ids[p]] = 0; pexp /= pexp.sum()
        exp += pexp * int(dbg.N[p]) * K
    m = exp > 5
    assert stats.chisquare(hist[m], exp[m] * hist[m].sum() / exp[m].sum()).pvalue > 1e-4
    assert st["loss_pairs"] == int(dbg.N.astype(np.int64).sum() * (K + 1))


# ---------------------------------------------------------------- init / alpha ---------------
def test_init_range_and_distribution():
    """Reading R10: M_in ~ U[-0.5/D, 0.5/D), M_out = 0, deterministic."""
    from scipy import stats
    V, D = 500, 40
    M_in, M_out = oracle.init(V, D, 123)
    assert np.all(M_out == 0)
    assert M_in.min() >= -0.5 / D and M_in.max() < 0.5 / D
    assert stats.kstest(M_in.ravel() * D + 0.5, "uniform").pvalue > 1e-4
    M2, _ = oracle.init(V, D, 123)
    assert np.array_equal(M_in, M2)
    M3, _ = oracle.init(V, D, 124)
    assert not np.array_equal(M_in, M3)


def test_alpha_schedule_endpoints():
    """alpha(0)=alpha0, alpha(end)=1e-4*alpha0 (floor), midpoint ~0.5*alpha0."""
    a0, n, Q = 0.025, 1_000_000, 10_000
    assert oracle.alpha(a0, 0, Q, 1, 1, n) == np.float32(a0)
    assert abs(oracle.alpha(a0, n, Q, 1, 1, n) - 1e-4 * a0) < 1e-9
    assert abs(oracle.alpha(a0, n // 2, Q, 1, 1, n) - 0.5 * a0) < 1e-6
    # quantised every Q words, non-increasing
    vals = [oracle.alpha(a0, pi, Q, 1, 1, n) for pi in range(0, n, 2500)]
    assert all(x >= y for x, y in zip(vals, vals[1:]))
    assert oracle.alpha(a0, Q - 1, Q, 1, 1, n) == oracle.alpha(a0, 0, Q, 1, 1, n)
    # W replicas each at pi/W progress see the single-run schedule
    assert oracle.alpha(a0, n // 4, Q, 2, 1, n) == oracle.alpha(a0, n // 2, Q, 1, 1, n)


# ---------------------------------------------------------------- brute-force loss, V=10 -----
def test_bruteforce_expected_loss_v10():
    """Frozen model (alpha=0), V=10, window=1, no subsampling: the Monte-Carlo SGNS loss of the
    run equals the exactly enumerated expectation over the renormalised unigram^0.75 negatives
    (reading R1/R2) within a CLT bound."""
    rng = np.random.default_rng(9)
    V, D, K = 10, 6, 4
    ids = rng.integers(0, V, 30_000).astype(np.int32)
    ids[ids == 9] = 8                               # a zero-count word is never drawn
    M_in = rng.normal(scale=0.6, size=(V, D)).astype(np.float32)
    M_out = rng.normal(scale=0.6, size=(V, D)).astype(np.float32)
    L = 30_000
    _, _, st, _ = oracle.train(ids, V, D, 1, K, 0.0, 0.0, 21, L, model=(M_in, M_out))
    c = np.bincount(ids, minlength=V).astype(np.float64)
    q = np.floor(np.power(c, 0.75) * 2**20)
    C = M_in.astype(np.float64) @ M_out.astype(np.float64).T
    sp = lambda x: np.logaddexp(0, x)
    exp_loss, var = 0.0, 0.0
    n = ids.size
    for p in range(n):
        tw = ids[p]
        pi = q.copy(); pi[tw] = 0; pi /= pi.sum()
        for pp in (p - 1, p + 1):
            if 0 <= pp < n:
                x = ids[pp]
                neg = sp(C[x]) @ pi
                neg2 = (sp(C[x]) ** 2) @ pi
                exp_loss += sp(-C[x, tw]) + K * neg
                var += K * (neg2 - neg ** 2)
    assert st["loss_pairs"] == (2 * n - 2) * (K + 1)
    assert abs(st["loss_sum"] - exp_loss) < 5 * math.sqrt(var), (st["loss_sum"], exp_loss, math.sqrt(var))


# ---------------------------------------------------------------- planted-cluster recall -----
def recall_at_k(M, words, C, k=10):
    X = M / np.maximum(np.linalg.norm(M, axis=1, keepdims=True), 1e-30)
    S = X[words] @ X.T
    S[np.arange(len(words)), words] = -np.inf
    nn = np.argpartition(-S, k, axis=1)[:, :k]
    return float(np.mean((nn % C) == (np.asarray(words)[:, None] % C)))


def test_planted_cluster_recall():
    """Similarity recovery (north star): on a planted-cluster corpus, same-cluster recall@10 of
    cosine neighbours on M_in is far above chance (M/V)."""
    V, C, D = 600, 30, 32
    cor = inputs.Corpus("planted", V, 1.07, 17, C, 20)
    ids = cor.tokens(0, 400_000)
    M_in, _, st, _ = oracle.train(ids, V, D, 5, 5, 0.025, 1e-3, 17, 20, prec="f32")
    words = np.arange(100)
    r = recall_at_k(M_in.astype(np.float64), words, C)
    chance = (V / C - 1) / (V - 1)
    assert r > 0.6 and r > 10 * chance, r
    assert st["loss_sum"] / st["loss_pairs"] < math.log(2)


# ---------------------------------------------------------------- averaging -----------------
def test_average_examples():
    """SPEC.md:403-405 / 417-419: mean of 0.2 and 0.4 is 0.3; identical replicas unchanged;
    W=1 identity; permutation invariant; zero discrepancy afterwards."""
    g = _gold("spec_values.json")
    a, b = np.full(5, 0.2), np.full(5, 0.4)
    oracle.average([a, b])
    assert np.allclose(a, g["mean_02_04"], atol=1e-15) and np.array_equal(a, b)
    rng = np.random.default_rng(10)
    x = rng.normal(size=100); y = x.copy()
    oracle.average([x, y])
    assert np.array_equal(x, y)
    z = rng.normal(size=100); z0 = z.copy()
    oracle.average([z])
    assert np.array_equal(z, z0)
    r = [rng.normal(size=50) for _ in range(3)]
    r1 = [v.copy() for v in r]; r2 = [r[2].copy(), r[0].copy(), r[1].copy()]
    oracle.average(r1); oracle.average(r2)
    assert np.allclose(r1[0], r2[0], rtol=1e-15, atol=1e-15)
    assert np.allclose(r1[0], np.mean(r, axis=0), atol=1e-15)


def test_threaded_hogwild_oracle_mode_counts():
    """The oracle's threaded Hogwild mode (CPU timing baseline only): one thread
    is the sequential run bit for bit; T threads process exactly the same batch stream (position-
    keyed RNG), so words/targets/row_touches/loss_pairs match the sequential run and the loss is
    close (the model interleaving differs)."""
    cfg = inputs.CONFIGS[2]
    n = 60_000
    ids = cfg.corpus().tokens(0, n)
    c = oracle.counts(ids, cfg.V)
    thr, P = oracle.thresholds(c, n, cfg.t), oracle.sampler(c)
    prm = oracle.make_params(cfg.V, 32, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed, cfg.L, 1, n)
    nch = (n + cfg.L - 1) // cfg.L
    res = {}
    for T in (0, 1, 4):
        mi, mo = oracle.init(cfg.V, 32, cfg.seed)
        M_in, M_out = mi.astype(np.float64), mo.astype(np.float64)
        st = oracle.OrcStats()
        if T == 0:
            oracle.train_range(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, st)
        else:
            oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, st, T)
        res[T] = (M_in, M_out, st.as_dict())
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    for k in ("words", "targets", "row_touches", "loss_pairs"):
        assert res[4][2][k] == res[0][2][k], k
    assert abs(res[4][2]["loss_sum"] / res[0][2]["loss_sum"] - 1) < 0.02


def test_counts_equal_bincount_and_reject_out_of_range():
    """a0 histogram (SPEC.md:49-57 word counts): orc_counts equals numpy's
    bincount exactly on Zipf, uniform and edge corpora (ids at 0 and V-1, V=1, empty corpus), and
    an id outside [0, V) — either side — is rejected (SPEC.md:253 precondition)."""
    rng = np.random.default_rng(11)
    cases = [(inputs.Corpus("iid", 1000, 1.0, 3).tokens(0, 50_000), 1000),
             (rng.integers(0, 77, 9_999).astype(np.int32), 77),
             (np.array([0, 4, 4, 0, 4], np.int32), 5),
             (np.zeros(17, np.int32), 1),
             (np.zeros(0, np.int32), 3)]
    for ids, V in cases:
        c = oracle.counts(ids, V)
        assert c.dtype == np.int64 and c.shape == (V,)
        assert np.array_equal(c, np.bincount(ids, minlength=V).astype(np.int64))
        assert int(c.sum()) == ids.size
    for bad in (np.array([1, 2, 5], np.int32), np.array([0, -1], np.int32)):
        with pytest.raises(ValueError):
            oracle.counts(bad, 5)
