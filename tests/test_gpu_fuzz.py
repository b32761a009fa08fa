"""Seeded random-shape parity sweep (deterministic mode) of the CUDA path against the oracle.

Each case draws a shape inside the library's envelope (include/w2v.h w2v_init: D % 4 == 0 up to
512 with the (D, K) register-tile limits; window up to 40 with the slab inside 227 KB; sentence_len
1-4096; ragged corpora, including empty, one-token and one-chunk ones; 1-2 epochs; subsampling on
or off; literal Alg.1 l.10 negatives or not) and checks, against the fp64 oracle (O-HB):
  * the batch stream (keep flags, b, N, context ids, negatives) bit-exact (1 epoch),
  * words / targets / row_touches / loss_pairs exact,
  * both matrices within the deterministic-mode bars of test_gpu_parity.assert_model_parity
    (the absolute 1e-5 of north_star only where an fp32 run of the oracle itself meets it: on
    degenerate draws — V <= 2, thousands of updates of the same rows — fp32 arithmetic alone
    drifts 4e-5-1e-4 from fp64, and the GPU must then match the fp32 oracle's accuracy),
for the default rows kernel and, where its window <= 15 limit allows, the ring kernel; and that the
conflict-ticketed mode 2 is bit-identical to mode 1 where it applies (2*window + K + 1 <= 32).
"""
import random

import numpy as np
import pytest

import inputs
import oracle
from test_gpu_parity import assert_model_parity, assert_stream_equal, rel_l2, run_gpu, w2v  # noqa: F401

pytestmark = pytest.mark.gpu

N_CASES = 96


def draw_case(seed):
    r = random.Random(1000 + seed)
    D = 4 * r.randint(1, 128)
    kmax = 31 if D <= 64 else 15 if D <= 192 else 7 if D <= 320 else 5
    K = r.randint(0, kmax)
    rs = 64 * ((D + 63) // 64)                       # the rows kernel's padded slab row (floats)
    kp1 = 1 << max(1, (K).bit_length())              # >= the register tile's KP1MAX
    wmax = max(1, min(40, ((200 * 1024) // (4 * rs) - kp1) // 2))
    window = r.randint(1, wmax)
    V = r.choice([1, 2, 7, 50, 300, 2000, 20000])
    L = r.choice([1, 2, 7, 20, 100, 1000, 4096])
    n = r.choice([0, 1, L + 1, r.randint(3, 15000), r.randint(3, 15000), r.randint(3, 15000), r.randint(3, 15000)])
    t = r.choice([0.0, 1e-2, 1e-3, 1e-4])
    epochs = r.choice([1, 1, 2])
    allow = r.choice([0, 0, 1])
    zipf = r.choice([0.8, 1.0, 1.2])
    return dict(V=V, D=D, window=window, K=K, L=L, n=n, t=t, epochs=epochs, allow=allow, zipf=zipf, seed=seed)


@pytest.mark.parametrize("case", range(N_CASES))
def test_random_shape_parity(w2v, case):  # noqa: F811
    c = draw_case(case)
    V, D, window, K, L, n, t = c["V"], c["D"], c["window"], c["K"], c["L"], c["n"], c["t"]
    ids = inputs.Corpus("iid", V, c["zipf"], 500 + case).tokens(0, n) if n else np.zeros(0, np.int32)
    # alpha scaled down for wide windows and tiny vocabularies (every input of a target hits the
    # same few rows there; alpha = 0.05 diverges to Inf at V = 2, window 24, D = 512)
    alpha = 0.025 * min(1.0, 5.0 / window) * (0.25 if V <= 7 else 1.0)
    seed = 11 + case
    tag = f"fuzz[{case}] V={V} D={D} w={window} K={K} L={L} n={n} t={t} E={c['epochs']} allow={c['allow']}"
    kernels = [1] + ([4] if window <= 15 else [])
    if n == 0:
        # an empty corpus is a successful no-op: the model stays at its init
        g = run_gpu(w2v, ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"])
        o_in, o_out, _, _ = oracle.train(ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"])
        assert np.array_equal(g["M_out"], np.zeros_like(g["M_out"])) and g["stats"]["words"] == 0
        assert np.allclose(g["M_in"], o_in, rtol=0, atol=0)
        return
    dbg = (0, n) if c["epochs"] == 1 else None
    o_in, o_out, o_st, o_dbg = oracle.train(ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"],
                                            allow_target_negative=bool(c["allow"]), debug=dbg)
    f_in, f_out, _, _ = oracle.train(ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"], prec="f32",
                                     allow_target_negative=bool(c["allow"]))
    results = {}
    for kernel in kernels:
        w2v.finalize()
        g = run_gpu(w2v, ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"], debug=dbg,
                    opts={"allow_target_negative": c["allow"], "kernel": kernel})
        if dbg:
            assert_stream_equal(g["dbg"], o_dbg)
        for k in ("words", "targets", "row_touches", "loss_pairs"):
            assert g["stats"][k] == o_st[k], (tag, kernel, k)
        assert_model_parity(f"{tag} kernel {kernel}", g["M_in"], g["M_out"], o_in, o_out, f_in, f_out,
                            abs_bar=max(rel_l2(f_in, o_in), rel_l2(f_out, o_out)) <= 1e-5)
        results[kernel] = g
    R = 2 * window + K + 1
    if R <= 32:
        w2v.finalize()
        # (a chunk's ticket table [L][R] u32 lives in shared memory, or in global memory when it
        # does not fit beside the slab: long chunks x many rows per target)
        g2 = run_gpu(w2v, ids, V, D, window, K, alpha, t, seed, L, epochs=c["epochs"], mode=2,
                     opts={"allow_target_negative": c["allow"], "kernel": 1})
        assert np.array_equal(g2["M_in"], results[1]["M_in"]) and np.array_equal(g2["M_out"], results[1]["M_out"]), tag
