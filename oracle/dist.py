"""TEST INFRASTRUCTURE ONLY — the oracle's data-parallel protocol (C13, reading R13).

PAPER.md:154-157 ("we employ data parallelism for distributed computation ... we skip the
details here") and PAPER.md:186 ("increase the model synchronization frequency"): W replicas,
each trains on its own contiguous chunk-aligned corpus shard, and every replica is replaced by
the elementwise mean of all replicas after each sync interval. Plain Python over the oracle's
`train_range`; the averaging is a callable so it can run in-process or over torch.distributed
(gloo) in the multi-process CPU tests.
"""
from __future__ import annotations

import numpy as np

from . import OrcStats, counts, init, make_params, real_dtype, sampler, thresholds, train_range


def shard_chunks(n: int, L: int, W: int, r: int) -> tuple[int, int]:
    """C13: S = ceil(n/L) chunks; rank r owns chunks [floor(r*S/W), floor((r+1)*S/W))."""
    S = (n + L - 1) // L
    return (r * S) // W, ((r + 1) * S) // W


def sync_intervals(n: int, L: int, W: int, r: int, P: int) -> list[tuple[int, int]]:
    """C13: I = max(1, P // L) chunks per interval; J = max(1, floor(min_r S_r / I)) intervals
    per epoch on every rank (so all ranks sync equally often); the last absorbs the remainder."""
    I = max(1, P // L)
    mins = min(shard_chunks(n, L, W, q)[1] - shard_chunks(n, L, W, q)[0] for q in range(W))
    J = max(1, mins // I)
    lo, hi = shard_chunks(n, L, W, r)
    return [(lo + k * I, hi if k == J - 1 else lo + (k + 1) * I) for k in range(J)]


def synced_rows(k: int, J: int, V: int, hot_rows: int = 0, cold_every: int = 1) -> list[tuple[int, int]]:
    """C14 (hot/cold averaging): row ranges averaged after interval k of
    J. Rows [0, H) (the Zipf-hot prefix: ids are frequency ranks) after every interval; rows
    [H, V) after every `cold_every`-th interval and after the last one of the epoch. H = 0 (or
    >= V) or cold_every = 1 is C13's full average after every interval."""
    H = V if hot_rows <= 0 or hot_rows >= V else hot_rows
    if H == V or cold_every <= 1 or (k + 1) % cold_every == 0 or k == J - 1:
        return [(0, V)]
    return [(0, H)]


def train_replica(ids_global, V, D, window, K, alpha0, t, seed, L, W, r, P, average, epochs=1,
                  prec="f64", counts_global=None, debug=None, lr_quantum=10_000, hot_rows=0, cold_every=1,
                  overlap=False):
    """Run replica r of W on its shard. `average(M_in, M_out)` must replace both matrices by the
    mean over replicas (called after every interval when W > 1, with row-slice views of the
    matrices when C14 averages only the hot prefix). Returns (M_in, M_out, stats, dbg).

    overlap=True is C15: the rows due after interval k are SNAPSHOT (S = C = M[rows]),
    S is averaged while interval k+1 trains, and after interval k+1 the replica applies
    M[rows] += S - C (the average's correction, one interval late). The last interval of an epoch
    applies any pending correction and then replaces the whole model by the plain mean (C13), so
    the replicas end identical.
    """
    from . import Debug
    n = ids_global.size
    lo, hi = shard_chunks(n, L, W, r)
    start, end = lo * L, min(hi * L, n)
    c = counts(ids_global, V) if counts_global is None else counts_global
    thr, Ptab = thresholds(c, n, t), sampler(c)
    dt = real_dtype(prec)
    mi, mo = init(V, D, seed)
    M_in, M_out = mi.astype(dt), mo.astype(dt)
    prm = make_params(V, D, window, K, alpha0, t, seed, L, epochs, n, W, lr_quantum)
    st = OrcStats()
    dbg = Debug(debug[0], debug[1], window, K) if debug else None
    shard = np.ascontiguousarray(ids_global[start:end])
    for e in range(epochs):
        iv = sync_intervals(n, L, W, r, P)
        pending = None  # C15: (lo, hi, S_in, S_out, C_in, C_out) of the average in flight
        for k, (a, b) in enumerate(iv):
            train_range(prm, thr, Ptab, shard, start, start, end - start, e, a, b, M_in, M_out, st, dbg, prec)
            if W == 1:
                continue
            if not overlap:
                for lo_r, hi_r in synced_rows(k, len(iv), V, hot_rows, cold_every):
                    average(M_in[lo_r:hi_r], M_out[lo_r:hi_r])
                continue
            if pending is not None:
                lo_p, hi_p, s_in, s_out, c_in, c_out = pending
                M_in[lo_p:hi_p] += s_in - c_in
                M_out[lo_p:hi_p] += s_out - c_out
                pending = None
            if k == len(iv) - 1:
                average(M_in, M_out)  # the epoch ends with the plain mean: identical replicas
                continue
            (lo_r, hi_r), = synced_rows(k, len(iv), V, hot_rows, cold_every)
            s_in, s_out = M_in[lo_r:hi_r].copy(), M_out[lo_r:hi_r].copy()
            c_in, c_out = s_in.copy(), s_out.copy()
            average(s_in, s_out)  # in flight during interval k+1 on the GPU
            pending = (lo_r, hi_r, s_in, s_out, c_in, c_out)
    return M_in, M_out, st.as_dict(), dbg
