"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the plain sequential CPU oracle (w2v_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this. It shares no code with the CUDA path (paper_1611_06172_b200/); both implement the
written contract of DESIGN.md §2. Citations are to /root/reference/PAPER.md lines; see the C
file's header for the map.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "w2v_oracle.c")
# -O2, no fast-math, no FMA contraction: the oracle's fp arithmetic is the C source's, op by op.
CFLAGS = ["-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math"]


# TIMING-ONLY build (bench.py's cpu_baseline / reference arm): the same source in fp32 with
# -O3 -march=native for the host it runs on, FMA contraction allowed. Never a parity value; built
# on the box that times it (build_native), because -march=native code may not run elsewhere.
CFLAGS_NATIVE = ["-O3", "-march=native", "-fPIC", "-shared", "-fno-fast-math"]


def _so(prec: str) -> str:
    return os.path.join(_HERE, f"liboracle_{prec}.so")


def build(force: bool = False) -> None:
    for prec, real in (("f64", "double"), ("f32", "float")):
        so = _so(prec)
        if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
            subprocess.check_call(["gcc", *CFLAGS, f"-DREAL={real}", _SRC, "-o", so, "-lm", "-pthread"])


def build_native() -> str:
    """(Re)build the timing-only fp32 -O3 -march=native oracle for THIS host; returns its flags."""
    subprocess.check_call(["gcc", *CFLAGS_NATIVE, "-DREAL=float", _SRC, "-o", _so("f32native"), "-lm", "-pthread"])
    _libs.pop("f32native", None)
    return " ".join(CFLAGS_NATIVE) + " -DREAL=float"


class OrcParams(ctypes.Structure):
    _fields_ = [("V", ctypes.c_int64), ("D", ctypes.c_int32), ("window", ctypes.c_int32),
                ("K", ctypes.c_int32), ("alpha0", ctypes.c_float), ("t", ctypes.c_float),
                ("seed", ctypes.c_uint64), ("L", ctypes.c_int32),
                ("allow_target_negative", ctypes.c_int32), ("lr_quantum", ctypes.c_int64),
                ("epochs", ctypes.c_int32), ("n_global", ctypes.c_int64), ("world", ctypes.c_int32),
                ("algorithm", ctypes.c_int32)]


class OrcStats(ctypes.Structure):
    _fields_ = [("words", ctypes.c_int64), ("targets", ctypes.c_int64),
                ("row_touches", ctypes.c_int64), ("loss_pairs", ctypes.c_int64),
                ("loss_sum", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class OrcDebug(ctypes.Structure):
    _fields_ = [("base", ctypes.c_int64), ("len", ctypes.c_int64),
                ("keep", ctypes.POINTER(ctypes.c_uint8)), ("b", ctypes.POINTER(ctypes.c_uint8)),
                ("N", ctypes.POINTER(ctypes.c_uint8)), ("ctx", ctypes.POINTER(ctypes.c_int32)),
                ("neg", ctypes.POINTER(ctypes.c_int32)), ("a1neg", ctypes.POINTER(ctypes.c_int32))]


_libs: dict = {}
TAG_POS, TAG_NEG, TAG_INIT, TAG_GEN, TAG_EVAL, TAG_A1NEG = 1, 2, 3, 4, 5, 6


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def lib(prec: str = "f64"):
    if prec not in _libs:
        if prec == "f32native":
            if not os.path.exists(_so(prec)):
                build_native()
        else:
            build()
        L = ctypes.CDLL(_so(prec))
        u32p, u64p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
        i32p, i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
        realp = ctypes.c_void_p
        L.orc_philox.argtypes = [u32p, u32p, u32p]
        L.orc_rng_block.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_uint32, u32p]
        L.orc_rng_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                  ctypes.c_uint32]
        L.orc_rng_u64.restype = ctypes.c_uint64
        L.orc_counts.argtypes = [i32p, ctypes.c_int64, ctypes.c_int64, i64p]
        L.orc_thresholds.argtypes = [i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_float, u64p]
        L.orc_sampler.argtypes = [i64p, ctypes.c_int64, u64p]
        L.orc_invcdf.argtypes = [u64p, ctypes.c_int64, ctypes.c_uint64]
        L.orc_invcdf.restype = ctypes.c_int64
        L.orc_init.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_alpha.argtypes = [ctypes.c_float, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int64]
        L.orc_alpha.restype = ctypes.c_float
        L.orc_hogbatch_step.argtypes = [realp, realp, ctypes.c_int32, i32p, ctypes.c_int32, i32p, ctypes.c_int32,
                                        ctypes.c_float]
        L.orc_hogbatch_step.restype = ctypes.c_double
        L.orc_alg1_step.argtypes = [realp, realp, ctypes.c_int32, i32p, ctypes.c_int32, ctypes.c_int32, i32p,
                                    ctypes.c_int32, ctypes.c_float]
        L.orc_alg1_step.restype = ctypes.c_double
        L.orc_draw_negative.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, u32p, u64p,
                                        ctypes.c_int64, ctypes.c_int32, ctypes.c_int]
        L.orc_draw_negative.restype = ctypes.c_int32
        L.orc_train_range.argtypes = [ctypes.POINTER(OrcParams), u64p, u64p, i32p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_int64, realp, realp, ctypes.POINTER(OrcStats),
                                      ctypes.POINTER(OrcDebug)]
        L.orc_average.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int64]
        L.orc_train_range_hogwild.argtypes = [ctypes.POINTER(OrcParams), u64p, u64p, i32p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.c_int64, ctypes.c_int64, realp, realp, ctypes.POINTER(OrcStats),
                                              ctypes.c_int32]
        L.orc_real_size.restype = ctypes.c_int
        _libs[prec] = L
    return _libs[prec]


def real_dtype(prec: str):
    return np.float64 if prec == "f64" else np.float32   # "f32" and the timing-only "f32native"


# ------------------------------------------------------------------ primitives ---------------
def philox(ctr, key) -> tuple:
    a, k, o = np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), np.zeros(4, np.uint32)
    lib().orc_philox(_p(a, ctypes.c_uint32), _p(k, ctypes.c_uint32), _p(o, ctypes.c_uint32))
    return tuple(int(x) for x in o)


def rng_block(seed, tag, e, p, idx) -> tuple:
    o = np.zeros(4, np.uint32)
    lib().orc_rng_block(seed, tag, e, p, idx, _p(o, ctypes.c_uint32))
    return tuple(int(x) for x in o)


def rng_u64(seed, tag, e, p, d) -> int:
    return int(lib().orc_rng_u64(seed, tag, e, p, d))


def counts(ids: np.ndarray, V: int) -> np.ndarray:
    ids = np.ascontiguousarray(ids, np.int32)
    c = np.zeros(V, np.int64)
    rc = lib().orc_counts(_p(ids, ctypes.c_int32), ids.size, V, _p(c, ctypes.c_int64))
    if rc != 0:
        raise ValueError("id outside [0, V)")
    return c


def thresholds(c: np.ndarray, T: int, t: float) -> np.ndarray:
    c = np.ascontiguousarray(c, np.int64)
    thr = np.zeros(c.size, np.uint64)
    lib().orc_thresholds(_p(c, ctypes.c_int64), c.size, T, t, _p(thr, ctypes.c_uint64))
    return thr


def sampler(c: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(c, np.int64)
    P = np.zeros(c.size + 1, np.uint64)
    if lib().orc_sampler(_p(c, ctypes.c_int64), c.size, _p(P, ctypes.c_uint64)) != 0:
        raise ValueError("sampler total P[V] is 0")
    return P


def invcdf(P: np.ndarray, x: int) -> int:
    return int(lib().orc_invcdf(_p(P, ctypes.c_uint64), P.size - 1, x))


def draw_negatives(seed, e, p, P, tw, K, allow_target_negative=False):
    d = ctypes.c_uint32(0)
    V = P.size - 1
    return [int(lib().orc_draw_negative(seed, e, p, ctypes.byref(d), _p(P, ctypes.c_uint64), V, tw,
                                        int(allow_target_negative))) for _ in range(K)]


def init(V: int, D: int, seed: int):
    M_in = np.zeros((V, D), np.float32)
    M_out = np.zeros((V, D), np.float32)
    lib().orc_init(V, D, seed, M_in.ctypes.data, M_out.ctypes.data)
    return M_in, M_out


def alpha(alpha0, pi, Q, W, E, n_global) -> float:
    return float(lib().orc_alpha(alpha0, pi, Q, W, E, n_global))


def hogbatch_step(M_in, M_out, ctx, outs, alpha, prec="f64") -> float:
    """In-place O-HB step on REAL arrays (float64 for f64, float32 for f32)."""
    dt = real_dtype(prec)
    assert M_in.dtype == dt and M_out.dtype == dt and M_in.flags.c_contiguous and M_out.flags.c_contiguous
    ctx = np.ascontiguousarray(ctx, np.int32)
    outs = np.ascontiguousarray(outs, np.int32)
    return float(lib(prec).orc_hogbatch_step(M_in.ctypes.data, M_out.ctypes.data, M_in.shape[1],
                                             _p(ctx, ctypes.c_int32), ctx.size, _p(outs, ctypes.c_int32),
                                             outs.size - 1, alpha))


def alg1_step(M_in, M_out, ctx, target, negs, alpha, prec="f64") -> float:
    """In-place Algorithm 1 for one target; negs is N x K."""
    dt = real_dtype(prec)
    assert M_in.dtype == dt and M_out.dtype == dt
    ctx = np.ascontiguousarray(ctx, np.int32)
    negs = np.ascontiguousarray(negs, np.int32).reshape(ctx.size, -1)
    K = negs.shape[1]
    return float(lib(prec).orc_alg1_step(M_in.ctypes.data, M_out.ctypes.data, M_in.shape[1],
                                         _p(ctx, ctypes.c_int32), ctx.size, int(target),
                                         _p(negs, ctypes.c_int32), K, alpha))


def average(reps: list) -> None:
    """In-place elementwise mean of W same-shaped REAL replicas (R13)."""
    prec = "f64" if reps[0].dtype == np.float64 else "f32"
    arr = (ctypes.c_void_p * len(reps))(*[r.ctypes.data for r in reps])
    lib(prec).orc_average(arr, len(reps), reps[0].size)


# ------------------------------------------------------------------ training -----------------
class Debug:
    """Batch stream for global positions [base, base+len) (DESIGN.md §2 C5-C7)."""

    def __init__(self, base: int, length: int, window: int, K: int):
        self.base, self.len = base, length
        self.keep = np.zeros(length, np.uint8)
        self.b = np.zeros(length, np.uint8)
        self.N = np.zeros(length, np.uint8)
        self.ctx = np.full((length, 2 * window), -1, np.int32)
        self.neg = np.full((length, max(K, 1)), -1, np.int32)
        self.a1neg = np.full((length, 2 * window, max(K, 1)), -1, np.int32)  # O-A1 per-input negatives
        self.c = OrcDebug(base, length, _p(self.keep, ctypes.c_uint8), _p(self.b, ctypes.c_uint8),
                          _p(self.N, ctypes.c_uint8), _p(self.ctx, ctypes.c_int32), _p(self.neg, ctypes.c_int32),
                          _p(self.a1neg, ctypes.c_int32))


def make_params(V, D, window, K, alpha0, t, seed, L, epochs, n_global, world=1, lr_quantum=10_000,
                allow_target_negative=False, algorithm=0) -> OrcParams:
    return OrcParams(V, D, window, K, alpha0, t, seed, L, int(allow_target_negative), lr_quantum, epochs,
                     n_global, world, algorithm)


def train_range(prm: OrcParams, thr, P, ids, ids_base, shard_start, n_local, e, chunk_lo, chunk_hi,
                M_in, M_out, stats: OrcStats, dbg: Debug | None = None, prec="f64") -> None:
    ids = np.ascontiguousarray(ids, np.int32)
    mi = M_in.ctypes.data if M_in is not None else None      # None: batch stream only
    mo = M_out.ctypes.data if M_out is not None else None
    rc = lib(prec).orc_train_range(ctypes.byref(prm), _p(thr, ctypes.c_uint64), _p(P, ctypes.c_uint64),
                                   _p(ids, ctypes.c_int32), ids_base, ids.size, shard_start, n_local, e,
                                   chunk_lo, chunk_hi, mi, mo, ctypes.byref(stats),
                                   ctypes.byref(dbg.c) if dbg is not None else None)
    if rc != 0:
        raise ValueError("orc_train_range: bad arguments")


def train_range_hogwild(prm: OrcParams, thr, P, ids, ids_base, shard_start, n_local, e, chunk_lo, chunk_hi,
                        M_in, M_out, stats: OrcStats, threads: int, prec="f64") -> None:
    """CPU TIMING BASELINE ONLY: `threads` Hogwild threads over contiguous chunk slices of the
    same model; the result depends on the interleaving — never a parity value."""
    ids = np.ascontiguousarray(ids, np.int32)
    lib(prec).orc_train_range_hogwild(ctypes.byref(prm), _p(thr, ctypes.c_uint64), _p(P, ctypes.c_uint64),
                                      _p(ids, ctypes.c_int32), ids_base, ids.size, shard_start, n_local, e,
                                      chunk_lo, chunk_hi, M_in.ctypes.data, M_out.ctypes.data, ctypes.byref(stats),
                                      threads)


def train(ids, V, D, window, K, alpha0, t, seed, L, epochs=1, prec="f64", lr_quantum=10_000,
          allow_target_negative=False, algorithm=0, debug: tuple | None = None, model=None):
    """Full sequential O-HB (or O-A1) run: counts -> thresholds -> sampler -> init -> epochs.

    Returns (M_in, M_out, stats dict, Debug|None). `debug=(base, len)` records the batch stream.
    `model=(M_in, M_out)` continues from given fp32 matrices instead of the contract init.
    """
    ids = np.ascontiguousarray(ids, np.int32)
    n = ids.size
    dt = real_dtype(prec)
    if model is None:
        mi, mo = init(V, D, seed)
    else:
        mi, mo = model
    M_in, M_out = np.ascontiguousarray(mi, dt).copy(), np.ascontiguousarray(mo, dt).copy()
    st = OrcStats()
    dbg = Debug(debug[0], debug[1], window, K) if debug else None
    if n == 0:
        return M_in, M_out, st.as_dict(), dbg
    c = counts(ids, V)
    thr = thresholds(c, n, t)
    P = sampler(c)
    prm = make_params(V, D, window, K, alpha0, t, seed, L, epochs, n, 1, lr_quantum, allow_target_negative,
                      algorithm)
    nchunks = (n + L - 1) // L
    for e in range(epochs):
        train_range(prm, thr, P, ids, 0, 0, n, e, 0, nchunks, M_in, M_out, st, dbg, prec)
    return M_in, M_out, st.as_dict(), dbg


def batches(ids, V, window, K, t, seed, L, debug, epoch=0, allow_target_negative=False, counts_global=None,
            ids_base=0, n_global=None):
    """Batch stream only (rows a1/a2: keep, b, ctx, negatives) for global positions `debug` =
    (base, len), without running the SGD step. `ids` holds positions [ids_base, ids_base+len);
    thresholds and sampler come from `counts_global` (default: counts of `ids`)."""
    ids = np.ascontiguousarray(ids, np.int32)
    n = ids.size if n_global is None else n_global
    c = counts(ids, V) if counts_global is None else counts_global
    thr, P = thresholds(c, n, t), sampler(c)
    prm = make_params(V, 4, window, K, 0.025, t, seed, L, 1, n, 1, 10_000, allow_target_negative, 0)
    dbg = Debug(debug[0], debug[1], window, K)
    st = OrcStats()
    lo = debug[0] // L
    hi = (debug[0] + debug[1] + L - 1) // L
    train_range(prm, thr, P, ids, ids_base, 0, n, epoch, lo, hi, None, None, st, dbg)
    return dbg
