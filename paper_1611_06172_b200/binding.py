"""Thin ctypes binding of libw2v.so (include/w2v.h). Argument marshalling only: every step of
the path runs in the library's CUDA kernels. Same names as the C-ABI, minus the `w2v_` prefix.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); pointers are passed as-is
and the library classifies them. There is no CPU fallback: if libw2v.so is missing this module
raises at import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_SO = os.environ.get("W2V_LIBRARY") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libw2v.so")
if not os.path.exists(_SO):
    raise ImportError(f"{_SO} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
_lib = ctypes.CDLL(_SO)

OK, EINVAL, ESTATE, ENOMEM, ECUDA, ENCCL, ENUMERIC, EPEER = 0, -1, -2, -3, -4, -5, -6, -7


class Stats(ctypes.Structure):
    _fields_ = [("words", ctypes.c_int64), ("targets", ctypes.c_int64), ("row_touches", ctypes.c_int64),
                ("loss_pairs", ctypes.c_int64), ("loss_sum", ctypes.c_double), ("syncs", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("ms_total", ctypes.c_double), ("ms_step", ctypes.c_double),
                ("ms_setup", ctypes.c_double), ("ms_sync", ctypes.c_double), ("ms_h2d", ctypes.c_double),
                ("step_launches", ctypes.c_int64), ("bytes_row", ctypes.c_int64),
                ("loss_tail_sum", ctypes.c_double), ("loss_tail_pairs", ctypes.c_int64), ("kernel", ctypes.c_int64),
                ("ms_batch", ctypes.c_double), ("l2_window_bytes", ctypes.c_int64), ("l2_carve_bytes", ctypes.c_int64),
                ("syncs_hot", ctypes.c_int64), ("units_per_sm", ctypes.c_int64),
                ("row_touches_cold", ctypes.c_int64), ("cold_from_row", ctypes.c_int64),
                ("bytes_moved", ctypes.c_int64), ("sync_path", ctypes.c_int64),
                ("sync_floats_owned", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp = ctypes.c_void_p
_lib.w2v_init.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_float,
                          ctypes.c_float, ctypes.c_uint64]
_lib.w2v_set_option.argtypes = [ctypes.c_char_p, ctypes.c_int64]
_lib.w2v_set_stream.argtypes = [_vp]
_lib.w2v_train.argtypes = [_vp, ctypes.c_int64, ctypes.c_int32]
_lib.w2v_sync.argtypes = []
_lib.w2v_prefetch.argtypes = [_vp, ctypes.c_int64]
_lib.w2v_get_embeddings.argtypes = [ctypes.c_int32, _vp]
_lib.w2v_set_embeddings.argtypes = [ctypes.c_int32, _vp]
_lib.w2v_get_stats.argtypes = [ctypes.POINTER(Stats)]
_lib.w2v_debug_batches.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.w2v_debug_alg1_negatives.argtypes = [_vp]
_lib.w2v_dist_unique_id.argtypes = [_vp]
_lib.w2v_dist_init.argtypes = [ctypes.c_int32, ctypes.c_int32, _vp]
_lib.w2v_dist_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                               ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
_lib.w2v_dist_plan.restype = ctypes.c_int64
_lib.w2v_dist_sync_slice.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.POINTER(ctypes.c_int64)]
_lib.w2v_finalize.argtypes = []
_lib.w2v_last_error.restype = ctypes.c_char_p


class W2VError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"w2v error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc < 0:
        raise W2VError(rc, _lib.w2v_last_error().decode())
    return rc


_dims = {}   # V, D, window, K of the live context (set by init): argument checks only


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):          # torch.Tensor (host or device)
        if not a.is_contiguous():
            raise ValueError("array must be contiguous")
        return a.data_ptr()
    if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
        raise ValueError("array must be a C-contiguous numpy array or a contiguous torch tensor")
    return a.ctypes.data


def _dtype_name(a) -> str:
    return str(a.dtype).replace("torch.", "")


def _numel(a) -> int:
    return int(a.numel()) if hasattr(a, "numel") else int(a.size)


def _checked(a, dtype: str, need: int, what: str):
    """Pointer of `a` after checking its element type and that it holds >= `need` elements: the
    library sees only a pointer, so an int64 corpus or a short buffer would be misread."""
    if a is None:
        raise ValueError(f"{what}: array is None")
    if _dtype_name(a) != dtype:
        raise TypeError(f"{what}: dtype {_dtype_name(a)}, expected {dtype}")
    if _numel(a) < need:
        raise ValueError(f"{what}: {_numel(a)} elements, need >= {need}")
    return _ptr(a)


def library_path() -> str:
    return _SO


def init(V, D, window, K, alpha, subsample, seed):
    rc = _check(_lib.w2v_init(V, D, window, K, alpha, subsample, seed))
    _dims.update(V=int(V), D=int(D), window=int(window), K=int(K))
    return rc


def set_option(key: str, value: int):
    return _check(_lib.w2v_set_option(key.encode(), int(value)))


def set_stream(stream_handle):
    return _check(_lib.w2v_set_stream(stream_handle))


def train(corpus_ids, n_tokens=None, epochs=1):
    n = _numel(corpus_ids) if n_tokens is None else int(n_tokens)
    return _check(_lib.w2v_train(_checked(corpus_ids, "int32", n, "train corpus_ids"), n, epochs))


def prefetch(corpus_ids, n_tokens=None):
    """w2v_prefetch: start the host->device copy of a host corpus on the copy stream."""
    n = _numel(corpus_ids) if n_tokens is None else int(n_tokens)
    return _check(_lib.w2v_prefetch(_checked(corpus_ids, "int32", n, "prefetch corpus_ids"), n))


def sync():
    return _check(_lib.w2v_sync())


def _model_elems() -> int:
    return _dims.get("V", 0) * _dims.get("D", 0)


def get_embeddings(which, dst):
    return _check(_lib.w2v_get_embeddings(which, _checked(dst, "float32", _model_elems(), "get_embeddings dst")))


def set_embeddings(which, src):
    return _check(_lib.w2v_set_embeddings(which, _checked(src, "float32", _model_elems(), "set_embeddings src")))


def get_stats() -> dict:
    s = Stats()
    _check(_lib.w2v_get_stats(ctypes.byref(s)))
    return s.as_dict()


def debug_batches(keep=None, b=None, N=None, ctx=None, neg=None):
    """Buffers sized for the recorded window (option debug_len): u8 keep/b/N [len], int32
    ctx [len][2*window], int32 neg [len][max(K,1)]; any may be None."""
    def chk(a, dt, what):
        if a is not None and _dtype_name(a) != dt:
            raise TypeError(f"debug_batches {what}: dtype {_dtype_name(a)}, expected {dt}")
        return _ptr(a)
    return _check(_lib.w2v_debug_batches(chk(keep, "uint8", "keep"), chk(b, "uint8", "b"), chk(N, "uint8", "N"),
                                         chk(ctx, "int32", "ctx"), chk(neg, "int32", "neg")))


def debug_alg1_negatives(neg):
    if _dtype_name(neg) != "int32":
        raise TypeError("debug_alg1_negatives: int32 buffer expected")
    return _check(_lib.w2v_debug_alg1_negatives(_ptr(neg)))


def dist_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.w2v_dist_unique_id(ctypes.cast(buf, _vp)))
    return bytes(buf)


def dist_init(rank, world, uid: bytes | None):
    buf = None
    if uid is not None:
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    return _check(_lib.w2v_dist_init(rank, world, ctypes.cast(buf, _vp) if buf is not None else None))


def dist_plan(n_global, L, world, rank, sync_period_words):
    """[(chunk_lo, chunk_hi), ...] sync intervals of `rank` (C13); pure host code."""
    cap = 1 << 16
    out = (ctypes.c_int64 * (3 + 2 * cap))()
    J = _check(_lib.w2v_dist_plan(n_global, L, world, rank, sync_period_words, out, cap))
    return [(out[3 + 2 * k], out[4 + 2 * k]) for k in range(min(J, cap))]


def dist_sync_slice(off, n, world, rank):
    """(s0, a0, a1, s1): rank's floats of an averaged range in the C17 device average; pure host."""
    out = (ctypes.c_int64 * 4)()
    _check(_lib.w2v_dist_sync_slice(off, n, world, rank, out))
    return tuple(out)


def dist_shard(n_global, L, world, rank):
    out = (ctypes.c_int64 * 3)()
    _check(_lib.w2v_dist_plan(n_global, L, world, rank, 1 << 62, out, 0))
    return out[0], out[1]


def finalize():
    _dims.clear()
    return _check(_lib.w2v_finalize())
