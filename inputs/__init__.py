"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic here).

The paper trains on the One Billion Word benchmark (Sec. "Experiments"), which
is not in this container; the corpora below stand in for it with the shapes BASELINE.json's
configs name (DESIGN.md §"Input recipe"). `gen.c` holds the generator; this file is its
ctypes wrapper plus the config table.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SO = os.path.join(_HERE, "libw2v_inputs.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", _SRC, "-o", _SO, "-lm"])
    return _SO


_SRC_CUDA = os.path.join(_HERE, "gen_cuda.cu")
_SO_CUDA = os.path.join(_HERE, "libw2v_inputs_cuda.so")


def build_cuda(force: bool = False) -> str:
    """The on-device copy of the generator (gen_cuda.cu), cross-compiled for sm_100a."""
    if force or not os.path.exists(_SO_CUDA) or os.path.getmtime(_SO_CUDA) < os.path.getmtime(_SRC_CUDA):
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", _SRC_CUDA, "-o", _SO_CUDA])
    return _SO_CUDA


_lib = None
_lib_cuda = None


def lib_cuda():
    global _lib_cuda
    if _lib_cuda is None:
        _lib_cuda = ctypes.CDLL(build_cuda())
        vp, i64, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        _lib_cuda.gen_cuda_guide.argtypes = [vp, i64, ctypes.c_int, ctypes.c_int, vp, vp]
        _lib_cuda.gen_cuda_iid.argtypes = [u64, vp, i64, vp, ctypes.c_int, i64, i64, vp, vp]
        _lib_cuda.gen_cuda_planted.argtypes = [u64, i64, i64, i64, vp, vp, vp, i64, i64, vp, vp]
    return _lib_cuda


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        _lib.gen_philox4x32_10.argtypes = [u32p, u32p, u32p]
        _lib.gen_zipf_prefix.argtypes = [ctypes.c_int64, ctypes.c_double, u64p]
        _lib.gen_planted_tables.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_int64, u64p, u64p, i64p]
        _lib.gen_iid.argtypes = [ctypes.c_uint64, u64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, i32p, ctypes.c_int]
        _lib.gen_planted.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, u64p, u64p,
                                     i64p, ctypes.c_int64, ctypes.c_int64, i32p, ctypes.c_int]
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def default_threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


@dataclass
class Corpus:
    """A generated corpus description; `tokens(i0, n)` materialises any slice."""
    kind: str          # "iid" | "planted"
    V: int
    s: float
    seed: int
    C: int = 0
    Lg: int = 20
    _tables: tuple = field(default=None, repr=False)

    def _prep(self):
        if self._tables is None:
            L = lib()
            if self.kind == "iid":
                pre = np.zeros(self.V + 1, np.uint64)
                L.gen_zipf_prefix(self.V, self.s, _p(pre, ctypes.c_uint64))
                self._tables = (pre,)
            else:
                cl = np.zeros(self.C + 1, np.uint64)
                mem = np.zeros(self.V + self.C, np.uint64)
                off = np.zeros(self.C + 1, np.int64)
                rc = L.gen_planted_tables(self.V, self.s, self.C, _p(cl, ctypes.c_uint64),
                                          _p(mem, ctypes.c_uint64), _p(off, ctypes.c_int64))
                assert rc == 0
                self._tables = (cl, mem, off)
        return self._tables

    def tokens(self, i0: int, n: int, threads: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        t = self._prep()
        if out is None:
            out = np.empty(n, np.int32)
        assert out.dtype == np.int32 and out.size >= n and out.flags.c_contiguous
        th = default_threads() if threads is None else threads
        if self.kind == "iid":
            lib().gen_iid(self.seed, _p(t[0], ctypes.c_uint64), self.V, i0, n, _p(out, ctypes.c_int32), th)
        else:
            lib().gen_planted(self.seed, self.V, self.C, self.Lg, _p(t[0], ctypes.c_uint64), _p(t[1], ctypes.c_uint64),
                              _p(t[2], ctypes.c_int64), i0, n, _p(out, ctypes.c_int32), th)
        return out

    def tokens_cuda(self, i0: int, n: int, out):
        """Tokens i0 .. i0+n-1 generated on the GPU into the int32 CUDA tensor `out` (torch), on
        torch's current stream; bit-identical to tokens() (integer-only kernel over the same
        host-built u64 tables)."""
        import torch
        assert out.is_cuda and out.dtype == torch.int32 and out.is_contiguous() and out.numel() >= n
        t = self._prep()
        dev = out.device
        st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        L = lib_cuda()
        if self.kind == "iid":
            pre = torch.from_numpy(t[0].view(np.int64)).to(dev)
            Z = int(t[0][self.V])
            bits = max(1, int(2 * self.V - 1).bit_length())
            shift = max(0, Z.bit_length() - bits)
            guide = torch.empty((1 << bits) + 1, dtype=torch.int32, device=dev)
            rc = L.gen_cuda_guide(pre.data_ptr(), self.V, bits, shift, guide.data_ptr(), st)
            rc = rc or L.gen_cuda_iid(self.seed, pre.data_ptr(), self.V, guide.data_ptr(), shift, i0, n,
                                      out.data_ptr(), st)
        else:
            cl = torch.from_numpy(t[0].view(np.int64)).to(dev)
            mem = torch.from_numpy(t[1].view(np.int64)).to(dev)
            off = torch.from_numpy(t[2]).to(dev)
            rc = L.gen_cuda_planted(self.seed, self.V, self.C, self.Lg, cl.data_ptr(), mem.data_ptr(), off.data_ptr(),
                                    i0, n, out.data_ptr(), st)
        torch.cuda.current_stream(dev).synchronize()
        if rc != 0:
            raise RuntimeError(f"gen_cuda launch failed: cudaError {rc}")
        return out

    def zipf_weights(self) -> np.ndarray:
        """Quantised per-word weights zq[w] (the exact marginal of the generator)."""
        if self.kind == "iid":
            return np.diff(self._prep()[0])
        cl, mem, off = self._prep()
        zq = np.empty(self.V, np.uint64)
        for c in range(self.C):
            M = (self.V - 1 - c) // self.C + 1
            zq[c::self.C][:M] = np.diff(mem[off[c]:off[c] + M + 1])
        return zq


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index 1..5). `L` is the training chunk length."""
    idx: int
    V: int
    D: int
    n: int
    window: int
    K: int
    t: float
    alpha: float
    epochs: int
    seed: int
    kind: str
    s: float
    C: int
    L: int

    def corpus(self) -> Corpus:
        return Corpus(self.kind, self.V, self.s, self.seed, self.C, self.L)


# BASELINE.json "configs". cfg2/cfg3 use the planted generator with
# reading B; sentence length 20 = training chunk length L.
CONFIGS = {
    1: Config(1, 1_000, 32, 20_000, 2, 3, 0.0, 0.025, 1, 1001, "iid", 1.0, 0, 1000),
    2: Config(2, 71_000, 300, 17_000_000, 5, 5, 1e-4, 0.025, 1, 1002, "planted", 1.07, 1_000, 20),
    3: Config(3, 1_000_000, 300, 800_000_000, 5, 5, 1e-4, 0.025, 1, 1003, "planted", 1.07, 10_000, 20),
    4: Config(4, 1_000_000, 128, 800_000_000, 8, 15, 1e-5, 0.025, 1, 1004, "iid", 1.07, 0, 1000),
    5: Config(5, 4_000_000, 300, 8_000_000_000, 5, 5, 1e-4, 0.025, 1, 1005, "iid", 1.05, 0, 1000),
}


def philox4x32_10(ctr, key) -> tuple:
    """The generator's own Philox block (exposed only for the known-answer test)."""
    a = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().gen_philox4x32_10(_p(a, ctypes.c_uint32), _p(k, ctypes.c_uint32), _p(o, ctypes.c_uint32))
    return tuple(int(x) for x in o)
