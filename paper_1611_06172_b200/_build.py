"""Build libw2v.so in-tree with nvcc for sm_100a (used by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libw2v.so")
BUILD = os.path.join(PKG, "build")
SOURCES = ["setup.cu", "batch.cu", "hogbatch.cu", "hogbatch_ring.cu", "hogbatch_win.cu", "hogbatch_wg.cu", "alg1.cu", "sync.cu", "sync_dev.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# IEEE division/sqrt are required for the bit-exact contract (C2, C9): no fast-math.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
         "-I", os.path.join(ROOT, "include")]


def _nccl_include() -> str:
    """The NCCL headers of the nvidia-nccl wheel torch loads at run time (2.28: the symmetric-memory
    device API sync_dev.cu uses; /usr/include holds an older 2.27 without it)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for d in (spec.submodule_search_locations or []) if spec else []:
        inc = os.path.join(d, "include")
        if os.path.exists(os.path.join(inc, "nccl_device.h")):
            return inc
    raise RuntimeError("nvidia-nccl wheel headers (nccl_device.h, NCCL >= 2.28) not found")


FLAGS += ["-I", _nccl_include()]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "w2v.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list | None = None) -> str:
    """Build libw2v.so (or an experiment variant `out` with `extra` nvcc flags)."""
    target = out or SO
    if out is None and not force and not _stale():
        return SO
    os.makedirs(BUILD, exist_ok=True)
    tag = "" if out is None else os.path.basename(out).replace(".so", "") + "_"

    def compile_one(src):
        obj = os.path.join(BUILD, tag + src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *(extra or []), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        res = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in res]
    tmp = target + ".tmp"
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, target)
    if verbose:
        for _, err in res:
            print(err)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
