"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol that
include/w2v.h declares, rejects out-of-order calls, and its pure-host C13 planner agrees with
the oracle's replica protocol."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding():
    import __graft_entry__
    __graft_entry__.build_library()
    from paper_1611_06172_b200 import binding as b
    return b


def test_exports_every_declared_symbol(binding):
    hdr = open(os.path.join(ROOT, "include", "w2v.h")).read()
    declared = set(re.findall(r"\b(w2v_[a-z_]+)\s*\(", hdr))
    assert {"w2v_init", "w2v_train", "w2v_sync", "w2v_get_embeddings"} <= declared
    for name in declared:
        assert hasattr(binding._lib, name), name


def test_out_of_order_calls_rejected(binding):
    with pytest.raises(binding.W2VError) as e:
        binding.set_option("mode", 1)
    assert e.value.code == binding.ESTATE
    with pytest.raises(binding.W2VError) as e:
        binding._check(binding._lib.w2v_train(None, 10, 1))
    assert e.value.code == binding.ESTATE
    with pytest.raises(binding.W2VError) as e:
        binding.get_stats()
    assert e.value.code == binding.ESTATE
    assert binding.finalize() == 0          # safe when not initialised


def test_init_argument_validation(binding):
    for args in [(0, 32, 2, 3), (10, 30, 2, 3), (10, 32, 0, 3), (10, 32, 2, -1), (10, 32, 2, 32), (10, 1024, 2, 3)]:
        with pytest.raises(binding.W2VError) as e:
            binding.init(*args, 0.025, 0.0, 1)
        assert e.value.code == binding.EINVAL
    with pytest.raises(binding.W2VError):
        binding.init(10, 32, 2, 3, 0.0, 0.0, 1)
    with pytest.raises(binding.W2VError):
        binding.init(10, 32, 2, 3, 0.025, -1.0, 1)


def test_dist_plan_matches_oracle_protocol(binding):
    from oracle import dist as odist
    for n, L, W, P in [(23_456, 50, 2, 2_000), (1_000_000, 20, 8, 1 << 16), (999, 1000, 3, 100),
                       (800_000_000, 20, 8, 1 << 20), (8_000_000_000, 1000, 8, 1 << 18)]:
        for r in range(W):
            assert binding.dist_plan(n, L, W, r, P)[:64] == odist.sync_intervals(n, L, W, r, P)[:64]
            lo, hi = odist.shard_chunks(n, L, W, r)
            assert binding.dist_shard(n, L, W, r) == (lo * L, min(hi * L, n))
    with pytest.raises(binding.W2VError):
        binding.dist_plan(10, 0, 1, 0, 5)


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: importing the binding with the CUDA library missing raises ImportError."""
    import subprocess
    import sys
    env = dict(os.environ, W2V_LIBRARY=str(tmp_path / "missing" / "libw2v.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_1611_06172_b200.binding"], capture_output=True,
                       text=True, env=env, cwd=ROOT, timeout=120)
    assert r.returncode != 0 and "ImportError" in r.stderr and "no CPU fallback" in r.stderr


def test_binding_rejects_wrong_dtypes_and_sizes(binding):
    """The binding checks element type and size before the C-ABI sees a bare pointer (ADVICE r01:
    an int64 corpus would be read as int32 pairs [id, 0, id, 0, ...], all valid ids)."""
    import numpy as np
    import torch
    with pytest.raises(TypeError):
        binding.train(np.arange(10, dtype=np.int64), 10, 1)
    with pytest.raises(TypeError):
        binding.train(torch.arange(10, dtype=torch.int64), 10, 1)
    with pytest.raises(ValueError):
        binding.train(np.arange(10, dtype=np.int32), 11, 1)          # n beyond the buffer
    with pytest.raises(ValueError):
        binding.train(np.arange(20, dtype=np.int32)[::2], 10, 1)     # not contiguous
    with pytest.raises(TypeError):
        binding.get_embeddings(0, np.zeros((4, 4), np.float64))
    with pytest.raises(TypeError):
        binding.set_embeddings(1, torch.zeros(4, 4, dtype=torch.float16))
    with pytest.raises(TypeError):
        binding.debug_batches(keep=np.zeros(4, np.int32))
    with pytest.raises(TypeError):
        binding.debug_alg1_negatives(np.zeros(4, np.int64))
    # a well-typed call reaches the library (which then reports its own state error)
    with pytest.raises(binding.W2VError) as e:
        binding.train(np.arange(10, dtype=np.int32), 10, 1)
    assert e.value.code == binding.ESTATE


def test_error_codes_match_header(binding):
    hdr = open(os.path.join(ROOT, "include", "w2v.h")).read()
    codes = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define W2V_(E[A-Z]+|OK)\s+\(?(-?\d+)\)?", hdr)}
    for name, val in codes.items():
        assert getattr(binding, name) == val, name
    assert codes["EPEER"] == -7


def test_dist_sync_slices_tile_every_range(binding):
    """C17 (sync_dev.cu): the W ranks' slices of an averaged range tile it exactly, in rank order,
    balanced to one float, each split into a scalar head of < 4 floats up to a 16-B boundary, a
    float4 body on 16-B boundaries and a scalar tail of < 4 floats — for the model ranges the
    library averages (multiples of 2*Ds floats) and for arbitrary offsets and sizes."""
    import random
    rng = random.Random(7)
    cases = [(0, 2 * 300 * 1_000_000, 8), (0, 2 * 320 * 1_000, 1), (2 * 300 * 5000, 2 * 300 * 45_000, 3),
             (0, 0, 4), (0, 3, 8), (5, 7, 2), (1, 1, 1)]
    cases += [(rng.randrange(0, 1 << 20), rng.randrange(0, 1 << 22), rng.randrange(1, 9)) for _ in range(300)]
    for off, n, W in cases:
        prev = off
        sizes = []
        for r in range(W):
            s0, a0, a1, s1 = binding.dist_sync_slice(off, n, W, r)
            assert s0 == prev and s0 <= a0 <= a1 <= s1, (off, n, W, r)
            assert (a1 - a0) % 4 == 0 and (a0 % 4 == 0 or a0 == s1)
            assert a0 - s0 < 4 and (s1 - a1 < 4), (off, n, W, r, s0, a0, a1, s1)
            if a1 > a0:
                assert a0 % 4 == 0
            sizes.append(s1 - s0)
            prev = s1
        assert prev == off + n and max(sizes) - min(sizes) <= 1
    with pytest.raises(binding.W2VError):
        binding.dist_sync_slice(0, 10, 2, 2)
